"""Summarise an ncu --csv launch list (time, DRAM bytes per kernel name)."""
import csv, io, collections, sys
txt = open(sys.argv[1]).read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(txt)))
agg = collections.OrderedDict()
for r in rows:
    agg.setdefault((r['ID'], r['Kernel Name'].split('(')[0][:58]), {})[r['Metric Name']] = (float(r['Metric Value'].replace(',', '')), r['Metric Unit'])
US = {'ms': 1e3, 'msecond': 1e3, 'us': 1, 'usecond': 1, 'ns': 1e-3, 'nsecond': 1e-3, 's': 1e6, 'second': 1e6}
GB = {'Gbyte': 1, 'Mbyte': 1e-3, 'Kbyte': 1e-6, 'byte': 1e-9, 'Tbyte': 1e3}
tot = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (_, name), m in agg.items():
    t = tot[name]; t[0] += 1
    v, u = m['gpu__time_duration.sum']; t[1] += v * US.get(u, 1)
    if 'dram__bytes_read.sum' in m:
        v, u = m['dram__bytes_read.sum']; t[2] += v * GB.get(u, 1)
        v, u = m['dram__bytes_write.sum']; t[3] += v * GB.get(u, 1)
allus = sum(t[1] for t in tot.values())
print(f"| kernel | launches | ms | share | DRAM rd GB | DRAM wr GB | achieved TB/s |\n|---|---|---|---|---|---|---|")
for name, (n, us, rd, wr) in sorted(tot.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"| `{name}` | {n} | {us/1e3:.2f} | {100*us/allus:.1f}% | {rd:.2f} | {wr:.2f} | {(rd+wr)/(us*1e-6)/1e3 if us else 0:.2f} |")
