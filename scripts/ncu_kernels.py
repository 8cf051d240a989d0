"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per launch."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr, data = None, collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            data[(int(d["ID"]), d["Kernel Name"].split("(")[0])].append((d["Metric Name"], d["Metric Value"]))
    print(path)
    for (i, k), v in sorted(data.items()):
        m = {a: float(b.replace(",", "")) for a, b in v}
        t = m["gpu__time_duration.sum"]
        rd, wr = m.get("dram__bytes_read.sum", 0), m.get("dram__bytes_write.sum", 0)
        print(f"  {i:4d} {k:32s} {t / 1e3:9.1f} us  read {rd / 1e6:9.1f} MB  write {wr / 1e6:9.1f} MB  {(rd + wr) / t:7.0f} GB/s")
