"""Print one line per kernel launch from an ncu --csv --metrics log."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = defaultdict(dict)
for r in rows[1:]:
    d[(int(r[ii]), r[ki].split("(")[0][:40])][r[mi]] = r[vi].replace(",", "")
for (i, k), v in sorted(d.items()):
    t = float(v.get("gpu__time_duration.sum", 0))
    rd = float(v.get("dram__bytes_read.sum", 0))
    wr = float(v.get("dram__bytes_write.sum", 0))
    print(f"{i:3d} {k:40s} {t / 1e3:8.3f} us  rd {rd / 1e9:6.2f} GB  wr {wr / 1e9:6.2f} GB  "
          f"{(rd + wr) / max(t, 1):7.0f} GB/s  L2hit {v.get('lts__t_sector_hit_rate.pct', '-')}")
