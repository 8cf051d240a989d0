"""Print one line per kernel launch from an ncu --csv --metrics log:
python scripts/ncu_table.py LOG [--rows N] [--last K].  With --rows, DRAM
traffic is per row of the workload (B/row) and a total line follows; --last
keeps the last K launches (one iteration of a repeated step)."""
import argparse
import csv
from collections import defaultdict

ap = argparse.ArgumentParser()
ap.add_argument("log")
ap.add_argument("--rows", type=int, default=0)
ap.add_argument("--last", type=int, default=0)
args = ap.parse_args()
rows = list(csv.reader(l for l in open(args.log) if l.startswith('"')))
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
d = defaultdict(dict)
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("void ", "").replace("ogm::", "")[:40]
    d[(int(r[ii]), name)][r[mi]] = r[vi].replace(",", "")
items = sorted(d.items())[-args.last:] if args.last else sorted(d.items())
tt = tb = 0.0
for (i, k), v in items:
    t = float(v.get("gpu__time_duration.sum", 0))
    rd = float(v.get("dram__bytes_read.sum", 0))
    wr = float(v.get("dram__bytes_write.sum", 0))
    tt, tb = tt + t, tb + rd + wr
    if args.rows:
        print(f"{i:5d} {k:40s} {t / 1e3:9.1f} us  R {rd / args.rows:6.1f} W {wr / args.rows:6.1f} B/row  "
              f"{(rd + wr) / max(t, 1):6.0f} GB/s")
    else:
        print(f"{i:3d} {k:40s} {t / 1e3:8.3f} us  rd {rd / 1e9:6.2f} GB  wr {wr / 1e9:6.2f} GB  "
              f"{(rd + wr) / max(t, 1):7.0f} GB/s  L2hit {v.get('lts__t_sector_hit_rate.pct', '-')}")
if args.rows:
    print(f"total {tt / 1e3:.1f} us  {tb / args.rows:.1f} B/row  {tb / max(tt, 1):.0f} GB/s")
