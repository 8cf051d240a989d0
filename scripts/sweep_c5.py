"""BASELINE configs[4]'s sweep through bench.py's own C5 legs (shuffle; fetch
of 1% / 10% / 100% of 129-bit rows), every size gated bit-exact:
python scripts/sweep_c5.py [min log2] [max log2] [step]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench_configs as bc  # noqa: E402
from paper_2209_03526_b200 import _lib  # noqa: E402

lo, hi, step = (int(x) for x in (sys.argv[1:4] + ["16", "28", "2"][len(sys.argv[1:4]):]))
_lib.check(_lib.load().ogm_init())
print(f"{'rows':>10s} {'shuffle ms':>11s} {'frac':>5s} | {'fetch 1% ms':>11s} {'frac':>5s} {'10% ms':>8s} {'frac':>5s} "
      f"{'100% ms':>8s} {'frac':>5s} | gates")
for lg in range(lo, hi + 1, step):
    sh = bc.c5_shuffle_leg(lg, 10, 3)
    fe = bc.c5_fetch_leg(lg, 10, 3)
    rows = 1 << lg
    frac = lambda e, per_row: per_row * rows / (e["ms"] * 1e-3) / 1e9 / bc.HBM_PEAK  # noqa: E731
    ok = all(sh["gate"].values()) and all(all(f["gate"].values()) for f in fe)
    cells = " ".join(f"{f['ms']:8.3f} {frac(f, f['algorithmic_bytes_per_row']):5.2f}" for f in fe)
    print(f"{'2^' + str(lg):>10s} {sh['ms']:11.3f} {frac(sh, 240):5.2f} | {cells} | {'ok' if ok else 'FAIL'}",
          flush=True)
    torch.cuda.empty_cache()
