"""Offline planned-gather construction (ogm_gather_plan + its run table) for
a random permutation of 16-byte rows: python scripts/time_gather_plan.py."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_2209_03526_b200 import _lib  # noqa: E402
from paper_2209_03526_b200.shuffle import GatherPlan  # noqa: E402

_lib.check(_lib.load().ogm_init())
for lg in (20, 24, 26, 28):
    n = 1 << lg
    idx = torch.randperm(n, device="cuda", dtype=torch.int32)
    GatherPlan(idx, 4)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        p = GatherPlan(idx, 4)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / 3 * 1e3
    print(f"2^{lg}: plan {ms:.2f} ms ({n / (ms * 1e-3) / 1e9:.2f} G rows/s)", flush=True)
    del p, idx
    torch.cuda.empty_cache()
