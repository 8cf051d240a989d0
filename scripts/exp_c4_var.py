"""C4 secEval run-to-run variation: per-step times over several calls."""
import sys

sys.path.insert(0, ".")
import torch

import bench_configs
from paper_2209_03526_b200 import _lib

_lib.check(_lib.load().ogm_init())
for rep in range(4):
    d = bench_configs.c4_sec_eval(2_000_000, 1 + rep, 10, 3, 0, 1)
    print(rep, round(d["ms_per_step"], 3))
    torch.cuda.empty_cache()
