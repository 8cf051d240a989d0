"""Why is the C4 leg slower inside bench.py than standalone?"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import bench
import bench_configs
from paper_2209_03526_b200 import _lib, fss

_lib.check(_lib.load().ogm_init())
print("fresh:", round(bench_configs.c4_sec_eval(2_000_000, 1, 10, 3, 0, 1)["ms_per_step"], 3))
K = 1 << 22
gen = torch.Generator(device="cuda").manual_seed(1)
alphas = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=gen)
pts = torch.randint(-(1 << 31), 1 << 31, (K,), dtype=torch.int32, device="cuda", generator=gen)
r0 = torch.randint(0, 256, (K, 16), dtype=torch.uint8, device="cuda", generator=gen)
b0, b1 = fss.gen_batch(True, 32, alphas, r0, r0)
out = torch.empty(((K + 31) // 32,), dtype=torch.int32, device="cuda")
for _ in range(5):
    fss.eval_points(b0, pts, out)
torch.cuda.synchronize()
print("after fss eval:", round(bench_configs.c4_sec_eval(2_000_000, 1, 10, 3, 0, 1)["ms_per_step"], 3))
q = bench.query_latency(5)
print("after query latency:", round(bench_configs.c4_sec_eval(2_000_000, 1, 10, 3, 0, 1)["ms_per_step"], 3))
print("again:", round(bench_configs.c4_sec_eval(2_000_000, 1, 10, 3, 0, 1)["ms_per_step"], 3))
