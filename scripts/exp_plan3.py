"""Is a window-local random gather L2-fast with random data?  (C5 study)"""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan, gather

_lib.check(_lib.load().ogm_init())


def t(fn, n=5):
    for _ in range(2):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    ev[0].record()
    for i in range(n):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(n))


rows = 1 << 28
M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
Mc = torch.ones_like(M)
out = torch.empty_like(M)
for wlg in (16, 18, 20):
    W = 1 << wlg
    key = torch.rand(rows, device="cuda") + torch.arange(rows, device="cuda").div(W, rounding_mode="floor").float()
    idx = torch.argsort(key.double()).to(torch.int32) if False else None
    # window-local permutation: within each window of W rows, a random perm
    r = torch.randint(0, 1 << 30, (rows,), device="cuda", dtype=torch.int64)
    k = (torch.arange(rows, device="cuda") // W) * (1 << 31) + r
    idx = torch.argsort(k).to(torch.int32)
    del k, r, key
    a = t(lambda: gather(rows, 128, out, inner=idx, m1=M))
    b = t(lambda: gather(rows, 128, out, inner=idx, m1=Mc))
    print(f"window {W * 16 >> 20:3d} MB: random data {a:.3f} ms, constant data {b:.3f} ms")
idx = torch.randperm(rows, device="cuda").to(torch.int32)
print(f"full perm: random data {t(lambda: gather(rows, 128, out, inner=idx, m1=M)):.3f} ms, "
      f"constant {t(lambda: gather(rows, 128, out, inner=idx, m1=Mc)):.3f} ms")
