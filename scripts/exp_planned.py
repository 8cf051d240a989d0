"""Time the two passes of the planned gather vs the direct gather (2^24, 2^28 rows of 128 bits)."""
import sys, statistics
sys.path.insert(0, ".")
import torch
from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan, gather

_lib.check(_lib.load().ogm_init())
def t(fn, n=5):
    for _ in range(2): fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    ev[0].record()
    for i in range(n):
        fn(); ev[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(n))
for lg in (24, 28):
    rows = 1 << lg
    M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
    idx = torch.randperm(rows, device="cuda").to(torch.int32)
    out = torch.empty_like(M); inter = torch.empty_like(M)
    plan = GatherPlan(idx, 4)
    d = t(lambda: gather(rows, 128, out, inner=idx, m1=M))
    p = t(lambda: plan.run(out, m1=M, inter=inter))
    ident = torch.arange(rows, device="cuda", dtype=torch.int32)
    seq = t(lambda: gather(rows, 128, out, inner=ident, m1=M))
    # pass 1 alone: scatter to pos1; pass 2 alone via plan with identity-like q2 is not separable -> report totals
    print(f"2^{lg}: direct {d:.3f} ms  planned {p:.3f} ms  sequential-gather {seq:.3f} ms  tile={plan.tile}")
