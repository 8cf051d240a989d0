"""Pass 2 alone at 2^lg x 16 B: window size x extra streamed input (m3)."""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan

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


rows = 1 << int(sys.argv[1])
ballast = [torch.empty((int(a[8:]) << 30,), dtype=torch.uint8, device="cuda").fill_(1)
           for a in sys.argv if a.startswith("ballast=")]
mk = lambda: torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")  # noqa: E731
M, R, M3, out, inter = mk(), mk(), mk(), mk(), mk()
idx = torch.randperm(rows, device="cuda").to(torch.int32)
for wmb in (1, 2, 4, 8):
    plan = GatherPlan(idx, 4, window_bytes=wmb << 20)
    plan.run(out, m1=M, inter=inter, passes=1)
    a = t(lambda: plan.run(out, m1=M, r=R, inter=inter, passes=2))
    b = t(lambda: plan.run(out, m1=M, r=R, m3=M3, inter=inter, passes=2))
    c = t(lambda: plan.run(out, m1=M, inter=inter, passes=2))
    p1 = t(lambda: plan.run(out, m1=M, inter=inter, passes=1))
    alt = t(lambda: plan.run(out, m1=M, r=R, inter=inter))
    print(f"window {wmb} MB: pass2 r {a:.3f}  r+m3 {b:.3f}  none {c:.3f}   pass1 {p1:.3f} ms  both {alt:.3f}")
    del plan
