"""C5-like chain of planned gathers at 2^lg x 16 B with per-pass events:
x1 = P_a(a^b)^U; y1 = P_b(c)^V; c1 = P_c(x1)^W; r3 = P_d(y1)^c1^Z."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan

_lib.check(_lib.load().ogm_init())
rows = 1 << int(sys.argv[1])
mk = lambda: torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")  # noqa: E731
a, b, c, U, V, W, Z = (mk() for _ in range(7))
x1, y1, c1, r3, inter = (torch.empty_like(a) for _ in range(5))
plans = [GatherPlan(torch.randperm(rows, device="cuda").to(torch.int32), 4) for _ in range(4)]
steps = [(plans[0], dict(m1=a, m2=b, r=U), x1), (plans[1], dict(m1=c, r=V), y1),
         (plans[2], dict(m1=x1, r=W), c1), (plans[3], dict(m1=y1, m3=c1, m4=Z), r3)]
fresh = "fresh" in sys.argv
ballast = [torch.empty((int(x) << 30,), dtype=torch.uint8, device="cuda").fill_(1)
           for x in [a[len("ballast="):] for a in sys.argv if a.startswith("ballast=")][:1] for _ in range(1)]
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
    ev[0].record()
    for k, (pl, kw, out) in enumerate(steps):
        it = torch.empty_like(a) if fresh else inter
        pl.run(out, inter=it, passes=1, **kw)
        ev[2 * k + 1].record()
        pl.run(out, inter=it, passes=2, **kw)
        ev[2 * k + 2].record()
    torch.cuda.synchronize()
    print([round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(8)])
