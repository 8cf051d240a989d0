"""Does a small L2 scrub between the passes restore the fast window pass?"""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan

_lib.check(_lib.load().ogm_init())
rows = 1 << 28
mk = lambda: torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")  # noqa: E731
M, R, M3, out, inter = mk(), mk(), mk(), mk(), mk()
plan = GatherPlan(torch.randperm(rows, device="cuda").to(torch.int32), 4)
scratch = torch.empty((512 << 20,), dtype=torch.uint8, device="cuda")
src = torch.empty_like(scratch)


def seq(label, mid):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ts = []
    for _ in range(5):
        ev[0].record()
        plan.run(out, m1=M, r=R, inter=inter, passes=1)
        ev[1].record()
        mid()
        ev[2].record()
        plan.run(out, m1=M, r=R, inter=inter, passes=2)
        ev[3].record()
        torch.cuda.synchronize()
        ts.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
    med = [round(statistics.median(t[i] for t in ts), 3) for i in range(3)]
    print(f"{label:28s} pass1 {med[0]}  mid {med[1]}  pass2 {med[2]}")


seq("nothing", lambda: None)
for mb in (32, 128, 512):
    seq(f"memset {mb} MB", lambda mb=mb: scratch[: mb << 20].zero_())
    seq(f"copy {mb} MB", lambda mb=mb: scratch[: mb << 20].copy_(src[: mb << 20]))
