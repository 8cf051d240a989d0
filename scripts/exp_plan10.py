"""Is the slow window pass a property of the buffer (physical placement)?
Pass 2 alone over 6 different `inter` buffers, 3 times each, 2^28 x 16 B."""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan

_lib.check(_lib.load().ogm_init())
rows = 1 << 28
mk = lambda: torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")  # noqa: E731
M, R, out = mk(), mk(), mk()
inters = [mk() for _ in range(6)]
plan = GatherPlan(torch.randperm(rows, device="cuda").to(torch.int32), 4)


def t(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b)


for rep in range(3):
    print([round(t(lambda: plan.run(out, m1=M, r=R, inter=it, passes=2)), 2) for it in inters])
print("r buffers:")
Rs = [mk() for _ in range(4)]
for rep in range(2):
    print([round(t(lambda: plan.run(out, m1=M, r=r_, inter=inters[0], passes=2)), 2) for r_ in Rs])
