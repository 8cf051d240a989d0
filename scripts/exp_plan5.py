"""ncu (application replay) target: 2^28 planned gather, p1 then p2 twice, then copy then p2."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan

_lib.check(_lib.load().ogm_init())
rows = 1 << 28
g = torch.Generator(device="cuda").manual_seed(5)
M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda", generator=g)
R = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda", generator=g)
idx = torch.randperm(rows, device="cuda", generator=g).to(torch.int32)
out = torch.empty_like(M)
inter = torch.empty_like(M)
tmp = torch.empty_like(M)
plan = GatherPlan(idx, 4, window_bytes=8 << 20, tile_rows=4096)
torch.cuda.synchronize()
for _ in range(2):
    plan.run(out, m1=M, r=R, inter=inter, passes=1)
    plan.run(out, m1=M, r=R, inter=inter, passes=2)
tmp.copy_(M)
plan.run(out, m1=M, r=R, inter=inter, passes=2)
torch.cuda.synchronize()
