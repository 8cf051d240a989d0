"""ncu --set full target: one planned gather at 2^28 x 16 B (8 MB windows, 4096-row tiles)."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan

_lib.check(_lib.load().ogm_init())
rows = 1 << int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
R = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
idx = torch.randperm(rows, device="cuda").to(torch.int32)
out = torch.empty_like(M)
inter = torch.empty_like(M)
plan = GatherPlan(idx, 4)
torch.cuda.synchronize()
plan.run(out, m1=M, r=R, inter=inter)
torch.cuda.synchronize()
