"""One planned (L2-window) gather at 2^28 x 128-bit rows, for an ncu launch list."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan, gather

_lib.check(_lib.load().ogm_init())
lg, wb = int(sys.argv[1]), int(sys.argv[2]) << 20
rows = 1 << lg
M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
R = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
idx = torch.randperm(rows, device="cuda").to(torch.int32)
out = torch.empty_like(M)
inter = torch.empty_like(M)
plan = GatherPlan(idx, 4, window_bytes=wb)
gather(rows, 128, out, inner=idx, m1=M, r=R)
plan.run(out, m1=M, r=R, inter=inter)
torch.cuda.synchronize()
print("ok")
