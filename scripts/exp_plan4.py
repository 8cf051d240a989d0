"""ncu target: planned gather at 2^lg x 16 B for given (window MB, tile rows, repeats) configs."""
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan

_lib.check(_lib.load().ogm_init())
lg = int(sys.argv[1])
rows = 1 << lg
M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
R = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
idx = torch.randperm(rows, device="cuda").to(torch.int32)
out = torch.empty_like(M)
inter = torch.empty_like(M)
for cfg in sys.argv[2:]:
    wmb, tr, rep = map(int, cfg.split(":"))
    plan = GatherPlan(idx, 4, window_bytes=wmb << 20, tile_rows=tr)
    torch.cuda.synchronize()
    for _ in range(rep):
        plan.run(out, m1=M, r=R, inter=inter)
    torch.cuda.synchronize()
    del plan
