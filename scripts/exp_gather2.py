"""Is the 16-B random row gather latency-bound?  Compare: our gather kernel,
torch advanced indexing, and 2 rows per thread via a (rows/2, 8)-word view trick."""
import sys, statistics
sys.path.insert(0, ".")
import torch
from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import gather
_lib.check(_lib.load().ogm_init())
def t(fn, n=5):
    for _ in range(2): fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    ev[0].record()
    for i in range(n): fn(); ev[i + 1].record()
    torch.cuda.synchronize()
    return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(n))
rows = 1 << 28
M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
idx = torch.randperm(rows, device="cuda").to(torch.int32)
idx64 = idx.long()
out = torch.empty_like(M)
print(f"ours            {t(lambda: gather(rows, 128, out, inner=idx, m1=M)):.3f} ms")
print(f"torch index     {t(lambda: torch.index_select(M, 0, idx64, out=out)):.3f} ms")
M2 = M.view(torch.int64).view(rows, 2)
out2 = torch.empty_like(M2)
print(f"torch index i64 {t(lambda: torch.index_select(M2, 0, idx64, out=out2)):.3f} ms")
# 32-B rows: half the rows, double width: same bytes, half the random accesses
Mh = M.view(rows // 2, 8); idxh = torch.randperm(rows // 2, device="cuda").to(torch.int32); outh = torch.empty_like(Mh)
print(f"ours 32B rows   {t(lambda: gather(rows // 2, 256, outh, inner=idxh, m1=Mh)):.3f} ms (same bytes, 2^27 rows)")
Mq = M.view(rows // 4, 16); idxq = torch.randperm(rows // 4, device="cuda").to(torch.int32); outq = torch.empty_like(Mq)
print(f"ours 64B rows   {t(lambda: gather(rows // 4, 512, outq, inner=idxq, m1=Mq)):.3f} ms (same bytes, 2^26 rows)")
