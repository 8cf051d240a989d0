"""C5 gather study: direct vs L2-window planned gather at 2^28 x 16 B rows,
with per-pass timing (CUDA events, median of 5)."""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import GatherPlan, gather

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


lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
rows = 1 << lg
M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
R = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
idx = torch.randperm(rows, device="cuda").to(torch.int32)
out = torch.empty_like(M)
inter = torch.empty_like(M)
print(f"direct            {t(lambda: gather(rows, 128, out, inner=idx, m1=M, r=R)):.3f} ms")
want = out.clone()
for wb in [int(x) << 20 for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["8"])]:
    for tr in (4096,):
        plan = GatherPlan(idx, 4, window_bytes=wb, tile_rows=tr)
        tt = t(lambda: plan.run(out, m1=M, r=R, inter=inter))
        assert torch.equal(out, want)
        t1 = t(lambda: plan.run(out, m1=M, r=R, inter=inter, passes=1))
        t2 = t(lambda: plan.run(out, m1=M, r=R, inter=inter, passes=2))
        print(f"planned window {wb >> 20:2d} MB tile {tr:5d}: {tt:.3f} ms (pass 1 alone {t1:.3f}, pass 2 alone {t2:.3f})")
if len(sys.argv) > 3:
    sys.exit(0)
# alternating sequence with an event after every pass: which pass slows down?
plan = GatherPlan(idx, 4, window_bytes=8 << 20, tile_rows=4096)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(13)]
ev[0].record()
for k in range(6):
    plan.run(out, m1=M, r=R, inter=inter, passes=1)
    ev[2 * k + 1].record()
    plan.run(out, m1=M, r=R, inter=inter, passes=2)
    ev[2 * k + 2].record()
torch.cuda.synchronize()
print("alternating p1/p2 ms:", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(12)])
# p1 then p2 with a different inter buffer / out buffer
inter2 = torch.empty_like(M)
ev[0].record()
for k in range(6):
    plan.run(out, m1=M, r=R, inter=inter2 if k % 2 else inter, passes=1)
    ev[2 * k + 1].record()
    plan.run(out, m1=M, r=R, inter=inter2 if k % 2 else inter, passes=2)
    ev[2 * k + 2].record()
torch.cuda.synchronize()
print("alternating, 2 inter bufs:", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(12)])
def seq(label, before):
    ev[0].record()
    for k in range(6):
        before(k)
        ev[2 * k + 1].record()
        plan.run(out, m1=M, r=R, inter=inter, passes=2)
        ev[2 * k + 2].record()
    torch.cuda.synchronize()
    print(label, [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(12)])


tmp = torch.empty_like(M)
seq("p1(inter2) then p2(inter):", lambda k: plan.run(out, m1=M, inter=inter2, passes=1))
seq("p1 + sleep 10ms then p2:", lambda k: (plan.run(out, m1=M, inter=inter, passes=1), torch.cuda._sleep(20_000_000)))
seq("inter.copy_(tmp) then p2:", lambda k: inter.copy_(tmp))
seq("tmp.copy_(M) then p2:", lambda k: tmp.copy_(M))
