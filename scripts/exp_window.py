"""Direct random gather vs planned two-pass gathers (shared-memory tiles, or
L2-sized windows of several sizes) on 128-bit rows; checks equality."""
import sys, statistics
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


for words in (4, 5):
    for lg in (20, 24, 26, 28):
        rows = 1 << lg
        M = torch.randint(-2**31, 2**31 - 1, (rows, words), dtype=torch.int32, device="cuda")
        R = torch.randint(-2**31, 2**31 - 1, (rows, words), dtype=torch.int32, device="cuda")
        idx = torch.randperm(rows, device="cuda").to(torch.int32)
        out = torch.empty_like(M)
        inter = torch.empty_like(M)
        gather(rows, 32 * words, out, inner=idx, m1=M, r=R)
        want = out.clone()
        d = t(lambda: gather(rows, 32 * words, out, inner=idx, m1=M, r=R))
        line = f"w={words} 2^{lg}: direct {d:.3f} ms"
        for wb in (None, 8 << 20, 16 << 20, 32 << 20, 64 << 20):
            plan = GatherPlan(idx, words, window_bytes=wb)
            out.zero_()
            plan.run(out, m1=M, r=R, inter=inter)
            ok = torch.equal(out, want)
            p = t(lambda: plan.run(out, m1=M, r=R, inter=inter))
            line += f" | {'smem' if wb is None else str(wb >> 20) + 'MB'} {p:.3f}{'' if ok else ' MISMATCH'}"
            del plan
        print(line, flush=True)
        del M, R, idx, out, inter, want
        torch.cuda.empty_cache()
