"""Experiment: random 16-B row gather vs L2 fetch granularity (cudaLimitMaxL2FetchGranularity)."""
import sys, statistics
sys.path.insert(0, ".")
import torch
from cuda.bindings import runtime as cudart
from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.shuffle import gather

_lib.check(_lib.load().ogm_init())
lim = cudart.cudaLimit.cudaLimitMaxL2FetchGranularity
print("initial limit", cudart.cudaDeviceGetLimit(lim))
for lg in (24, 28):
    rows = 1 << lg
    M = torch.randint(-2**31, 2**31 - 1, (rows, 4), dtype=torch.int32, device="cuda")
    perm = torch.randperm(rows, device="cuda", dtype=torch.int64).to(torch.int32)
    out = torch.empty_like(M)
    for g in (128, 64, 32, 0):
        err = cudart.cudaDeviceSetLimit(lim, g)
        got = cudart.cudaDeviceGetLimit(lim)
        for _ in range(3):
            gather(rows, 128, out, inner=perm, m1=M)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        for i in range(5):
            gather(rows, 128, out, inner=perm, m1=M)
            ev[i + 1].record()
        torch.cuda.synchronize()
        ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(5))
        print(f"2^{lg} set={g} err={err[0]} read={got} ms={ms:.3f} algo_GBps={rows*(16+4+16)/ms/1e6:.0f}")
    # sequential gather (identity) for comparison
    ident = torch.arange(rows, device="cuda", dtype=torch.int32)
    gather(rows, 128, out, inner=ident, m1=M); torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record(); gather(rows, 128, out, inner=ident, m1=M); ev[1].record(); torch.cuda.synchronize()
    print(f"2^{lg} identity ms={ev[0].elapsed_time(ev[1]):.3f} GBps={rows*36/ev[0].elapsed_time(ev[1])/1e6:.0f}")
