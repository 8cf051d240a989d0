"""Timeline of one C3 online fetch (trio path): kernels vs host/runtime gaps."""
import sys, types
sys.path.insert(0, ".")
import torch
from torch.profiler import profile, ProfilerActivity
import bench_configs as bc
from paper_2209_03526_b200.trio import Trio

args = types.SimpleNamespace(rows=200_000, seed=3)
group, kiv, keq, n0, n2, want = bc.c3p_setup(args)
X = args.rows


def one(prof=None):
    trio = Trio(b"\x35" * 16)
    b_iv = trio.sec_eval(group, kiv, "a0", n0, {})
    b_eq = trio.sec_eval(group, keq, "a2", n2, {})
    flags = trio.combine([b_iv, b_eq], "ALL", "or", X)
    trio.prepare_shuffle(X, 1 + X + n0 + n2)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    if prof is not None:
        with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
            recs = trio.fetch_multi(group, flags, [])
            torch.cuda.synchronize()
        print(p.key_averages().table(sort_by="self_cpu_time_total", row_limit=25))
        p.export_chrome_trace("gpurun_out/c3p_fetch_trace.json")
    else:
        recs = trio.fetch_multi(group, flags, [])
    ev[1].record()
    torch.cuda.synchronize()
    print("fetch ms (events, no cache flush):", ev[0].elapsed_time(ev[1]))
    return recs


for _ in range(2):
    one()
one(prof=True)
