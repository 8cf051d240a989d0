"""Where does a tiny (C1) query spend its time?  Host-side profile of one party thread + kernel counts."""
import sys, time, collections, threading
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2209_03526_b200 import workloads, _lib
from paper_2209_03526_b200.graphs import encrypt_graph, device_trio
from paper_2209_03526_b200.query import load_query, gen_token
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
from paper_2209_03526_b200.engine import sec_match, EngineConfig, open_results
import paper_2209_03526_b200._lib as L

g = workloads.tiny_graph(1); q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng); d = device_trio(shares)
tokens = gen_token(load_query(q, schema), schema, rng)
calls = collections.Counter(); ctime = collections.Counter()
orig = L.call
lock = threading.Lock()
def counting(name, *a):
    t = time.perf_counter(); r = orig(name, *a)
    with lock:
        calls[name] += 1; ctime[name] += time.perf_counter() - t
    return r
L.call = counting
import paper_2209_03526_b200.engine as E, paper_2209_03526_b200.shuffle as S, paper_2209_03526_b200.rss as R, paper_2209_03526_b200.fss as F, paper_2209_03526_b200.prf as P
for m in (E, S, R, F, P):
    if hasattr(m, "_lib"): m._lib.call = counting
def one():
    rts = local_runtimes(make_session_configs(b"\x5a" * 16))
    res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig()), rts)
    return open_results(res[:2], schema)
for _ in range(3): one()
calls.clear(); ctime.clear()
t = time.perf_counter(); one(); el = time.perf_counter() - t
print(f"one query: {el*1e3:.1f} ms; C-ABI calls (all 3 parties): {sum(calls.values())}")
for k, v in calls.most_common(): print(f"  {k:32s} {v:5d} calls  {ctime[k]*1e3:8.2f} ms (sum over threads)")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    one()
ka = prof.key_averages()
cuda_k = [e for e in ka if e.device_type is not None and "cuda" in str(e.device_type).lower()]
print("top host ops:")
print(ka.table(sort_by="cpu_time_total", row_limit=25))
