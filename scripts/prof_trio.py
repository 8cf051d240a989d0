"""Host/GPU breakdown of one trio-path C1 query."""
import sys, time, collections
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2209_03526_b200 import workloads, _lib
from paper_2209_03526_b200.graphs import encrypt_graph, device_trio
from paper_2209_03526_b200.query import load_query, gen_token
from paper_2209_03526_b200.trio import Trio
from paper_2209_03526_b200.engine import open_results
import paper_2209_03526_b200._lib as L

g = workloads.tiny_graph(1); q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng); d = list(device_trio(shares))
tokens = list(gen_token(load_query(q, schema), schema, rng))
calls = collections.Counter(); ctime = collections.Counter()
orig = L.call
def counting(name, *a):
    t = time.perf_counter(); r = orig(name, *a); calls[name] += 1; ctime[name] += time.perf_counter() - t; return r
L.call = counting
for _ in range(3): Trio(b"\x5a" * 16).match(tokens, d)
calls.clear(); ctime.clear()
torch.cuda.synchronize(); t = time.perf_counter(); res = Trio(b"\x5a" * 16).match(tokens, d); torch.cuda.synchronize()
el = time.perf_counter() - t
print(f"trio match: {el*1e3:.2f} ms, C-ABI calls {sum(calls.values())}, time in calls {sum(ctime.values())*1e3:.2f} ms")
for k, v in calls.most_common(): print(f"  {k:32s} {v:4d}  {ctime[k]*1e3:7.2f} ms")
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    Trio(b"\x5a" * 16).match(tokens, d); torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=14))
