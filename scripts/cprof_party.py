"""cProfile of the per-party drop-in C1 query (3 party threads): where the host time goes."""
import cProfile, pstats, sys, time, threading
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2209_03526_b200 import workloads
from paper_2209_03526_b200.graphs import encrypt_graph, device_trio
from paper_2209_03526_b200.query import load_query, gen_token
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
from paper_2209_03526_b200.engine import sec_match, EngineConfig, open_results

g = workloads.tiny_graph(1); q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng); d = device_trio(shares)
tokens = gen_token(load_query(q, schema), schema, rng)


def one():
    rts = local_runtimes(make_session_configs(b"\x5a" * 16))
    res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig()), rts)
    return open_results(res[:2], schema)


for _ in range(3):
    one()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10):
    one()
torch.cuda.synchronize()
print(f"per query {100 * (time.perf_counter() - t):.2f} ms")
# profile one party's thread (cProfile is per-thread): wrap sec_match
profs = {}
def wrapped(rt):
    if rt.index != 1:  # one profiler at a time (3.12 sys.monitoring)
        return sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig())
    pr = profs.setdefault(1, cProfile.Profile())
    pr.enable()
    r = sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig())
    pr.disable()
    return r
for _ in range(5):
    rts = local_runtimes(make_session_configs(b"\x5a" * 16))
    run_trio(wrapped, rts)
pstats.Stats(profs[1]).sort_stats("tottime").print_stats(25)
pstats.Stats(profs[1]).sort_stats("cumtime").print_stats(30)
