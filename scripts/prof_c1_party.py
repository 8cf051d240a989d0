"""Host-side profile of the C1 tiny query through the per-party drop-in API
(run_trio + sec_match + open_results, as bench.py's query_latency times it):
party 1's thread and open_results profiled (cProfile allows one
active profiler per process).  python scripts/prof_c1_party.py."""
import cProfile
import pstats
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_03526_b200 import _lib, workloads  # noqa: E402
from paper_2209_03526_b200.engine import EngineConfig, open_results, sec_match  # noqa: E402
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph  # noqa: E402
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio  # noqa: E402
from paper_2209_03526_b200.query import gen_token, load_query  # noqa: E402

_lib.check(_lib.load().ogm_init())
graph = workloads.tiny_graph(1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(graph, 2, rng)
dshares = device_trio(shares)
query = load_query(workloads.tiny_query(graph, 1), schema)
tokens = gen_token(query, schema, rng)
master = b"\x5a" * 16
profs: dict = {}
party_s: dict = {1: [], 2: [], 3: []}


def party(rt, prof):
    t = time.perf_counter()
    prof = prof is True and rt.index == 1   # one profiler per process (sys.monitoring)
    if prof:
        p = profs.setdefault(rt.index, cProfile.Profile())
        p.enable()
    r = sec_match(rt, tokens[rt.index - 1], dshares[rt.index - 1], EngineConfig())
    if prof:
        p.disable()
    party_s[rt.index].append(time.perf_counter() - t)
    return r


def once(prof=False):
    rts = local_runtimes(make_session_configs(master))
    t0 = time.perf_counter()
    res = run_trio(lambda rt: party(rt, prof), rts)
    t1 = time.perf_counter()
    if prof == "open":
        po = profs.setdefault("open", cProfile.Profile())
        po.enable()
    got = open_results(res[:2], schema)[0]
    if prof == "open":
        po.disable()
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


for _ in range(20):
    once()
for k in party_s:
    party_s[k].clear()
tt = [once() for _ in range(200)]
print("median ms: run_trio %.3f  open_results %.3f  party bodies %s" % (
    1e3 * statistics.median(t[0] for t in tt), 1e3 * statistics.median(t[1] for t in tt),
    " ".join("%.3f" % (1e3 * statistics.median(v)) for v in party_s.values())))
rts = local_runtimes(make_session_configs(master))
res = run_trio(lambda rt: party(rt, False), rts)
for name, fn in (("open_results", lambda: open_results(res[:2], schema)),
                 ("_trio.open", lambda: res[0]._trio.open(schema)),
                 ("open_results", lambda: open_results(res[:2], schema))):
    for _ in range(10):
        fn()
    ts = []
    for _ in range(100):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    print("  same result, %s: %.3f ms" % (name, 1e3 * statistics.median(ts)))
for _ in range(30):
    once(prof=True)
for _ in range(30):
    once(prof="open")
for idx, p in profs.items():
    print(f"==== party {idx} (30 queries) ====")
    pstats.Stats(p).sort_stats("tottime").print_stats(18)
