"""Time the REFERENCE (oblivgm, pure Python, CPU) on exactly the C1 workload the
bench uses (same graph text, query, seeds, session master).  Runs only where
/root/reference exists (the build container); results go to profiles/."""
import json, statistics, sys, time
sys.path.insert(0, ".")
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
from paper_2209_03526_b200 import workloads
from oblivgm.datagen import graph_to_text
from oblivgm.graphs import encrypt_graph, parse_graph_text
from oblivgm.query import gen_token, load_query
from oblivgm.net import local_runtimes, make_session_configs, run_trio
from oblivgm.engine import sec_match, EngineConfig, open_results
from oblivgm.oracle import oracle_match
import os, platform

g_mine = workloads.tiny_graph(1)
qtext = workloads.tiny_query(g_mine, 1)
text = "\n".join(f"V {v.vtype} {v.ext_id} " + " ".join(f"{k}={x}" for k, x in v.attrs.items()) for v in g_mine.vertices)
edges = sorted(g_mine._edges)
text += "\n" + "\n".join(f"E {g_mine.vertices[a].ext_id} {g_mine.vertices[b].ext_id}" for a, b in edges)
graph = parse_graph_text(text)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(graph, 2, rng)
query = load_query(qtext, schema)
tokens = gen_token(query, schema, rng)
want = oracle_match(graph, query, schema)
lat = []
for it in range(13):
    rts = local_runtimes(make_session_configs(b"\x5a" * 16))
    t0 = time.perf_counter()
    res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], shares[rt.index - 1], EngineConfig()), rts)
    m, _ = open_results(res[:2], schema)
    if it >= 3:
        lat.append(time.perf_counter() - t0)
assert set(m) == want
print(json.dumps({"config": "C1 tiny (same graph/query/seeds as bench_configs.py c1)", "impl": "reference (oblivgm 0.1.0, pure Python)",
                  "metric": "query_latency_ms", "value": 1e3 * statistics.median(lat), "unit": "ms",
                  "min_ms": 1e3 * min(lat), "matches": len(m), "host": platform.processor() or platform.machine(),
                  "cpus": os.cpu_count(), "where": "build container (no GPU); the reference cannot run on the GPU box"}))
