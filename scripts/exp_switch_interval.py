"""Per-party C1 latency vs the interpreter's GIL switch interval (3 party threads)."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2209_03526_b200 import workloads
from paper_2209_03526_b200.engine import EngineConfig, open_results, sec_match
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
from paper_2209_03526_b200.query import gen_token, load_query

g = workloads.tiny_graph(1)
q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng)
d = device_trio(shares)
tokens = gen_token(load_query(q, schema), schema, rng)


def one():
    rts = local_runtimes(make_session_configs(b"\x5a" * 16))
    res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig()), rts)
    return open_results(res[:2], schema)


for iv in (0.005, 0.001, 0.0005, 0.0002, 0.0001, 0.00005):
    sys.setswitchinterval(iv)
    for _ in range(5):
        one()
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        t = time.perf_counter()
        one()
        ts.append(time.perf_counter() - t)
    print(f"switch interval {iv * 1e3:.3f} ms: median {statistics.median(ts) * 1e3:.2f} ms, min {min(ts) * 1e3:.2f}", flush=True)
