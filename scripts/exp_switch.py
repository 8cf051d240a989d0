"""Per-party C1 latency vs the interpreter's GIL switch interval."""
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


for si in (5e-3, 1e-3, 2e-4, 5e-5, 1e-5):
    sys.setswitchinterval(si)
    for _ in range(3):
        one()
    lat = []
    for _ in range(20):
        torch.cuda.synchronize()
        t = time.perf_counter()
        one()
        lat.append(1e3 * (time.perf_counter() - t))
    print(f"switch interval {si * 1e3:.3f} ms: per-party C1 {statistics.median(lat):.2f} ms (min {min(lat):.2f})")
