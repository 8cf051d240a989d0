"""Breakdown of the per-party drop-in C1 query (bench.py query_latency's
per_party leg): runtimes, run_trio + sec_match, open_results."""

import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2209_03526_b200 import workloads  # noqa: E402
from paper_2209_03526_b200.engine import EngineConfig, open_results, sec_match  # noqa: E402
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph  # noqa: E402
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio  # noqa: E402
from paper_2209_03526_b200.query import gen_token, load_query  # noqa: E402


def main():
    graph = workloads.tiny_graph(1)
    rng = np.random.default_rng(1)
    schema, shares = encrypt_graph(graph, 2, rng)
    d = device_trio(shares)
    tokens = gen_token(load_query(workloads.tiny_query(graph, 1), schema), schema, rng)
    cfgs = make_session_configs(b"\x5a" * 16)
    t = {"runtimes": [], "match": [], "open": [], "total": []}
    for it in range(25):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rts = local_runtimes(cfgs)
        t1 = time.perf_counter()
        res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig()), rts)
        t2 = time.perf_counter()
        open_results(res[:2], schema)
        t3 = time.perf_counter()
        if it >= 5:
            for k, v in zip(t, (t1 - t0, t2 - t1, t3 - t2, t3 - t0)):
                t[k].append(1e3 * v)
    print({k: round(statistics.median(v), 3) for k, v in t.items()})
    from paper_2209_03526_b200.trio import Trio
    tr, th = [], []
    for it in range(25):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = Trio(b"\x5a" * 16).match(list(tokens), list(d))
        r.party_results()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        run_trio(lambda rt: None, local_runtimes(cfgs))
        t2 = time.perf_counter()
        if it >= 5:
            tr.append(1e3 * (t1 - t0))
            th.append(1e3 * (t2 - t1))
    print({"trio_match+party_results": round(statistics.median(tr), 3), "run_trio_empty": round(statistics.median(th), 3)})


if __name__ == "__main__":
    main()
