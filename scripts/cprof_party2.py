"""cProfile of ONE party thread (party 2) on the per-party C1 path."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import numpy as np

from paper_2209_03526_b200 import workloads
from paper_2209_03526_b200.engine import EngineConfig, sec_match
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
from paper_2209_03526_b200.query import gen_token, load_query

g = workloads.tiny_graph(1)
q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng)
d = device_trio(shares)
tokens = gen_token(load_query(q, schema), schema, rng)
pr = cProfile.Profile()


def worker(rt, prof):
    if prof and rt.index == 2:
        pr.enable()
    r = sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig())
    if prof and rt.index == 2:
        pr.disable()
    return r


for i in range(25):
    run_trio(lambda rt: worker(rt, i >= 5), local_runtimes(make_session_configs(b"\x5a" * 16)))
pstats.Stats(pr).sort_stats(sys.argv[1] if len(sys.argv) > 1 else "tottime").print_stats(30)
