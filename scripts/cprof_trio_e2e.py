"""cProfile of the C1 trio query as bench_configs times it: Trio(master).match + open_results."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2209_03526_b200 import workloads
from paper_2209_03526_b200.engine import open_results
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph
from paper_2209_03526_b200.query import gen_token, load_query
from paper_2209_03526_b200.trio import Trio

g = workloads.tiny_graph(1)
q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng)
d = list(device_trio(shares))
tokens = list(gen_token(load_query(q, schema), schema, rng))


def one():
    res = Trio(b"\x5a" * 16).match(tokens, d)
    return res.open(schema)


for _ in range(5):
    one()
torch.cuda.synchronize()
ts = []
for _ in range(30):
    t0 = time.perf_counter()
    one()
    ts.append(time.perf_counter() - t0)
print("median ms", 1e3 * sorted(ts)[15])
pr = cProfile.Profile()
pr.enable()
for _ in range(30):
    one()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(45)
st.sort_stats("tottime").print_stats(30)
