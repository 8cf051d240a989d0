"""cProfile of the native trio match + open_results (C1)."""
import cProfile
import pstats
import sys

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
for _ in range(3):
    open_results(Trio(b"\x5a" * 16).match(tokens, d).party_results()[:2], schema)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    open_results(Trio(b"\x5a" * 16).match(tokens, d).party_results()[:2], schema)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats(sys.argv[1] if len(sys.argv) > 1 else "cumulative").print_stats(30)
