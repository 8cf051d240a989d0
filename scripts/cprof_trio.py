"""cProfile of the trio C1 match (single host thread): where the host time goes."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2209_03526_b200 import workloads
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
    Trio(b"\x5a" * 16).match(tokens, d)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    Trio(b"\x5a" * 16).match(tokens, d)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats(sys.argv[1] if len(sys.argv) > 1 else "tottime").print_stats(int(sys.argv[2]) if len(sys.argv) > 2 else 25)
