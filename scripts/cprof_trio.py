import cProfile, pstats, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2209_03526_b200 import workloads
from paper_2209_03526_b200.graphs import encrypt_graph, device_trio
from paper_2209_03526_b200.query import load_query, gen_token
from paper_2209_03526_b200.trio import Trio
g = workloads.tiny_graph(1); q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng); d = list(device_trio(shares))
tokens = list(gen_token(load_query(q, schema), schema, rng))
for _ in range(3): Trio(b"\x5a" * 16).match(tokens, d)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(10): Trio(b"\x5a" * 16).match(tokens, d)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
