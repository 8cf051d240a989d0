"""ncu target: exactly one trio C1 match after warm-up (for the per-kernel GPU time sum)."""
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
torch.cuda.cudart().cudaProfilerStart()
Trio(b"\x5a" * 16).match(tokens, d)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
