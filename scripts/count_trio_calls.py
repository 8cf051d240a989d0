"""Count C-ABI calls and tensor allocations per trio C1 match."""
import collections
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2209_03526_b200._lib as L
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
Trio(b"\x5a" * 16).match(tokens, d)
calls = collections.Counter()
orig = L.call


def counting(name, *a):
    calls[name] += 1
    return orig(name, *a)


L.call = counting
Trio(b"\x5a" * 16).match(tokens, d)
torch.cuda.synchronize()
print(sum(calls.values()), "calls")
for k, v in calls.most_common():
    print(f"  {k:32s} {v}")
