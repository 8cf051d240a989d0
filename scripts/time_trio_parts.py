"""Wall-time split of one C1 trio query: Trio(), plan building, ogm_trio_match, result views, open."""
import statistics
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2209_03526_b200 import _lib, trio_native, workloads
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph
from paper_2209_03526_b200.query import gen_token, load_query
from paper_2209_03526_b200.trio import Trio

g = workloads.tiny_graph(1)
q = workloads.tiny_query(g, 1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(g, 2, rng)
d = list(device_trio(shares))
tokens = list(gen_token(load_query(q, schema), schema, rng))
lib = _lib.load()
orig = lib.ogm_trio_match
acc = {"call": []}


def timed_call(*a):
    t = time.perf_counter()
    r = orig(*a)
    acc["call"].append(time.perf_counter() - t)
    return r


class Wrap:
    def __getattr__(self, k):
        return timed_call if k == "ogm_trio_match" else getattr(lib, k)


trio_native._lib = type("L", (), {})()
for k in dir(_lib):
    if not k.startswith("__"):
        setattr(trio_native._lib, k, getattr(_lib, k))
trio_native._lib.load = lambda: Wrap()
parts = {"Trio()": [], "match_native": [], "open": [], "total": []}
for it in range(60):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tr = Trio(b"\x5a" * 16)
    t1 = time.perf_counter()
    res = tr.match(tokens, d)
    t2 = time.perf_counter()
    res.open(schema)
    t3 = time.perf_counter()
    if it >= 10:
        parts["Trio()"].append(t1 - t0)
        parts["match_native"].append(t2 - t1)
        parts["open"].append(t3 - t2)
        parts["total"].append(t3 - t0)
for k, v in parts.items():
    print(f"{k:14s} {1e3 * statistics.median(v):.3f} ms")
print(f"{'  ogm_trio_match':14s} {1e3 * statistics.median(acc['call'][10:]):.3f} ms")
