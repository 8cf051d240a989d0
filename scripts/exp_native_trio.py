"""Native trio executor vs the Python trio path: C1 latency and equality."""
import statistics
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
a = Trio(b"\x5a" * 16).match(tokens, d, native=False)
b = Trio(b"\x5a" * 16).match(tokens, d, native=True)
print("py", sorted(open_results(a.party_results()[:2], schema)[0]))
print("nat", sorted(open_results(b.party_results()[:2], schema)[0]))
for native in (False, True):
    for _ in range(3):
        Trio(b"\x5a" * 16).match(tokens, d, native=native)
    lat = []
    for _ in range(20):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = Trio(b"\x5a" * 16).match(tokens, d, native=native)
        open_results(r.party_results()[:2], schema)
        lat.append(1e3 * (time.perf_counter() - t))
    print("native" if native else "python", f"{statistics.median(lat):.3f} ms")

# phase breakdown of the native path
import paper_2209_03526_b200.trio_native as tn
orig_fn = None
t_call = []


class Timed:
    def __init__(self, fn):
        self.fn = fn

    def __call__(self, *a):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = self.fn(*a)
        t_call.append(1e3 * (time.perf_counter() - t))
        return r


from paper_2209_03526_b200 import _lib
lib = _lib.load()
real = lib.ogm_trio_match


class Shim:
    def __getattr__(self, n):
        return Timed(real) if n == "ogm_trio_match" else getattr(lib, n)


_lib_load = _lib.load
tn._lib.load = lambda *a, **k: Shim() if True else _lib_load()
tot = []
for _ in range(20):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = Trio(b"\x5a" * 16).match(tokens, d, native=True)
    torch.cuda.synchronize()
    tot.append(1e3 * (time.perf_counter() - t))
print(f"native total {statistics.median(tot):.3f} ms, inside ogm_trio_match {statistics.median(t_call[-20:]):.3f} ms")
