"""Host-side profile of the C1 tiny query through the trio fast path
(Trio.match + open, as bench.py's query_latency times it): where the
1.4 ms goes between Python preparation, the native executor call (which
synchronises on every open) and the reconstruction.
python scripts/prof_c1_host.py [iters]."""
import cProfile
import pstats
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_03526_b200 import _lib, trio_native, workloads  # noqa: E402
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph  # noqa: E402
from paper_2209_03526_b200.query import gen_token, load_query  # noqa: E402
from paper_2209_03526_b200.trio import Trio  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
_lib.check(_lib.load().ogm_init())
graph = workloads.tiny_graph(1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(graph, 2, rng)
dshares = device_trio(shares)
query = load_query(workloads.tiny_query(graph, 1), schema)
tokens = gen_token(query, schema, rng)
master = b"\x5a" * 16

# time the native call itself by wrapping the ctypes function the executor looks up
lib = _lib.load()
native_fn = lib.ogm_trio_match
spent: list = []


class _Timed:
    def __call__(self, *a):
        t = time.perf_counter()
        r = native_fn(*a)
        spent.append(time.perf_counter() - t)
        return r


class _LibProxy:
    def __getattr__(self, k):
        return _Timed() if k == "ogm_trio_match" else getattr(lib, k)


real_load = _lib.load
trio_native._lib.load = lambda: _LibProxy()
phase = {"match": [], "open": [], "total": []}
for it in range(iters + 20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = Trio(master).match(list(tokens), list(dshares))
    t1 = time.perf_counter()
    got = set(res.open(schema)[0])
    t2 = time.perf_counter()
    if it >= 20:
        phase["match"].append(t1 - t0)
        phase["open"].append(t2 - t1)
        phase["total"].append(t2 - t0)
spent = spent[20:]
print("median ms: total %.3f  match %.3f (native call %.3f, python around it %.3f)  open %.3f" % (
    1e3 * statistics.median(phase["total"]), 1e3 * statistics.median(phase["match"]),
    1e3 * statistics.median(spent), 1e3 * (statistics.median(phase["match"]) - statistics.median(spent)),
    1e3 * statistics.median(phase["open"])))
trio_native._lib.load = real_load
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    res = Trio(master).match(list(tokens), list(dshares))
    set(res.open(schema)[0])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
