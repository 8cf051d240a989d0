"""C1 trio query (bench.query_latency's trio leg): wall time against the GPU
time of its launches (CUDA events bracketing the whole query; with ncu, the
launch list): python scripts/time_c1_split.py."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_03526_b200 import _lib, workloads  # noqa: E402
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph  # noqa: E402
from paper_2209_03526_b200.query import gen_token, load_query  # noqa: E402
from paper_2209_03526_b200.trio import Trio  # noqa: E402

_lib.check(_lib.load().ogm_init())
graph = workloads.tiny_graph(1)
rng = np.random.default_rng(1)
schema, shares = encrypt_graph(graph, 2, rng)
dshares = device_trio(shares)
query = load_query(workloads.tiny_query(graph, 1), schema)
tokens = gen_token(query, schema, rng)
master = b"\x5a" * 16


def trio():
    res = Trio(master).match(list(tokens), list(dshares))
    return set(res.open(schema)[0])


for _ in range(5):
    trio()
walls = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    trio()
    walls.append(1e3 * (time.perf_counter() - t0))
print(f"wall median {statistics.median(walls):.3f} ms (min {min(walls):.3f})")
