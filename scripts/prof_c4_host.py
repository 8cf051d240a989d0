"""Host-side profile of the C4 root slot's online step (secEval x2, combine,
fetch): cProfile over the timed calls, to find the Python/host work that
leaves the GPU idle between launches.  python scripts/prof_c4_host.py [rows]."""
import cProfile
import gc
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_03526_b200 import _lib, fss  # noqa: E402
from paper_2209_03526_b200 import workloads  # noqa: E402
from paper_2209_03526_b200.sharded_trio import ShardedGroup, ShardedTrio  # noqa: E402
from paper_2209_03526_b200.sharding import ShardPlan, ThreadComm  # noqa: E402
from paper_2209_03526_b200.trio import TrioGroup  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
_lib.check(_lib.load().ogm_init())
n = 10_000
plan = ShardPlan(rows, 1)
rng = np.random.default_rng(0)
pz = 1.0 / np.arange(1, n + 1) ** 1.1
pz /= pz.sum()
a2 = rng.choice(n, size=rows, p=pz).astype(np.int32)
a3 = rng.choice(n, size=rows, p=pz).astype(np.int32)
c2 = list(workloads.shared_one_hot(torch.from_numpy(a2).cuda(), n, 0, 40, row0=0))
c3 = list(workloads.shared_one_hot(torch.from_numpy(a3).cuda(), n, 0, 50, row0=0))
ids_dummy = [torch.zeros((rows, 1), dtype=torch.int32, device="cuda") for _ in range(3)]
group = ShardedGroup(None, None, rows, 32, ids_dummy, {"a2": c2, "a3": c3}, {"a2": n, "a3": n}, plan=plan, rank=0)
krng = np.random.default_rng(1)


def split(pairs):
    (k11, k21), (k12, k22), (k13, k23) = pairs
    return [(k11, k12), (k22, k13), (k23, k21)]


kiv = split([fss.ic_gen(100, 4000, n, krng) for _ in range(3)])
keq = split(list(fss.bundle_gen("eq", (7,), n, krng).pairs))
plain = torch.from_numpy(np.stack([np.arange(rows, dtype=np.int32), a2, a3, np.zeros(rows, np.int32)], 1)).cuda()
r1 = workloads.device_random_words(rows * 4, 0, 60).reshape(rows, 4)
r2 = workloads.device_random_words(rows * 4, 0, 61).reshape(rows, 4)
rec = [r1, r2, plain ^ r1 ^ r2]


def step(trio, t):
    t0 = time.perf_counter()
    b_iv = trio.sec_eval(group, kiv, "a2", n, {})
    t1 = time.perf_counter()
    b_eq = trio.sec_eval(group, keq, "a3", n, {})
    t2 = time.perf_counter()
    flags = trio.combine([b_iv, b_eq], "ALL", "or", rows)
    t3 = time.perf_counter()
    recs = trio.fetch_multi(TrioGroup(None, None, rows, 128, rec, {}, {}), flags, [])
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    for k, v in zip(("sec_iv", "sec_eq", "combine", "fetch", "tail_sync"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
        t.setdefault(k, []).append(v * 1e3)
    return recs


gc.disable()
trios = []
for _ in range(16):
    tr = ShardedTrio(b"\x4c" * 16, ThreadComm(1).rank_view(0))
    tr.prepare_fetch(rows)
    trios.append(tr)
torch.cuda.synchronize()
t: dict = {}
for i in range(3):
    step(trios[i], {})
t = {}
for i in range(3, 13):
    step(trios[i], t)
print("host ms per phase (median of 10; enqueue time, the GPU runs behind):")
for k, v in t.items():
    print(f"  {k:10s} {np.median(v):7.3f}")
pr = cProfile.Profile()
pr.enable()
for i in range(13, 16):
    step(trios[i], {})
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
st.sort_stats("cumulative").print_stats(45)
