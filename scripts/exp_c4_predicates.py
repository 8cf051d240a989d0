import sys, time, torch, numpy as np
sys.path.insert(0, ".")
import bench_configs as bc
from paper_2209_03526_b200 import _lib, fss, workloads
from paper_2209_03526_b200.sharded_trio import ShardedGroup, ShardedTrio
from paper_2209_03526_b200.sharding import ShardPlan, ThreadComm
_lib.check(_lib.load().ogm_init())
rows, n, seed = 2_000_000, 10_000, 1
plan = ShardPlan(rows, 1)
rng = np.random.default_rng(seed)
pz = 1.0 / np.arange(1, n + 1) ** 1.1; pz /= pz.sum()
a2 = rng.choice(n, size=rows, p=pz).astype(np.int32); a3 = rng.choice(n, size=rows, p=pz).astype(np.int32)
c2 = list(workloads.shared_one_hot(torch.from_numpy(a2).cuda(), n, seed, 40))
c3 = list(workloads.shared_one_hot(torch.from_numpy(a3).cuda(), n, seed, 50))
ids = [torch.zeros((rows, 1), dtype=torch.int32, device="cuda") for _ in range(3)]
g = ShardedGroup(None, None, rows, 32, ids, {"a2": c2, "a3": c3}, {"a2": n, "a3": n}, plan=plan, rank=0)
krng = np.random.default_rng(2)
def split(pairs):
    (k11, k21), (k12, k22), (k13, k23) = pairs
    return [(k11, k12), (k22, k13), (k23, k21)]
kiv = split([fss.ic_gen(100, 4000, n, krng) for _ in range(3)])
keq = split(list(fss.bundle_gen("eq", (7,), n, krng).pairs))
for name, keys, attr in (("iv", kiv, "a2"), ("eq", keq, "a3")):
    ts = []
    for it in range(8):
        tr = ShardedTrio(b"\x4c" * 16, ThreadComm(1).rank_view(0))
        cache = {}
        tr._pass_indicators(keys, n, cache)   # FDE outside the timing
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize(); e[0].record()
        tr.sec_eval(g, keys, attr, n, cache)
        e[1].record(); torch.cuda.synchronize()
        ts.append(e[0].elapsed_time(e[1]))
    print(name, sorted(ts)[len(ts)//2])
