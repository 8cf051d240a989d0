"""Does returning freed device memory to the driver (torch.cuda.empty_cache)
right before the C4 secEval leg slow its first steps?  Frees ~9 GB (the C2
keys' size) with or without empty_cache, allocates the C4 tables and times
the folded secEval step by step (CUDA events per step).
python scripts/diag_c4_alloc.py [empty|keep] [reps]."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2209_03526_b200 import _lib, fss, workloads  # noqa: E402
from paper_2209_03526_b200.bits import words_for  # noqa: E402
from paper_2209_03526_b200.net import make_session_configs  # noqa: E402
from paper_2209_03526_b200.sharding import ShardPlan, fold_indicators, sharded_sec_eval_trio  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "empty"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
_lib.check(_lib.load().ogm_init())
rows, n = 2_000_000, 10_000
w = words_for(n)
plan = ShardPlan(rows, 1)
rng = np.random.default_rng(1)
p = 1.0 / np.arange(1, n + 1) ** 1.1
vals = torch.from_numpy(rng.choice(n, size=rows, p=p / p.sum()).astype(np.int32)).cuda()
krng = np.random.default_rng(2)
(k11, k21), (k12, k22), (k13, k23) = [fss.ic_gen(100, 4000, n, krng) for _ in range(3)]
keys = [(k11, k12), (k22, k13), (k23, k21)]
inds = [[(fss.full_domain(fss.KeyBatch.from_keys([fss.key_parts_for_engine(keys[q][0])[ps]]), n)[0],
          fss.full_domain(fss.KeyBatch.from_keys([fss.key_parts_for_engine(keys[q][1])[ps]]), n)[0])
         for q in range(3)] for ps in range(2)]
folded = fold_indicators(inds)
zk = [(c.zero_key_own, c.zero_key_prev) for c in make_session_configs(b"\x44" * 16)]
for rep in range(reps):
    big = torch.empty((9 << 30,), dtype=torch.uint8, device="cuda")
    big.fill_(1)
    torch.cuda.synchronize()
    del big
    if mode == "empty":
        torch.cuda.empty_cache()
    comps = list(workloads.shared_one_hot(vals, n, 1, 40, row0=0))
    step = lambda: sharded_sec_eval_trio(comps, w, plan, 0, folded, zk, [0, 1], fold=True)  # noqa: E731
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
    ev[0].record()
    for i in range(10):
        step()
        ev[i + 1].record()
    torch.cuda.synchronize()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(10)]
    print(f"{mode} rep {rep}: total {ev[0].elapsed_time(ev[10]) / 10:.3f} ms/step; per step "
          + " ".join(f"{x:.2f}" for x in per) + f"; median {statistics.median(per):.3f}", flush=True)
    del comps, step
    if mode == "empty":
        torch.cuda.empty_cache()
