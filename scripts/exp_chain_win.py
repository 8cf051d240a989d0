"""Chained online shuffle: window size of the c1 / R3 plans x dual-or-split last pass (2^lg rows).
usage: python scripts/exp_chain_win.py lg win_mb [win_mb ...] [--all]  (--all: every plan, not just c1/R3)"""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib, workloads
from paper_2209_03526_b200.net import make_session_configs
from paper_2209_03526_b200.shuffle import GatherPlan, ShuffleOffline, shuffle_online_planned

_lib.check(_lib.load().ogm_init())
lg = int(sys.argv[1])
rows = 1 << lg
cfg = make_session_configs(b"\x77" * 16)
comps = [workloads.device_random_words(rows * 4, 1, 20 + c).reshape(rows, 4) for c in range(3)]
off = [ShuffleOffline(p + 1, cfg[p].seed_with_next, cfg[p].seed_with_prev, 0, rows, 128, plan=True) for p in range(3)]
for o in off:
    o.chain_blinds()
e = lambda: torch.empty_like(comps[0])  # noqa: E731
want = shuffle_online_planned(off, comps[0], comps[1], comps[2], e())
inter = [e() for _ in range(3)]
r3 = e()
ALL = "--all" in sys.argv
for wmb in [float(x) for x in sys.argv[2:] if not x.startswith("--")]:
    wb = int(wmb * (1 << 20))
    off[1].plan_c1 = GatherPlan(off[1].pi23, 4, window_bytes=wb)
    off[2].plan_r3 = GatherPlan(off[2].k3, 4, window_bytes=wb)
    if ALL:  # the first two plans too (their windows feed the chained kernels)
        off[0].plan_x1 = GatherPlan(off[0].k1, 4, window_bytes=wb)
        off[1].plan_y1 = GatherPlan(off[1].pi12, 4, window_bytes=wb)
    fn = lambda: shuffle_online_planned(off, comps[0], comps[1], comps[2], r3, inter=inter)  # noqa: E731
    fn()
    ok = torch.equal(r3, want)
    for _ in range(3):
        fn()
    ts = []
    for _ in range(7):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    print(f"2^{lg} window {wmb} MB equal={ok}: {ms:.4f} ms ({240 * rows / (ms * 1e-3) / 1e9 / 6535:.3f})", flush=True)
