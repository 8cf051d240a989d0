"""Cooperative one-launch online shuffle vs planned/direct steps at 2^lg (L2 flushed between iterations)."""
import statistics
import sys

sys.path.insert(0, ".")
import torch

from paper_2209_03526_b200 import _lib, workloads
from paper_2209_03526_b200.net import make_session_configs
from paper_2209_03526_b200.shuffle import ShuffleOffline, shuffle_online_fused

_lib.check(_lib.load().ogm_init())
flush = torch.empty((512 << 20,), dtype=torch.uint8, device="cuda")
for lg in map(int, sys.argv[1:]):
    rows = 1 << lg
    cfg = make_session_configs(b"\x77" * 16)
    comps = [workloads.device_random_words(rows * 4, 1, 20 + c).reshape(rows, 4) for c in range(3)]
    e = lambda: torch.empty_like(comps[0])  # noqa: E731
    x1, y1, c1, r3 = e(), e(), e(), e()
    res = {}
    for mode in ("fused", "direct", "planned"):
        off = [ShuffleOffline(p + 1, cfg[p].seed_with_next, cfg[p].seed_with_prev, 0, rows, 128,
                              plan=(mode == "planned")) for p in range(3)]

        def step():
            if mode == "fused":
                shuffle_online_fused(off, comps[0], comps[1], comps[2], x1, y1, c1, r3)
            else:
                off[0].step_x1(comps[0], comps[1], x1)
                off[1].step_y1(comps[2], y1)
                off[1].step_c1(x1, c1)
                off[2].step_r3(y1, c1, r3)
        for _ in range(3):
            step()
        ts = []
        for _ in range(7):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[mode] = statistics.median(ts)
        del off
    print(f"2^{lg}: " + "  ".join(f"{k} {v:.4f} ms ({240 * rows / (v * 1e-3) / 1e9 / 6535:.3f})" for k, v in res.items()))
