"""C5 online shuffle at one size, a few iterations (for ncu launch lists):
python scripts/prof_c5_shuffle.py [log2 rows] [iterations]; OGM_GDST=1 reads
gdst instead of the plans' run tables, OGM_FLAT_ORDER=slot runs the
slot-order hand-over, OGM_FUSED=0/1 forces the chained / one-launch path (A/B)."""

import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench_configs as bc  # noqa: E402
from paper_2209_03526_b200 import _lib, shuffle, workloads  # noqa: E402
from paper_2209_03526_b200.net import make_session_configs  # noqa: E402
from paper_2209_03526_b200.shuffle import (FUSED_MAX_BYTES, ShuffleOffline, shuffle_online_fused,  # noqa: E402
                                           shuffle_online_planned)


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    shuffle.USE_RUN_TABLES = not os.environ.get("OGM_GDST")
    shuffle.FLAT_ORDER = os.environ.get("OGM_FLAT_ORDER", shuffle.FLAT_ORDER)
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    _lib.check(_lib.load().ogm_init())
    rows = 1 << lg
    cfg = make_session_configs(b"\x77" * 16)
    seeds = (cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next)
    comps = [workloads.device_random_words(rows * 4, 1, 20 + c).reshape(rows, 4) for c in range(3)]
    fused = rows * 16 <= FUSED_MAX_BYTES if not os.environ.get("OGM_FUSED") else os.environ["OGM_FUSED"] == "1"
    pairs = [(seeds[0], seeds[2]), (seeds[1], seeds[0]), (seeds[2], seeds[1])]
    pc = {}
    off = [ShuffleOffline(p + 1, *pairs[p], 0, rows, 128, perm_cache=pc, plan=not fused) for p in range(3)]
    if not fused:
        for o in off:
            o.chain_blinds()
    r3 = torch.empty_like(comps[0])
    inter = [torch.empty_like(comps[0]) for _ in range(3)]

    def online():
        if fused:
            shuffle_online_fused(off, comps[0], comps[1], comps[2], inter[0], inter[1], None, r3)
        else:
            shuffle_online_planned(off, comps[0], comps[1], comps[2], r3, inter=inter)

    ms = bc._timed_steps(online, iters, 2, None)
    print(f"2^{lg}: {ms:.4f} ms/step, {rows * 240 / (ms * 1e-3) / 1e9:.0f} GB/s algorithmic", flush=True)


if __name__ == "__main__":
    main()
