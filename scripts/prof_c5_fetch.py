"""C5 fetch at one size: per-launch device times of the online phase (for
ncu launch lists) -- python scripts/prof_c5_fetch.py [log2 rows] [p ...];
OGM_FLAG_TAIL=0/1 forces the flag column's layout (A/B)."""

import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench_configs as bc  # noqa: E402
from paper_2209_03526_b200 import _lib  # noqa: E402
from paper_2209_03526_b200.fetch import FlaggedFetch  # noqa: E402
from paper_2209_03526_b200.net import make_session_configs  # noqa: E402
from paper_2209_03526_b200 import workloads  # noqa: E402


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    ps = [float(x) for x in sys.argv[2:]] or [0.01, 1.0]
    _lib.check(_lib.load().ogm_init())
    rows = 1 << lg
    cfg = make_session_configs(b"\x78" * 16)
    seeds = (cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next)
    payload = [workloads.device_random_words(rows * 4, 1, 30 + c).reshape(rows, 4) for c in range(3)]
    f12 = [bc._random_bits(rows, 1, 40), bc._random_bits(rows, 1, 41)]
    tail = os.environ.get("OGM_FLAG_TAIL")
    ff = FlaggedFetch(seeds, 0, rows, flag_tail=None if tail is None else tail == "1")
    for p in ps:
        fp = bc._bernoulli_bits(rows, p, 7)
        flags = [f12[0], f12[1], fp ^ f12[0] ^ f12[1]]
        ms = bc._timed_steps(lambda: ff.online(flags, payload), 5, 3, None)
        print(f"2^{lg} p={p}: {ms:.3f} ms, kept {ff.kept()}", flush=True)


if __name__ == "__main__":
    main()
