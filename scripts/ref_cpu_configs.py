"""Time the REFERENCE (oblivgm 0.1.0, pure Python + numpy, CPU) on the C3 / C4
root-slot secEval and the C5 shuffle, the CPU paths SURVEY 8(d) puts beside
those configs.  Runs only where /root/reference exists (the build container;
the reference cannot travel to the GPU box).  Bounded samples, extrapolated
linearly in the candidate / row count from two sample sizes.  Output:
profiles/r01_reference_cpu_configs.jsonl."""
import json
import os
import platform
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np

from oblivgm import fss
from oblivgm.engine import CandidateGroup, sec_eval
from oblivgm.net import local_runtimes, make_session_configs, run_trio
from oblivgm import rss
from oblivgm.bits import BitVector
from oblivgm.shuffle import MatchTable, sec_shuffle


def words_for(n):
    return (n + 31) // 32


def one_hot_shares(values, n, rng):
    w = words_for(n)
    plain = np.zeros((len(values), w), np.uint32)
    plain[np.arange(len(values)), values // 32] = (1 << (values % 32)).astype(np.uint32)
    s1 = rng.integers(0, 1 << 32, size=plain.shape, dtype=np.uint32)
    s2 = rng.integers(0, 1 << 32, size=plain.shape, dtype=np.uint32)
    if n % 32:
        s1[:, -1] &= (1 << (n % 32)) - 1
        s2[:, -1] &= (1 << (n % 32)) - 1
    return s1, s2, plain ^ s1 ^ s2


def time_sec_eval(count, n, lo, hi, values_fn, reps=2):
    rng = np.random.default_rng(7)
    vals = values_fn(rng, count)
    comps = one_hot_shares(vals, n, rng)
    ids = np.zeros((count, 1), np.uint32)
    groups = [CandidateGroup(None, None, count, 1, ids, ids, {"a": (comps[p], comps[(p + 1) % 3])}, {"a": n})
              for p in range(3)]
    pairs = tuple(fss.ic_gen(lo, hi, n, rng) for _ in range(3))
    (k11, k21), (k12, k22), (k13, k23) = pairs
    keys = [(k11, k12), (k22, k13), (k23, k21)]
    best = None
    for _ in range(reps):
        rts = local_runtimes(make_session_configs(b"\x44" * 16))
        t = time.perf_counter()
        run_trio(lambda rt: sec_eval(rt, groups[rt.index - 1], keys[rt.index - 1], "a", n), rts)
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
    return best


def uniform(n):
    return lambda rng, c: rng.integers(0, n, size=c)


def zipf(n):
    p = 1.0 / np.arange(1, n + 1) ** 1.1
    p /= p.sum()
    return lambda rng, c: rng.choice(n, size=c, p=p)


def emit(d):
    d.update({"impl": "reference (oblivgm 0.1.0, pure Python + numpy)", "host": platform.processor() or
              platform.machine(), "cpus": os.cpu_count(),
              "where": "build container (no GPU); the reference cannot run on the GPU box"})
    print(json.dumps(d), flush=True)


for name, full, n, lo, hi, dist, samples in (
        ("C3 root secEval, uniform attr (n=182083, w=5691), interval", 200_000, 182_083, 1000, 20_000,
         uniform(1 << 20), (1000, 4000)),
        ("C3 root secEval, Zipf attr (n=8969, w=281), interval", 200_000, 8_969, 100, 4000, zipf(8_969),
         (10_000, 40_000)),
        ("C4 root secEval, Zipf attr (n=10000, w=313), interval", 2_000_000, 10_000, 100, 4000, zipf(10_000),
         (20_000, 80_000))):
    t = [time_sec_eval(c, n, lo, hi, (lambda d: (lambda rng, c: d(rng, c) % n))(dist)) for c in samples]
    slope = (t[1] - t[0]) / (samples[1] - samples[0])
    est = t[0] + slope * (full - samples[0])
    emit({"config": name, "metric": "secEval_protocol_ms", "candidates": full, "value": 1e3 * est,
          "unit": "ms", "extrapolated_from": {str(c): round(1e3 * x, 1) for c, x in zip(samples, t)},
          "path": "run_trio + sec_eval (3 party threads), FDE + masked parity + re-share, one interval predicate"})

for lg in (12, 14, 16):
    rows, width = 1 << lg, 128
    rng = np.random.default_rng(lg)
    plain = rng.integers(0, 1 << 32, size=(rows, 4), dtype=np.uint32)
    s1 = rng.integers(0, 1 << 32, size=(rows, 4), dtype=np.uint32)
    s2 = rng.integers(0, 1 << 32, size=(rows, 4), dtype=np.uint32)
    comps = (s1, s2, plain ^ s1 ^ s2)
    tables = [MatchTable(p + 1, width, comps[p], comps[(p + 1) % 3]) for p in range(3)]
    rts = local_runtimes(make_session_configs(b"\x77" * 16))
    t = time.perf_counter()
    run_trio(lambda rt: sec_shuffle(rt, tables[rt.index - 1]), rts)
    dt = time.perf_counter() - t
    emit({"config": f"C5 shuffle 2^{lg} rows x 128-bit", "metric": "shuffle_ms", "value": 1e3 * dt, "unit": "ms",
          "rows_per_s": rows / dt, "algorithmic_GBps": rows * 240 / dt / 1e9,
          "path": "run_trio + sec_shuffle (3 party threads), permutations + blinds generated inline"})
