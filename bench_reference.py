"""The LIVE reference (oblivgm 0.1.0, pure Python) timed on this host, beside
the GPU numbers of bench.py (rank 0, one GPU).

The package is installed from the read-only reference tree into
``baseline/_ref`` (``pip install --no-index --no-deps --target baseline/_ref``,
see DESIGN.md); that directory travels to the GPU box with the repo, so the
reference's own public API runs here on the box's host cores:

* C1 (BASELINE configs[0]): ``run_trio`` + ``sec_match`` (src/net.py:320-351,
  src/engine.py:352-417) on the same graph, query, seeds and session master
  as bench.py's query_latency leg; its matches must equal ours.
* C3 / C4 root secEval (configs[2], [3]): ``engine.sec_eval``
  (src/engine.py:139-165), interval predicate over the uniform attribute
  (C3, n = 182,083) and the Zipf attribute (C4, n = 10^4), three party
  threads, on a bounded sample of the candidates, extrapolated linearly.
* C5 (configs[4]): ``shuffle.sec_shuffle`` (src/shuffle.py:80-144) of
  128-bit rows and ``engine.sec_fetch_multi`` (src/engine.py:220-270) of
  flag + 128-bit id rows at 10% flagged, on bounded table sizes,
  extrapolated linearly to the bench sizes.

Everything here is a reported baseline, not an optimisation target; each
entry states its sample and the host threads the reference used (its three
party threads share the GIL, effectively about one core).
"""

from __future__ import annotations

import statistics
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
REF = ROOT / "baseline" / "_ref"


def _load():
    if not (REF / "oblivgm").is_dir():
        return None
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import oblivgm  # noqa: F401
    return oblivgm


def c1(repeats: int = 5) -> dict:
    from oblivgm.engine import EngineConfig, open_results, sec_match
    from oblivgm.graphs import encrypt_graph, parse_graph_text
    from oblivgm.net import local_runtimes, make_session_configs, run_trio
    from oblivgm.query import gen_token, load_query

    from paper_2209_03526_b200 import workloads

    text = workloads.tiny_graph_text(1)
    graph = parse_graph_text(text)
    rng = np.random.default_rng(1)
    schema, shares = encrypt_graph(graph, 2, rng)
    qtext = workloads.tiny_query(workloads.tiny_graph(1), 1)
    tokens = gen_token(load_query(qtext, schema), schema, rng)
    lat, matches = [], None
    for _ in range(repeats + 1):
        rts = local_runtimes(make_session_configs(b"\x5a" * 16))
        t0 = time.perf_counter()
        res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], shares[rt.index - 1], EngineConfig()), rts)
        matches = set(open_results(res[:2], schema)[0])
        lat.append(1e3 * (time.perf_counter() - t0))
    return {"ms": statistics.median(lat[1:]), "unit": "ms", "matches": sorted(list(m) for m in matches),
            "sample": f"the full C1 query, median of {repeats} runs (run_trio + sec_match + open_results)"}


def _sec_eval_sample(n: int, values: np.ndarray, rows_full: int, lo: int, hi: int, master: bytes, label: str) -> dict:
    """The reference's engine.sec_eval (src/engine.py:139-165) of an interval
    predicate [lo, hi] over one-hot shares of ``values`` (a sample of the
    candidates), three party threads; extrapolated linearly to rows_full."""
    from oblivgm import fss
    from oblivgm.engine import CandidateGroup, sec_eval
    from oblivgm.net import local_runtimes, make_session_configs, run_trio

    rng = np.random.default_rng(7)
    sample = values.size
    w = (n + 31) // 32
    onehot = np.zeros((sample, w), np.uint32)
    onehot[np.arange(sample), values // 32] = (np.uint32(1) << (values % 32).astype(np.uint32))
    s1 = rng.integers(0, 1 << 32, size=onehot.shape, dtype=np.uint32)
    s2 = rng.integers(0, 1 << 32, size=onehot.shape, dtype=np.uint32)
    if n % 32:
        s1[:, -1] &= (1 << (n % 32)) - 1
        s2[:, -1] &= (1 << (n % 32)) - 1
    comps = [s1, s2, onehot ^ s1 ^ s2]
    ids = np.zeros((sample, 1), np.uint32)
    groups = [CandidateGroup(None, None, sample, 32, ids, ids, {"z": (comps[q], comps[(q + 1) % 3])}, {"z": n})
              for q in range(3)]
    pairs = [fss.ic_gen(lo, hi, n, rng) for _ in range(3)]
    (k11, k21), (k12, k22), (k13, k23) = pairs
    keys = [(k11, k12), (k22, k13), (k23, k21)]
    rts = local_runtimes(make_session_configs(master))
    t0 = time.perf_counter()
    run_trio(lambda rt: sec_eval(rt, groups[rt.index - 1], keys[rt.index - 1], "z", n), rts)
    dt = time.perf_counter() - t0
    return {"ms": 1e3 * dt * rows_full / sample, "unit": "ms", "rows": rows_full,
            "sample": f"{sample} of {rows_full} candidates ({label}, n={n}, interval, 3 party threads) in "
                      f"{dt:.2f}s, extrapolated linearly"}


def c4_sec_eval(rows_full: int = 2_000_000, sample: int = 1 << 16) -> dict:
    n = 10_000
    rng = np.random.default_rng(1)
    p = 1.0 / np.arange(1, n + 1) ** 1.1
    vals = rng.choice(n, size=sample, p=p / p.sum())
    return _sec_eval_sample(n, vals, rows_full, 100, 4000, b"\x44" * 16, "Zipf attr")


def c3_sec_eval(rows_full: int = 200_000, sample: int = 8192) -> dict:
    """C3's expensive predicate: the interval over the uniform attribute
    (n = 182,083 values, 5,691 words per one-hot row)."""
    n = 182_083
    vals = np.random.default_rng(2).integers(0, n, size=sample)
    return _sec_eval_sample(n, vals, rows_full, 1000, 1000 + n // 10, b"\x35" * 16, "uniform attr")


def c5(logs: list, sample_log: int = 15) -> dict:
    from oblivgm import rss
    from oblivgm.bits import BitVector
    from oblivgm.engine import CandidateGroup, _OpenLabels, sec_fetch_multi
    from oblivgm.net import local_runtimes, make_session_configs, run_trio
    from oblivgm.shuffle import MatchTable, sec_shuffle

    rows = 1 << sample_log
    rng = np.random.default_rng(5)
    comps = [rng.integers(0, 1 << 32, size=(rows, 4), dtype=np.uint32) for _ in range(3)]
    rts = local_runtimes(make_session_configs(b"\x77" * 16))
    t0 = time.perf_counter()
    run_trio(lambda rt: sec_shuffle(rt, MatchTable(rt.index, 128, comps[rt.index - 1], comps[rt.index % 3])), rts)
    t_sh = time.perf_counter() - t0
    plain = (rng.random(rows) < 0.1).astype(np.uint8)
    fsh = rss.share(BitVector.from_bits(plain), rng)
    groups = [CandidateGroup(None, None, rows, 128, comps[q], comps[(q + 1) % 3], {}, {}) for q in range(3)]
    rts = local_runtimes(make_session_configs(b"\x78" * 16))
    t0 = time.perf_counter()
    run_trio(lambda rt: sec_fetch_multi(rt, groups[rt.index - 1], fsh[rt.index - 1], _OpenLabels(), []), rts)
    t_fe = time.perf_counter() - t0
    out = {"unit": "ms", "sample_rows": rows,
           "sample": f"2^{sample_log} rows x 128 bits: sec_shuffle {t_sh:.2f}s, sec_fetch_multi (p=0.1) "
                     f"{t_fe:.2f}s (3 party threads), extrapolated linearly"}
    for lg in logs:
        out[f"shuffle_2^{lg}_ms"] = 1e3 * t_sh * (1 << lg) / rows
        out[f"fetch_p0.1_2^{lg}_ms"] = 1e3 * t_fe * (1 << lg) / rows
    return out


def live_reference(logs: list) -> dict:
    """Every leg above; {"unavailable": why} when baseline/_ref is absent."""
    try:
        if _load() is None:
            return {"unavailable": "baseline/_ref not installed (see DESIGN.md)"}
    except Exception as exc:  # noqa: BLE001
        return {"unavailable": f"baseline/_ref import failed: {exc!r}"}
    import os
    import platform
    out = {"package": "oblivgm 0.1.0 (pure Python) from baseline/_ref", "host_threads": 3,
           "host_cores": os.cpu_count(), "python": platform.python_version()}
    out["c1"] = c1()
    out["c3_sec_eval_uniform"] = c3_sec_eval()
    out["c4_sec_eval"] = c4_sec_eval()
    out["c5"] = c5(logs)
    return out
