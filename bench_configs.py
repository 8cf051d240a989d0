#!/usr/bin/env python
"""Secondary benchmarks for BASELINE configs 1, 3 and 5 (bench.py covers config 2).

    python bench_configs.py c1 [--steps K]      tiny end-to-end query latency
    python bench_configs.py c3 [--rows X]       root-slot secEval (HBM-bound)
    python bench_configs.py c5 [--max-log 28]   shuffle / fetch bandwidth sweep

Each prints one JSON line per measurement.  Device times use CUDA events on
the launching stream(s) after warm-up; wall-clock is used only for the
three-thread end-to-end protocol runs, as the reference does
(src/bench.py:47-49).
"""

from __future__ import annotations

import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2209_03526_b200 import _lib, fss  # noqa: E402
from paper_2209_03526_b200.bits import words_for  # noqa: E402
from paper_2209_03526_b200.engine import CandidateGroup, EngineConfig, open_results, sec_eval, sec_match  # noqa: E402
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph  # noqa: E402
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio  # noqa: E402
from paper_2209_03526_b200.query import gen_token, load_query  # noqa: E402
from paper_2209_03526_b200.shuffle import (FUSED_MAX_BYTES, ShuffleOffline, blind_table, gather,  # noqa: E402
                                            shuffle_online_fused, shuffle_online_planned)
from paper_2209_03526_b200.prf import seeded_permutation_device  # noqa: E402
from paper_2209_03526_b200 import workloads  # noqa: E402
from paper_2209_03526_b200.trio import TrioGroup  # noqa: E402

def _hbm_peak() -> float:
    """GB/s: MEASURED_PEAKS.json (driver-written copy benchmark) when present,
    else its last recorded value for this pool."""
    try:
        return float(json.load(open(Path(__file__).resolve().parent / "MEASURED_PEAKS.json"))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6535.4


HBM_PEAK = _hbm_peak()


def emit(d):
    print(json.dumps(d), flush=True)


def events(n):
    return [torch.cuda.Event(enable_timing=True) for _ in range(n)]


# ---------------------------------------------------------------------------
# C1: tiny end-to-end
# ---------------------------------------------------------------------------


def cpu_port_sec_eval(comps, words: int, ind_of, gpu_bits_of, sample: int, folded: bool = False) -> dict:
    """The CPU path beside a secEval line: the oracle port's masked parity
    (oracle/, C, one core; src/engine.py:76-80) for all 3 parties x 2 passes
    on the first `sample` candidate rows, timed and extrapolated linearly to
    the full row count.  Its bits are checked against the GPU result (per
    pass, or -- ``folded`` -- the XOR of the two passes against
    gpu_bits_of(p, None))."""
    import oracle

    rows = comps[0].shape[0]
    sample = min(sample, rows)
    host = [c[:sample, :words].cpu().numpy().view(np.uint32) for c in comps]
    dt, same = 0.0, True
    acc = {}
    for ps in range(2):
        for p in range(3):
            ia = ind_of(p, ps)[0].cpu().numpy().view(np.uint32)[:words]
            ib = ind_of(p, ps)[1].cpu().numpy().view(np.uint32)[:words]
            t = time.perf_counter()
            bits = oracle.masked_parity(host[p], host[(p + 1) % 3], ia, ib)
            dt += time.perf_counter() - t
            if folded:
                acc[p] = bits if ps == 0 else acc[p] ^ bits
                if ps == 1:
                    got = oracle.unpack_bits(gpu_bits_of(p, None), rows)[:sample]
                    same = same and bool(np.array_equal(acc[p], got))
                continue
            got = oracle.unpack_bits(gpu_bits_of(p, ps), rows)[:sample]
            same = same and bool(np.array_equal(bits, got))
    return {"value": 1e3 * dt * rows / sample, "unit": "ms", "cores": 1, "kind": "port",
            "sample": f"{sample} of {rows} candidates, 3 parties x 2 passes, oracle.masked_parity "
                      f"(C, src/engine.py:76-80) in {dt:.2f}s, extrapolated linearly",
            "gpu_bits_equal_on_sample": same}


def run_c1(args):
    import oracle.matcher as om

    graph = workloads.tiny_graph(args.seed)
    qtext = workloads.tiny_query(graph, args.seed)
    rng = np.random.default_rng(args.seed)
    t0 = time.perf_counter()
    schema, shares = encrypt_graph(graph, 2, rng)
    t_enc = time.perf_counter() - t0
    dshares = device_trio(shares)
    query = load_query(qtext, schema)
    t0 = time.perf_counter()
    tokens = gen_token(query, schema, rng)
    t_tok = time.perf_counter() - t0
    want = om.oracle_match(graph, query, schema)
    master = b"\x5a" * 16

    def one():
        rts = local_runtimes(make_session_configs(master))
        res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], dshares[rt.index - 1], EngineConfig()), rts)
        matches, _ = open_results(res[:2], schema)
        return set(matches), rts

    for _ in range(args.warmup):
        got, _ = one()
    if got != want:
        raise SystemExit(f"C1 result differs from the plaintext oracle: {got} vs {want}")
    lat = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got, rts = one()
        lat.append(time.perf_counter() - t0)
    phases = {ph: st.bytes_sent for ph, st in rts[0].meter.phases.items()}

    from paper_2209_03526_b200.trio import Trio

    def one_trio():
        res = Trio(master).match(list(tokens), list(dshares))
        matches, _ = res.open(schema)   # == open_results(res.party_results()[:2], schema), tested
        return set(matches)

    for _ in range(args.warmup):
        got_t = one_trio()
    lat_t = []
    for _ in range(args.steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got_t = one_trio()
        lat_t.append(time.perf_counter() - t0)
    emit({"config": "C1 tiny (1000 vertices, 3 types, 3-vertex path, k=2)", "metric": "query_latency_ms",
          "value": 1e3 * statistics.median(lat_t), "unit": "ms", "higher_is_better": False,
          "min_ms": 1e3 * min(lat_t), "max_ms": 1e3 * max(lat_t), "steps": args.steps, "matches": len(got_t),
          "oracle_equal": got_t == want,
          "path": "trio fast path: 3 co-resident servers in one thread, one launch per step for all parties"})
    emit({"config": "C1 tiny (1000 vertices, 3 types, 3-vertex path, k=2)", "metric": "query_latency_ms",
          "value": 1e3 * statistics.median(lat), "unit": "ms", "higher_is_better": False,
          "min_ms": 1e3 * min(lat), "max_ms": 1e3 * max(lat), "steps": args.steps, "matches": len(got),
          "oracle_equal": got == want, "bytes_per_party_by_phase": phases,
          "offline": {"encrypt_graph_s": t_enc, "gen_token_s": t_tok},
          "path": "per-party drop-in API: 3 party threads, device messages, run_trio + sec_match + open_results"})


# ---------------------------------------------------------------------------
# C3: root-slot secEval on the medium graph shapes
# ---------------------------------------------------------------------------


def run_c3(args):
    X = args.rows
    dev = torch.device("cuda")
    rng = np.random.default_rng(args.seed)
    for name, n in (("uniform", 182083), ("zipf", 8969)):
        vals = torch.from_numpy(rng.integers(0, n, size=X).astype(np.int32)).to(dev)
        c1, c2, c3 = workloads.shared_one_hot(vals, n, args.seed, 10)
        comps = [c1, c2, c3]
        w = words_for(n)
        lo = int(rng.integers(0, n // 2))
        pairs = [fss.ic_gen(lo, lo + n // 10, n, rng) for _ in range(3)]
        (k11, k21), (k12, k22), (k13, k23) = pairs
        keys = [(k11, k12), (k22, k13), (k23, k21)]
        # full-domain indicators once (cached per key in sec_match)
        inds = []
        for p in range(3):
            row = []
            for pi in range(2):
                ka = fss.key_parts_for_engine(keys[p][0])[pi]
                kb = fss.key_parts_for_engine(keys[p][1])[pi]
                row.append((fss.full_domain(fss.KeyBatch.from_keys([ka]), n)[0],
                            fss.full_domain(fss.KeyBatch.from_keys([kb]), n)[0]))
            inds.append(row)
        outs = [torch.empty(words_for(X), dtype=torch.int32, device=dev) for _ in range(6)]
        A = _lib.ptr_array

        def per_party(p):
            ind = [inds[p][0][0], inds[p][0][1], inds[p][1][0], inds[p][1][1]]
            _lib.call("ogm_masked_parity", X, w, comps[0].stride(0), 2, A([comps[p], comps[(p + 1) % 3]]), 1, _lib.int_array([0]),
                      _lib.int_array([1]), 2, A(ind), A(outs[2 * p:2 * p + 2]), _lib.stream_ptr())

        def trio():
            ind = []
            for pi in range(2):
                for p in range(3):
                    ind += [inds[p][pi][0], inds[p][pi][1]]
            _lib.call("ogm_masked_parity", X, w, comps[0].stride(0), 3, A(comps), 3, _lib.int_array([0, 1, 2]),
                      _lib.int_array([1, 2, 0]), 2, A(ind), A(outs), _lib.stream_ptr())

        # parity check: trio == per-party results
        for p in range(3):
            per_party(p)
        ref = [o.clone() for o in outs]
        trio()
        ok = all(torch.equal(ref[2 * p + pi], outs[pi * 3 + p]) for p in range(3) for pi in range(2))
        cpu = cpu_port_sec_eval(comps, w, lambda p, ps: inds[p][ps],
                                lambda p, ps: ref[2 * p + ps].cpu().numpy().view(np.uint32),
                                2000 if w > 1000 else 20000)
        for mode, fn, nbytes in (("per-party (3 launches)", lambda: [per_party(p) for p in range(3)], 3 * 2 * X * w * 4),
                                 ("trio-fused", trio, 3 * X * w * 4)):
            for _ in range(args.warmup):
                fn()
            ev = events(args.steps + 1)
            ev[0].record()
            for s in range(args.steps):
                fn()
                ev[s + 1].record()
            torch.cuda.synchronize()
            ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps))
            emit({"config": f"C3 root secEval, {X} candidates, {name} attr n={n} (w={w} words), interval "
                            "(2 passes fused)", "metric": "secEval_local_GBps", "mode": mode,
                  "value": nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms": ms,
                  "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / HBM_PEAK, "algorithmic_bytes": nbytes,
                  "trio_equals_per_party": ok, "cpu_baseline": cpu})
        # the full protocol step (3 threads, fused passes + 2 reshares per party)
        group = [CandidateGroup(None, None, X, X, comps[p][:, :1], comps[(p + 1) % 3][:, :1],
                                {"a": (comps[p], comps[(p + 1) % 3])}, {"a": n}) for p in range(3)]
        caches = [dict() for _ in range(3)]
        lat = []
        for it in range(args.warmup + args.steps):
            rts = local_runtimes(make_session_configs(b"\x33" * 16))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run_trio(lambda rt: sec_eval(rt, group[rt.index - 1], keys[rt.index - 1], "a", n,
                                         caches[rt.index - 1]), rts)
            if it >= args.warmup:
                lat.append(time.perf_counter() - t0)
        emit({"config": f"C3 root secEval {name}", "metric": "secEval_protocol_ms", "value": 1e3 * statistics.median(lat),
              "unit": "ms", "path": "per-party drop-in sec_eval x3 threads (indicators cached)"})
        del c1, c2, c3, comps, group
        torch.cuda.empty_cache()


# ---------------------------------------------------------------------------
# Per-function throughput beside the CPU port
# ---------------------------------------------------------------------------


def run_funcs(args):
    """One line per primitive of the path at a GPU-filling size, device-timed,
    with the oracle port timed on the host (one core) on a bounded sample;
    results of the two are compared on the sample where that is cheap."""
    import oracle

    dev = torch.device("cuda")
    gen = torch.Generator(device="cuda").manual_seed(args.seed)

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        ev = events(reps + 1)
        ev[0].record()
        for i in range(reps):
            fn()
            ev[i + 1].record()
        torch.cuda.synchronize()
        return statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(reps)) * 1e-3

    def cpu(fn):
        t = time.perf_counter()
        r = fn()
        return time.perf_counter() - t, r

    def line(row, ref, name, unit, gpu_rate, n_gpu, cpu_rate, n_cpu, equal, survey):
        emit({"row": row, "reference": ref, "function": name, "unit": unit, "value": gpu_rate,
              "gpu_sample": n_gpu, "cpu_baseline": {"value": cpu_rate, "unit": unit, "cores": 1, "kind": "port",
                                                      "sample": n_cpu},
              "gpu_equals_port_on_sample": equal, "survey_time_today_1core": survey})

    # a1 prg_expand (src/prf.py:41-57): 3 AES per seed
    n = 1 << 24
    seeds = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device=dev, generator=gen)
    from paper_2209_03526_b200 import prf
    t = timed(lambda: prf.prg_expand(seeds))
    sm = seeds[: 1 << 16].cpu().numpy().view(np.uint64).reshape(-1, 2)
    tc, ref = cpu(lambda: oracle.prg_expand(sm))
    got = prf.prg_expand(seeds[: 1 << 16])
    eq = bool(np.array_equal(got[0].cpu().numpy().view(np.uint64).reshape(-1, 2), ref[0]))
    line("a1", "src/prf.py:41-57", "prg_expand", "seeds/s", n / t, n, (1 << 16) / tc, 1 << 16, eq,
         "8-15 M nodes/s batched")
    del seeds
    # a2 prf_stream (src/prf.py:70-92): AES-CTR
    nw = 1 << 28
    out = torch.empty((nw,), dtype=torch.int32, device=dev)
    key = bytes(range(16))
    t = timed(lambda: prf.prf_words_device(key, b"SHTB", 7, nw, out=out))
    tc, ref = cpu(lambda: oracle.prf_stream(key, b"SHTB", 7, 1 << 24))
    eq = out[: 1 << 22].cpu().numpy().tobytes() == ref
    line("a2", "src/prf.py:70-92", "prf_stream (AES-128-CTR)", "GB/s", 4 * nw / t / 1e9, 4 * nw,
         (1 << 24) / tc / 1e9, 1 << 24, eq, "0.33 GB/s")
    del out
    # a3 seeded_permutation (src/prf.py:95-105): Fisher-Yates
    n = 1 << 24
    t = timed(lambda: prf.seeded_permutation_device(key, b"SHPI", 3, n), reps=3)
    tc, ref = cpu(lambda: oracle.seeded_permutation(key, b"SHPI", 3, 1 << 20))
    eq = bool(np.array_equal(prf.seeded_permutation_device(key, b"SHPI", 3, 1 << 20).cpu().numpy(), ref))
    line("a3", "src/prf.py:95-105", "seeded_permutation", "swaps/s", (n - 1) / t, n, ((1 << 20) - 1) / tc, 1 << 20,
         eq, "0.85 M swaps/s")
    # a6 keygen (src/fss.py:116-157): DCF, 32-bit domain
    k = 1 << 22
    alphas = torch.randint(-(1 << 31), 1 << 31, (k,), dtype=torch.int32, device=dev, generator=gen)
    r0 = torch.randint(0, 256, (k, 16), dtype=torch.uint8, device=dev, generator=gen)
    r1 = torch.randint(0, 256, (k, 16), dtype=torch.uint8, device=dev, generator=gen)
    t = timed(lambda: fss.gen_batch(True, 32, alphas, r0, r1), reps=3)
    ks = 4096
    a_h = alphas[:ks].cpu().numpy().view(np.uint32).astype(np.uint64)
    tc, (o0, _) = cpu(lambda: oracle.tree_gen_batch(a_h, 32, r0[:ks].cpu().numpy(), r1[:ks].cpu().numpy(), True,
                                                     nthreads=1))
    b0, _ = fss.gen_batch(True, 32, alphas[:ks], r0[:ks], r1[:ks])
    eq = bool(np.array_equal(b0.seed_cw.cpu().numpy().transpose(1, 0, 2), o0.seed_cw))
    line("a6", "src/fss.py:116-157", "dcf keygen (_tree_gen, 32-bit)", "key pairs/s", k / t, k, ks / tc, ks, eq,
         "1.39 ms/pair")
    del alphas, r0, r1
    # a8 full-domain eval (src/fss.py:302-337): 16 keys x 2^20 leaves
    nk, dom = 16, 1 << 20
    al = torch.randint(0, dom, (nk,), dtype=torch.int32, device=dev, generator=gen)
    rr = torch.randint(0, 256, (nk, 16), dtype=torch.uint8, device=dev, generator=gen)
    kb, _ = fss.gen_batch(True, 20, al, rr, rr)
    fd = fss.full_domain(kb, dom)
    t = timed(lambda: fss.full_domain(kb, dom, out=fd))
    ok0, _ = oracle.tree_gen_batch(al[:1].cpu().numpy().view(np.uint32).astype(np.uint64), 20, rr[:1].cpu().numpy(),
                                   rr[:1].cpu().numpy(), True)
    tc, ref = cpu(lambda: oracle.full_domain(ok0, 0, dom))
    eq = bool(np.array_equal(fd[0].cpu().numpy().view(np.uint32), ref))
    line("a8", "src/fss.py:302-337", "full-domain eval (DCF, 2^20 leaves)", "leaves/s", nk * dom / t, nk * dom,
         dom / tc, dom, eq, "~9.5 M leaves/s")
    # a10 zero shares, three parties per launch (src/rss.py:143-148)
    nbits = 1 << 32
    outs = [torch.empty((nbits // 32,), dtype=torch.int32, device=dev) for _ in range(3)]
    cfgs = make_session_configs(b"\x12" * 16)
    zk = [c.zero_key_own for c in cfgs]
    A = _lib.ptr_array
    t = timed(lambda: _lib.call("ogm_zero_share_trio", zk[0], zk[1], zk[2], 9, nbits, None, A(outs),
                                _lib.stream_ptr()))
    tc, ref = cpu(lambda: oracle.zero_share(zk[0], zk[2], 9, 1 << 24))
    eq = bool(np.array_equal(outs[0][: (1 << 24) // 32].cpu().numpy().view(np.uint32), ref))
    line("a10", "src/rss.py:143-148", "zero shares, 3 parties per launch", "GB/s of shares",
         3 * nbits / 8 / t / 1e9, 3 * nbits, (1 << 24) / 8 / tc / 1e9, 1 << 24, eq, "AES-CTR 0.33 GB/s")
    del outs
    # a11 and_terms (src/rss.py:115-126), three parties per launch: z_q = a_q b_q ^ a_q b_q+1 ^ a_q+1 b_q
    nw = 1 << 26
    va = [torch.randint(-2**31, 2**31 - 1, (nw,), dtype=torch.int32, device=dev, generator=gen) for _ in range(3)]
    vb = [torch.randint(-2**31, 2**31 - 1, (nw,), dtype=torch.int32, device=dev, generator=gen) for _ in range(3)]
    zo = [torch.empty_like(va[0]) for _ in range(3)]
    nx = [1, 2, 0]
    args = (A([va[q] for q in range(3)]), A([va[nx[q]] for q in range(3)]), A([vb[q] for q in range(3)]),
            A([vb[nx[q]] for q in range(3)]), A(zo))
    t = timed(lambda: _lib.call("ogm_and_terms", nw, 3, *args, _lib.stream_ptr()))
    ns = 1 << 22
    ha = [v[:ns].cpu().numpy().view(np.uint32) for v in va]
    hb = [v[:ns].cpu().numpy().view(np.uint32) for v in vb]
    tc, ref = cpu(lambda: (ha[0] & hb[0]) ^ (ha[0] & hb[1]) ^ (ha[1] & hb[0]))
    eq = bool(np.array_equal(zo[0][:ns].cpu().numpy().view(np.uint32), ref))
    line("a11", "src/rss.py:115-126", "and_terms, 3 parties per launch (6 input + 3 output vectors)", "GB/s",
         9 * 4 * nw / t / 1e9, 32 * nw, 5 * 4 * ns / tc / 1e9, 32 * ns, eq, "negligible")
    del va, vb, zo
    # a12 Case I fold (src/engine.py:95-102,197-217), 3 parties: out_q = XOR_c fa_q(c)(A_q^B_q)[c] ^ fb_q(c) A_q[c]
    rows, words = 200_000, 1024
    comps = [torch.randint(-2**31, 2**31 - 1, (rows, words), dtype=torch.int32, device=dev, generator=gen)
             for _ in range(3)]
    fl = [torch.randint(-2**31, 2**31 - 1, ((rows + 31) // 32,), dtype=torch.int32, device=dev, generator=gen)
          for _ in range(3)]
    fo = [torch.empty((words,), dtype=torch.int32, device=dev) for _ in range(3)]
    fargs = (A(comps), A([comps[nx[q]] for q in range(3)]), A(fl), A([fl[nx[q]] for q in range(3)]), A(fo))
    t = timed(lambda: _lib.call("ogm_select_fold", rows, words, words, 3, *fargs, _lib.stream_ptr()))
    rs = 2048
    _lib.call("ogm_select_fold", rs, words, words, 3, *fargs, _lib.stream_ptr())
    hA = comps[0][:rs].cpu().numpy().view(np.uint32)
    hB = comps[1][:rs].cpu().numpy().view(np.uint32)
    bits_a = np.unpackbits(fl[0][:rs // 32].cpu().numpy().view(np.uint8), bitorder="little").astype(bool)
    bits_b = np.unpackbits(fl[1][:rs // 32].cpu().numpy().view(np.uint8), bitorder="little").astype(bool)
    tc, ref = cpu(lambda: np.bitwise_xor.reduce(np.where(bits_a[:, None], hA ^ hB, 0)
                                               ^ np.where(bits_b[:, None], hA, 0), axis=0))
    eq = bool(np.array_equal(fo[0].cpu().numpy().view(np.uint32), ref))
    line("a12", "src/engine.py:95-102", "Case I fold (select_fold, 3 parties, 200K x 1024-word rows)", "GB/s",
         3 * rows * words * 4 / t / 1e9, rows, 2 * rs * words * 4 / tc / 1e9, rs, eq, "small")
    del comps, fl, fo


# ---------------------------------------------------------------------------
# Edge-list fetch (sec_access posting fold, src/engine.py:309-311) at scale
# ---------------------------------------------------------------------------


def run_access(args):
    """The oblivious edge-list fetch's bandwidth kernel: the matched parent's
    one-hot id folded over the posting tensor (X parents x L_max slots x
    w(X_ne) words per component), all three parties in one launch.  The
    dense reference layout is infeasible at C3 (L_max = 4096 -> ~4 TB per
    component), so the C3 shape is scaled to X = X_ne =
    20,000 and L_max = 64 (3.2 GB per component).  Check: XOR of the three
    parties' additive folds equals the selected parent's plaintext posting
    row (RSS reconstruction, size-independent)."""
    dev = torch.device("cuda")
    X, L, xne = args.access_rows, 64, args.access_rows
    w = words_for(xne)
    words = L * w
    pitch = (words + 3) // 4 * 4
    comps = [workloads.device_random_words(X * pitch, args.seed, 60 + c).reshape(X, pitch) for c in range(3)]
    for c in comps:
        c[:, words:] = 0
    target = int(np.random.default_rng(args.seed).integers(0, X))
    onehot = torch.zeros((words_for(X),), dtype=torch.int32, device=dev)
    onehot[target // 32] = int(np.int32(np.uint32(1 << (target % 32))))
    s1 = workloads.device_random_words(words_for(X), args.seed, 70)
    s2 = workloads.device_random_words(words_for(X), args.seed, 71)
    if X % 32:
        s1[-1] &= (1 << (X % 32)) - 1
        s2[-1] &= (1 << (X % 32)) - 1
    sel = [s1, s2, onehot ^ s1 ^ s2]
    outs = [torch.empty((words,), dtype=torch.int32, device=dev) for _ in range(3)]
    A = _lib.ptr_array

    def fold():
        _lib.call("ogm_select_fold", X, words, pitch, 3, A(comps), A([comps[(q + 1) % 3] for q in range(3)]),
                  A(sel), A([sel[(q + 1) % 3] for q in range(3)]), A(outs), _lib.stream_ptr())

    fold()
    got = outs[0] ^ outs[1] ^ outs[2]
    want = (comps[0][target] ^ comps[1][target] ^ comps[2][target])[:words]
    ok = bool(torch.equal(got, want))
    for _ in range(args.warmup):
        fold()
    ev = events(args.steps + 1)
    ev[0].record()
    for s_ in range(args.steps):
        fold()
        ev[s_ + 1].record()
    torch.cuda.synchronize()
    ms = statistics.median(ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps))
    nbytes = 3 * X * words * 4
    emit({"config": f"edge-list fetch fold: {X} parents x L_max {L} x w(X_ne={xne})={w} words, 3 parties",
          "metric": "access_fold_GBps", "value": nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms": ms,
          "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / HBM_PEAK, "algorithmic_bytes": nbytes,
          "reconstructs_selected_row": ok})


# ---------------------------------------------------------------------------
# C5: shuffle / fetch sweep
# ---------------------------------------------------------------------------


def run_c5(args):
    import oracle

    dev = torch.device("cuda")
    cfg = make_session_configs(b"\x77" * 16)
    s12, s23, s31 = cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next
    width = 128
    W = 4
    for lg in range(args.min_log, args.max_log + 1, args.log_step):
        rows = 1 << lg
        comps = [workloads.device_random_words(rows * W, args.seed, 20 + c).reshape(rows, W) for c in range(3)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        perms = {s: seeded_permutation_device(s, b"SHPI", 0, rows) for s in (s12, s23, s31)}
        torch.cuda.synchronize()
        t_perm = time.perf_counter() - t0
        t0 = time.perf_counter()
        blinds = {
            "T12": blind_table(s12, b"SHTB", 0, rows, width), "T23": blind_table(s23, b"SHTB", 0, rows, width),
            "T31": blind_table(s31, b"SHTB", 0, rows, width), "R1": blind_table(s31, b"SHRD", 0, rows, width),
            "R2": blind_table(s12, b"SHRD", 0, rows, width)}
        torch.cuda.synchronize()
        t_blind = time.perf_counter() - t0
        pi12, pi23, pi31 = perms[s12], perms[s23], perms[s31]
        x1 = torch.empty_like(comps[0])
        y1 = torch.empty_like(comps[0])
        c1 = torch.empty_like(comps[0])
        r3 = torch.empty_like(comps[0])
        # offline phase per party (ShuffleOffline): composed perms + permuted, combined blinds
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pc = {(s, 0, rows): perms[s] for s in perms}
        # one cooperative launch up to 2^21 rows (shuffle.FUSED_MAX_BYTES), the chained planned gathers above
        fused = rows * 16 <= FUSED_MAX_BYTES
        off = [ShuffleOffline(p + 1, cfg[p].seed_with_next, cfg[p].seed_with_prev, 0, rows, width, perm_cache=pc,
                              plan=not fused)
               for p in range(3)]
        if not fused:
            for o in off:
                o.chain_blinds()
        torch.cuda.synchronize()
        t_off = time.perf_counter() - t0

        def online(pre: bool, marks=None):
            # the four party-local steps of src/shuffle.py:106-143 in protocol order
            if pre and fused and marks is None:
                shuffle_online_fused(off, comps[0], comps[1], comps[2], x1, y1, None, r3)
                return
            if pre and marks is None:
                # x1, y1, c1 handed over in shared memory; their buffers are the scratch
                shuffle_online_planned(off, comps[0], comps[1], comps[2], r3, inter=[x1, y1, c1])
                return
            if pre:
                off[0].step_x1(comps[0], comps[1], x1)
                marks and marks[1].record()
                off[1].step_y1(comps[2], y1)
                marks and marks[2].record()
                off[1].step_c1(x1, c1)
                marks and marks[3].record()
                off[2].step_r3(y1, c1, r3)
                marks and marks[4].record()
                return
            gather(rows, width, x1, outer=pi31, inner=pi12, m1=comps[0], m2=comps[1],
                   t1=(s12, b"SHTB", 0), t2=(s31, b"SHTB", 0))
            gather(rows, width, y1, inner=pi12, m1=comps[2], t1=(s12, b"SHTB", 0))
            gather(rows, width, c1, inner=pi23, m1=x1, t1=(s23, b"SHTB", 0), r=(s12, b"SHRD", 0))
            gather(rows, width, r3, outer=pi23, inner=pi31, m1=y1, t1=(s31, b"SHTB", 0),
                   t2=(s23, b"SHTB", 0), m3=c1, r=(s31, b"SHRD", 0))

        # correctness: R1 ^ R2 ^ R3 == composed-permuted plaintext (size-independent check)
        online(True)
        perm = pi12.long()[pi31.long()[pi23.long()]]
        plain = comps[0] ^ comps[1] ^ comps[2]
        ok = bool(torch.equal(blinds["R1"] ^ blinds["R2"] ^ r3, plain[perm]))
        r3_pre = r3.clone()
        online(False)
        ok = ok and bool(torch.equal(r3, r3_pre))
        # the CPU path beside it: the oracle port of src/shuffle.py:80-144 (numpy, one core) on
        # min(rows, 2^16) rows; at those sizes its R3 must equal ours bit for bit
        srows = min(rows, 1 << 16)
        host = [c[:srows].cpu().numpy().view(np.uint32) for c in comps]
        t0 = time.perf_counter()
        (_, _, o_r3), _ = oracle.shuffle_trio(s12, s23, s31, 0, host, width)
        cpu_s = time.perf_counter() - t0
        cpu = {"value": 1e3 * cpu_s * rows / srows, "unit": "ms", "cores": 1, "kind": "port",
               "sample": f"{srows} rows: oracle.shuffle_trio (numpy, src/shuffle.py:80-144) in {cpu_s:.2f}s"
                         + (", extrapolated linearly" if srows < rows else ""),
               "r3_equal": bool(np.array_equal(o_r3, r3.cpu().numpy().view(np.uint32))) if srows == rows else None}
        del perm, plain
        # tables below ~4x L2: flush L2 (write 512 MB) between timed iterations, outside the events
        flush = torch.empty((512 << 20,), dtype=torch.uint8, device=dev) if rows * 16 * 4 < (512 << 20) else None
        for pre in (True, False):
            for _ in range(args.warmup):
                online(pre)
            ev = events(2 * args.steps)
            for s in range(args.steps):
                if flush is not None:
                    flush.zero_()
                ev[2 * s].record()
                online(pre)
                ev[2 * s + 1].record()
            torch.cuda.synchronize()
            ms = statistics.median(ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(args.steps))
            step_ms = None
            if pre:
                marks = events(5)
                marks[0].record()
                online(True, marks)
                torch.cuda.synchronize()
                step_ms = {k: round(marks[i].elapsed_time(marks[i + 1]), 4)
                           for i, k in enumerate(("x1 (P1)", "y1 (P2)", "c1 (P2)", "R3 (P3)"))}
                step_ms["note"] = "the per-party steps (drop-in path), one untimed-loop run, for the breakdown"
            if pre:
                # algorithmic (protocol) bytes: x1: 2 gathers + U1 + write; y1: gather + V + write;
                # c1: gather + W + write; R3: gather + c1 + Z + write = 14 row moves (16 B) + 4 index
                # reads.  The planned two-pass execution moves more bytes physically (scratch pass).
                nbytes = rows * (14 * 16 + 4 * 4)
            else:
                # 10 row moves + 6 index reads (2 of them dependent/random); blinds by AES
                nbytes = rows * (10 * 16 + 6 * 4)
            emit({"config": f"C5 shuffle 2^{lg} rows x 128-bit", "metric": "shuffle_online_GBps",
                  "l2": "flushed between timed iterations" if flush is not None else "tables larger than L2",
                  "blinds": ("offline (ShuffleOffline: composed perms + permuted combined blinds"
                             + (", planned gathers chained through shared memory)" if not fused
                                else ", one cooperative launch)"))
                  if pre
                  else "AES-CTR on the fly, nested permutation lookups",
                  "value": nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms": ms,
                  "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / HBM_PEAK, "algorithmic_bytes_per_row": nbytes // rows,
                  "rows_per_s": rows / (ms * 1e-3), "step_ms": step_ms, "cpu_baseline": cpu, "offline_perm_s": t_perm, "offline_blinds_s": t_blind,
                  "offline_party_material_s": t_off, "bit_exact_recombination": ok})
        del off, pc
        del comps, perms, blinds, x1, y1, c1, r3, r3_pre
        torch.cuda.empty_cache()


# ---------------------------------------------------------------------------
# C5 leg of bench.py: shuffle of 128-bit rows + the 1% / 10% / 100% fetch
# ---------------------------------------------------------------------------


def _timed_steps(fn, steps: int, warmup: int, flush: torch.Tensor | None) -> float:
    """ms per step: CUDA events around each step on the launching stream,
    the L2 flush (when given) outside them."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = events(2 * steps)
    for k in range(steps):
        if flush is not None:
            flush.zero_()
        ev[2 * k].record()
        fn()
        ev[2 * k + 1].record()
    torch.cuda.synchronize()
    return sum(ev[2 * k].elapsed_time(ev[2 * k + 1]) for k in range(steps)) / steps


def _bits_of(words: torch.Tensor, n: int) -> torch.Tensor:
    """Packed bit vector -> (n,) int32 0/1 (device)."""
    sh = torch.arange(32, device=words.device, dtype=torch.int32)
    return ((words[: (n + 31) // 32].unsqueeze(1) >> sh) & 1).reshape(-1)[:n]


def _random_bits(n: int, seed: int, stream_id: int) -> torch.Tensor:
    w = workloads.device_random_words(words_for(n), seed, stream_id)
    if n % 32:
        w[-1] &= (1 << (n % 32)) - 1
    return w


def _bernoulli_bits(n: int, p: float, seed: int) -> torch.Tensor:
    """Packed Bernoulli(p) bits (device, seeded)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    b = (torch.rand(n, device="cuda", generator=g) < p).to(torch.int64)
    pad = (-n) % 32
    if pad:
        b = torch.cat([b, torch.zeros(pad, dtype=torch.int64, device="cuda")])
    w = (b.reshape(-1, 32) << torch.arange(32, device="cuda", dtype=torch.int64)).sum(1)
    return torch.where(w >= (1 << 31), w - (1 << 32), w).to(torch.int32)


def c5_shuffle_leg(lg: int, steps: int, warmup: int, seed: int = 1) -> dict:
    """C5 (BASELINE configs[4]): the three-party shuffle of 2^lg rows x 128
    bits, offline material prepared (ShuffleOffline), online phase timed:
    one cooperative launch up to 2^21 rows, the chained planned gathers above.
    Gate: R1 ^ R2 ^ R3 == the plaintext table under the composed permutation,
    at full size, plus the oracle port's R3 bit for bit on a 2^16-row run."""
    import oracle

    rows = 1 << lg
    cfg = make_session_configs(b"\x77" * 16)
    seeds = (cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next)
    comps = [workloads.device_random_words(rows * 4, seed, 20 + c).reshape(rows, 4) for c in range(3)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pc: dict = {}
    fused = rows * 16 <= FUSED_MAX_BYTES
    pairs = [(seeds[0], seeds[2]), (seeds[1], seeds[0]), (seeds[2], seeds[1])]
    off = [ShuffleOffline(p + 1, *pairs[p], 0, rows, 128, perm_cache=pc, plan=not fused) for p in range(3)]
    if not fused:
        for o in off:
            o.chain_blinds()
    torch.cuda.synchronize()
    t_off = time.perf_counter() - t0
    r3 = torch.empty_like(comps[0])
    inter = [torch.empty_like(comps[0]) for _ in range(3)]

    def online():
        if fused:
            shuffle_online_fused(off, comps[0], comps[1], comps[2], inter[0], inter[1], None, r3)
        else:
            shuffle_online_planned(off, comps[0], comps[1], comps[2], r3, inter=inter)

    flush = torch.empty((512 << 20,), dtype=torch.uint8, device="cuda") if rows * 16 * 4 < (512 << 20) else None
    ms = _timed_steps(online, steps, warmup, flush)
    pi12, pi23, pi31 = (pc[(s, 0, rows)].long() for s in seeds)
    perm = pi12[pi31[pi23]]
    ok = bool(torch.equal(off[0].out_a ^ off[0].out_b ^ r3, (comps[0] ^ comps[1] ^ comps[2])[perm]))
    del perm, pi12, pi23, pi31, off, pc, inter
    torch.cuda.empty_cache()
    # CPU path beside it: oracle.shuffle_trio (numpy, 1 core) on a 2^16-row run, R3 compared
    srows = min(rows, 1 << 16)
    sc = [c[:srows].contiguous() for c in comps]
    soff = [ShuffleOffline(p + 1, *pairs[p], 0, srows, 128, plan=False) for p in range(3)]
    sr3 = torch.empty_like(sc[0])
    shuffle_online_fused(soff, sc[0], sc[1], sc[2], torch.empty_like(sc[0]), torch.empty_like(sc[0]), None, sr3)
    host = [c.cpu().numpy().view(np.uint32) for c in sc]
    t0 = time.perf_counter()
    (_, _, o_r3), _ = oracle.shuffle_trio(*seeds, 0, host, 128)
    cpu_s = time.perf_counter() - t0
    sample_equal = bool(np.array_equal(o_r3, sr3.cpu().numpy().view(np.uint32)))
    nbytes = rows * (14 * 16 + 4 * 4)
    return {"rows": rows, "ms": ms, "GBps": nbytes / (ms * 1e-3) / 1e9,
            "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / HBM_PEAK, "algorithmic_bytes_per_row": 240,
            "path": "one cooperative launch" if fused else "chained planned gathers (5 launches)",
            "offline_s": t_off, "l2": "flushed between steps" if flush is not None else "tables larger than L2",
            "gate": {"recombination_full_size": ok, "r3_equal_to_oracle_on_2^16_run": sample_equal},
            "cpu_baseline": {"value": 1e3 * cpu_s * rows / srows, "unit": "ms", "cores": 1, "kind": "port",
                             "sample": f"{srows} rows: oracle.shuffle_trio (numpy, src/shuffle.py:80-144) in "
                                       f"{cpu_s:.3f}s, extrapolated linearly to {rows} rows"}}


def c5_fetch_leg(lg: int, steps: int, warmup: int, ps=(0.01, 0.1, 1.0), seed: int = 1) -> list:
    """C5 fetch (BASELINE configs[4], "oblivious fetch of 1%, 10% and 100% of
    rows"): sec_fetch_multi (src/engine.py:220-270) of rows = flag + 128-bit
    id (129 bits), shuffled, flag column opened, flagged rows kept; the
    flag-split trio path (fetch.FlaggedFetch), offline material prepared once
    per size, online phase timed per p.  Gates at full size: the opened
    column equals the plaintext flags under the composed permutation, and
    the kept records recombine to the plaintext rows in shuffled order; on a
    2^16-row run every record share equals the oracle's sec_fetch_multi."""
    import oracle
    from paper_2209_03526_b200.fetch import FlaggedFetch

    rows = 1 << lg
    cfg = make_session_configs(b"\x78" * 16)
    seeds = (cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next)
    payload = [workloads.device_random_words(rows * 4, seed, 30 + c).reshape(rows, 4) for c in range(3)]
    f12 = [_random_bits(rows, seed, 40), _random_bits(rows, seed, 41)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pc: dict = {}
    ff = FlaggedFetch(seeds, 0, rows, perm_cache=pc)
    torch.cuda.synchronize()
    t_off = time.perf_counter() - t0
    pi12, pi23, pi31 = (pc[(s, 0, rows)].long() for s in seeds)
    perm = pi12[pi31[pi23]]
    del pi12, pi23, pi31
    plain_rows = (payload[0] ^ payload[1] ^ payload[2])[perm]
    flush = torch.empty((512 << 20,), dtype=torch.uint8, device="cuda") if rows * 16 * 4 < (512 << 20) else None
    out = []
    for i, p in enumerate(ps):
        fp = _bernoulli_bits(rows, p, seed + 100 + i)
        flags = [f12[0], f12[1], fp ^ f12[0] ^ f12[1]]
        ms = _timed_steps(lambda: ff.online(flags, payload), steps, warmup, flush)
        k = ff.kept()
        opened = _bits_of(ff.plain, rows)
        ok_open = bool(torch.equal(opened, _bits_of(fp, rows)[perm]))
        kept_idx = torch.nonzero(opened).reshape(-1)
        recs = ff.records()
        ok_recs = k == kept_idx.numel() and bool(torch.equal(recs[0] ^ recs[1] ^ recs[2], plain_rows[kept_idx]))
        del kept_idx, opened, recs
        # algorithmic bytes: 14 moves of a 129-bit row + 4 index reads (the shuffle), the open's
        # three flag columns, and per kept row three 16-B payload reads + writes
        nbytes = rows * (14 * 129 / 8 + 16 + 3 / 8) + k * 6 * 16
        out.append({"rows": rows, "p": p, "kept": k, "ms": ms, "GBps": nbytes / (ms * 1e-3) / 1e9,
                    "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / HBM_PEAK,
                    "algorithmic_bytes_per_row": nbytes / rows,
                    "survey_bytes_per_row": 248 + 12 * p * 16,
                    "path": ("flag-split: 16-B payload shuffle ("
                             + ("one cooperative launch" if ff.fused else "chained planned gathers")
                             + ") + flag-column bit gathers (2 launches) + hand-written keep (3 launches)"),
                    "offline_s": t_off, "l2": "flushed between steps" if flush is not None else "tables larger than L2",
                    "gate": {"opened_equals_permuted_flags": ok_open, "records_recombine": ok_recs}})
        if not (ok_open and ok_recs):
            raise SystemExit(f"C5 fetch gate failed at 2^{lg} rows, p={p}")
    del ff, pc, perm, plain_rows, payload, f12
    torch.cuda.empty_cache()
    # the CPU path beside it: oracle.fetch_multi_trio (numpy, 1 core) on 2^16 rows at p = 0.1, and our
    # fetch on the same 2^16-row inputs, record share for record share
    srows = min(rows, 1 << 16)
    rng = np.random.default_rng(seed)
    ids = [rng.integers(0, 1 << 32, size=(srows, 4), dtype=np.uint32) for _ in range(3)]
    fl = [oracle.pack_bits(rng.integers(0, 2, srows, dtype=np.uint8)) for _ in range(2)]
    fl.append(oracle.pack_bits((rng.random(srows) < 0.1).astype(np.uint8)) ^ fl[0] ^ fl[1])
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32).copy()).cuda()  # noqa: E731
    sf = FlaggedFetch(seeds, 0, srows)
    sf.online([dev(f) for f in fl], [dev(m) for m in ids])
    t0 = time.perf_counter()
    keep, _, want = oracle.fetch_multi_trio(*seeds, 0, fl, ids, 128)
    cpu_s = time.perf_counter() - t0
    got = sf.records()
    equal = keep.size == got[0].shape[0] and all(
        np.array_equal(g.cpu().numpy().view(np.uint32), w) for g, w in zip(got, want))
    for o in out:
        o["gate"]["records_equal_to_oracle_on_2^16_run"] = equal
        o["cpu_baseline"] = {"value": 1e3 * cpu_s * rows / srows, "unit": "ms", "cores": 1, "kind": "port",
                             "sample": f"{srows} rows, p=0.1: oracle.fetch_multi_trio (numpy, src/engine.py:220-270) "
                                       f"in {cpu_s:.3f}s, extrapolated linearly to {rows} rows"}
    if not equal:
        raise SystemExit("C5 fetch differs from the oracle on the 2^16-row run")
    return out


# ---------------------------------------------------------------------------
# C3 root-slot pipeline (trio fast path): secEval x2 -> combine -> Case II fetch
# ---------------------------------------------------------------------------


def c3p_setup(args):
    """Root-slot shares and tokens of the C3 pipeline (seeded, on the device)."""
    from paper_2209_03526_b200.trio import TrioGroup

    X = args.rows
    dev = torch.device("cuda")
    rng = np.random.default_rng(args.seed)
    n0, n2 = 182083, 8969
    v0 = torch.from_numpy(rng.integers(0, n0, size=X).astype(np.int32)).to(dev)
    ranks = np.arange(1, n2 + 1)
    pz = 1.0 / ranks ** 1.1
    v2h = rng.choice(n2, size=X, p=pz / pz.sum()).astype(np.int32)
    v2 = torch.from_numpy(v2h).to(dev)
    ids = workloads.shared_one_hot(torch.arange(X, dtype=torch.int32, device=dev), X, args.seed, 60)
    a0 = workloads.shared_one_hot(v0, n0, args.seed, 70)
    a2 = workloads.shared_one_hot(v2, n2, args.seed, 80)
    torch.cuda.synchronize()
    lo = int(rng.integers(0, n0 // 2))
    hi = lo + n0 // 10
    v0h = v0.cpu().numpy()
    inside = (v0h >= lo) & (v0h <= hi)
    cnt_all = np.bincount(v2h, minlength=n2)
    cnt_in = np.bincount(v2h[inside], minlength=n2)
    cand = np.nonzero((cnt_in >= 1) & (cnt_all <= 6))[0]  # a rare Zipf value with matches in range
    rare = int(cand[0])
    match_rows = np.flatnonzero((v2h == rare) & inside)
    want = int(match_rows.size)
    krng = np.random.default_rng(args.seed + 5)
    iv = [fss.ic_gen(lo, hi, n0, krng) for _ in range(3)]
    eq = list(fss.bundle_gen("eq", (rare,), n2, krng).pairs)

    def split(pairs):
        (k11, k21), (k12, k22), (k13, k23) = pairs
        return [(k11, k12), (k22, k13), (k23, k21)]

    kiv, keq = split(iv), split(eq)
    group = TrioGroup(None, None, X, X, list(ids), {"a0": list(a0), "a2": list(a2)}, {"a0": n0, "a2": n2})
    group.expected_rows = set(int(r) for r in match_rows)   # the plaintext answer, for the gates
    return group, kiv, keq, n0, n2, want


def run_c3_pipeline(args):
    """Root slot of the medium graph: 200K centre vertices, one-hot ids (200K
    bits) and two needed attributes (uniform a0, n=182,083; Zipf a2, n=8,969).
    Predicates: a0 in [lo, hi] (interval, 2 passes) AND a2 = rare value (DPF);
    combine (1 AND); Case II fetch: shuffle of 200K rows x 391,053 bits (48.9 KB
    per row, 9.8 GB per component -- SURVEY 8(d) C3 'feasible' row), open the
    flags, keep the matches.  Blinds on the fly (memory-lean)."""
    from paper_2209_03526_b200.trio import Trio

    X = args.rows
    group, kiv, keq, n0, n2, want = c3p_setup(args)
    phases = {}
    lat = []
    for it in range(args.warmup + args.steps):
        trio = Trio(b"\x35" * 16)
        audit: list = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        b_iv = trio.sec_eval(group, kiv, "a0", n0, {})
        b_eq = trio.sec_eval(group, keq, "a2", n2, {})
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        flags = trio.combine([b_iv, b_eq], "ALL", "or", X)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        # offline phase of the fetch's shuffle (data-independent), timed apart
        trio.prepare_shuffle(X, 1 + X + n0 + n2)
        torch.cuda.synchronize()
        t_off = time.perf_counter()
        recs = trio.fetch_multi(group, flags, audit)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        if it >= args.warmup:
            lat.append((t3 - t_off) + (t2 - t0))
            for k, v in (("secEval_ms", t1 - t0), ("combine_ms", t2 - t1), ("fetch_online_ms", t3 - t_off),
                         ("fetch_offline_prep_ms", t_off - t2)):
                phases.setdefault(k, []).append(1e3 * v)
        recs_count = recs.count
        del recs, flags, b_iv, b_eq  # buffers return to the caching allocator (warm, as in a serving loop)
    torch.cuda.empty_cache()
    row_width = 1 + X + n0 + n2
    emit({"config": f"C3 root-slot pipeline: {X} candidates, a0 interval + a2 eq, ALL, Case II fetch of "
                    f"{row_width}-bit rows", "metric": "root_slot_latency_ms", "value": 1e3 * statistics.median(lat),
          "unit": "ms", "higher_is_better": False, "phases_ms": {k: statistics.median(v) for k, v in phases.items()},
          "matches_expected": want, "opened_ones": int(audit[0][1].sum()) if audit else None,
          "fetch_table_GB_per_component": X * words_for(row_width) * 4 / 1e9,
          "kept_records": int(recs_count), "path": "trio fast path; latency = online (shuffle material prepared "
          "offline, reported separately)"})


def c3_leg(steps: int, warmup: int, rows: int = 200_000, seed: int = 1) -> dict:
    """C3 (BASELINE configs[2]) root slot for bench.py: the run_c3_pipeline
    workload (200K centre vertices; a0 interval over the uniform attribute
    (w = 5691 words) AND a2 = rare value over the Zipf attribute; combine;
    Case II fetch of 391,053-bit rows = 9.8 GB per component), one trio
    query per step with the fetch's shuffle material prepared offline.
    Gates: the opened flags equal the plaintext predicate for every
    candidate, the kept records decode to exactly the matching vertices, and
    the secEval bits equal the oracle port's on a 2,000-row sample."""
    import types

    from paper_2209_03526_b200.trio import Trio

    args = types.SimpleNamespace(rows=rows, seed=seed)
    group, kiv, keq, n0, n2, want = c3p_setup(args)
    online, secev, fetch_ms, offline = [], [], [], []
    for it in range(warmup + steps):
        trio = Trio(b"\x35" * 16)
        audit: list = []
        ev = events(4)
        torch.cuda.synchronize()
        ev[0].record()
        b_iv = trio.sec_eval(group, kiv, "a0", n0, {})
        b_eq = trio.sec_eval(group, keq, "a2", n2, {})
        flags = trio.combine([b_iv, b_eq], "ALL", "or", rows)
        ev[1].record()
        t0 = time.perf_counter()
        trio.prepare_shuffle(rows, 1 + rows + n0 + n2)    # offline (data-independent), timed apart
        torch.cuda.synchronize()
        t_off = time.perf_counter() - t0
        ev[2].record()
        recs = trio.fetch_multi(group, flags, audit)
        ev[3].record()
        torch.cuda.synchronize()
        if it >= warmup:
            secev.append(ev[0].elapsed_time(ev[1]))
            fetch_ms.append(ev[2].elapsed_time(ev[3]))
            online.append(secev[-1] + fetch_ms[-1])
            offline.append(1e3 * t_off)
        if it < warmup + steps - 1:
            del recs, flags, b_iv, b_eq
    # gates: opened flags == plaintext predicate; records decode to exactly the matching vertices
    opened = audit[0][1].astype(bool)
    kept = int(opened.sum())
    ids = [c.cpu().numpy().view(np.uint32) for c in recs.ids]
    onehot = ids[0] ^ ids[1] ^ ids[2]
    got = set()
    for r in range(onehot.shape[0]):
        nz = np.flatnonzero(onehot[r])
        got.add(int(nz[0]) * 32 + int(onehot[r, nz[0]]).bit_length() - 1 if nz.size else -1)
    return {"config": f"C3 root slot: {rows} candidates, a0 interval (n={n0}) AND a2 eq (n={n2}); Case II fetch of "
                      f"{1 + rows + n0 + n2}-bit rows ({rows * words_for(1 + rows + n0 + n2) * 4 / 1e9:.1f} GB per "
                      "component)",
            "metric": "root_slot_online_ms", "ms": statistics.median(online), "unit": "ms",
            "secEval_combine_ms": statistics.median(secev), "fetch_online_ms": statistics.median(fetch_ms),
            "fetch_offline_ms": statistics.median(offline),
            # the trio path reads each share component once for all parties and both interval passes
            "secEval_read_GB": 3 * rows * (words_for(n0) + words_for(n2)) * 4 / 1e9,
            "secEval_hbm_frac": 3 * rows * (words_for(n0) + words_for(n2)) * 4 / (statistics.median(secev) * 1e-3)
            / 1e9 / HBM_PEAK,
            # fetch: 14 moves of the 16-byte-pitched row (the shuffle), blinds generated on the fly
            "fetch_row_bytes": 4 * ((words_for(1 + rows + n0 + n2) + 3) // 4 * 4),
            "fetch_hbm_frac": 14 * rows * 4 * ((words_for(1 + rows + n0 + n2) + 3) // 4 * 4)
            / (statistics.median(fetch_ms) * 1e-3) / 1e9 / HBM_PEAK,
            "gate": {"kept_equals_plaintext_count": kept == want and recs.count == want,
                     "records_are_the_matching_vertices": got == group.expected_rows},
            "matches": want, "path": "trio fast path (Trio.sec_eval x2, combine, fetch_multi with prepared material)"}


# ---------------------------------------------------------------------------
# C4: large graph, root-slot secEval on the Zipf attribute, rows sharded
# across ranks (torchrun, one process per GPU; NCCL all-gather of match bits)
# ---------------------------------------------------------------------------


def c4_root_slot(rows: int, seed: int, steps: int, warmup: int, rank: int, world: int) -> dict:
    """C4 (BASELINE configs[3]) root slot end to end: two predicates over the
    two Zipf attributes (a2 in [100, 4000]: DCF interval, 2 passes; a3 = v*:
    DPF), combined with AND, then the Case II fetch of the matches.

    secEval runs row-sharded (sharded_trio.ShardedTrio: one all-gather per
    predicate); combine is replicated.  The fetch cannot use the reference's
    row layout here (a one-hot id over 2M vertices is 250 KB per row, 500 GB
    per component -- SURVEY Appendix B), so it fetches flag + a 128-bit
    compact record per vertex (vertex index and the two attribute values)
    through the pinned C5 fetch path (Trio.fetch_multi, flag-split), with the
    32 MB record table replicated on every rank.  The record encoding is
    outside the reference layout (parity of that choice unpinned); the
    secEval, combine and fetch arithmetic are the pinned paths.  Gates: the
    opened flags equal the plaintext predicate on every row and the kept
    records recombine to the matching vertices' records."""
    import torch.distributed as dist

    from paper_2209_03526_b200.sharded_trio import ShardedGroup, ShardedTrio
    from paper_2209_03526_b200.sharding import ShardPlan, ThreadComm

    n = 10_000
    plan = ShardPlan(rows, world)
    lo, hi = plan.bounds(rank)
    rng = np.random.default_rng(seed)
    pz = 1.0 / np.arange(1, n + 1) ** 1.1
    pz /= pz.sum()
    a2 = rng.choice(n, size=rows, p=pz).astype(np.int32)
    a3 = rng.choice(n, size=rows, p=pz).astype(np.int32)
    v_star = 7                                    # a3 value with ~1% frequency under Zipf(1.1)
    want = (a2 >= 100) & (a2 <= 4000) & (a3 == v_star)
    c2 = list(workloads.shared_one_hot(torch.from_numpy(a2[lo:hi]).cuda(), n, seed, 40, row0=lo))
    c3 = list(workloads.shared_one_hot(torch.from_numpy(a3[lo:hi]).cuda(), n, seed, 50, row0=lo))
    ids_dummy = [torch.zeros((hi - lo, 1), dtype=torch.int32, device="cuda") for _ in range(3)]
    group = ShardedGroup(None, None, rows, 32, ids_dummy, {"a2": c2, "a3": c3}, {"a2": n, "a3": n},
                         plan=plan, rank=rank)
    krng = np.random.default_rng(seed + 1)          # identical keys on every rank

    def split(pairs):
        (k11, k21), (k12, k22), (k13, k23) = pairs
        return [(k11, k12), (k22, k13), (k23, k21)]

    kiv = split([fss.ic_gen(100, 4000, n, krng) for _ in range(3)])
    keq = split(list(fss.bundle_gen("eq", (v_star,), n, krng).pairs))
    # compact records: (vertex index, a2, a3, 0) shared three ways, replicated (32 MB per component)
    plain = torch.from_numpy(np.stack([np.arange(rows, dtype=np.int32), a2, a3, np.zeros(rows, np.int32)], 1)).cuda()
    r1 = workloads.device_random_words(rows * 4, seed, 60).reshape(rows, 4)
    r2 = workloads.device_random_words(rows * 4, seed, 61).reshape(rows, 4)
    rec_comps = [r1, r2, plain ^ r1 ^ r2]
    fetch_group = None
    tim = {"secEval_ms": [], "combine_ms": [], "fetch_ms": [], "total_ms": []}
    for it in range(warmup + steps):
        trio = ShardedTrio(b"\x4c" * 16, None if world > 1 else ThreadComm(1).rank_view(0))
        trio.prepare_fetch(rows)                    # offline: the fetch's shuffle material (table id 0)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev = events(4)
        ev[0].record()
        b_iv = trio.sec_eval(group, kiv, "a2", n, {})
        b_eq = trio.sec_eval(group, keq, "a3", n, {})
        ev[1].record()
        flags = trio.combine([b_iv, b_eq], "ALL", "or", rows)
        ev[2].record()
        fetch_group = TrioGroup(None, None, rows, 128, rec_comps, {}, {})
        audit: list = []
        recs = trio.fetch_multi(fetch_group, flags, audit)
        ev[3].record()
        torch.cuda.synchronize()
        if it >= warmup:
            for k, (a, b) in (("secEval_ms", (0, 1)), ("combine_ms", (1, 2)), ("fetch_ms", (2, 3)),
                              ("total_ms", (0, 3))):
                tim[k].append(ev[a].elapsed_time(ev[b]))
    med = {k: statistics.median(v) for k, v in tim.items()}
    if world > 1:
        t = torch.tensor([med["total_ms"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        med["total_ms"] = float(t.item())
    opened = audit[0][1].astype(bool)
    got = (recs.ids[0] ^ recs.ids[1] ^ recs.ids[2]).cpu().numpy()
    ok_open = int(opened.sum()) == int(want.sum())
    ok_recs = bool(np.array_equal(np.sort(got[:, 0]), np.flatnonzero(want))) and bool(
        np.array_equal(got[np.argsort(got[:, 0]), 1:3], np.stack([a2, a3], 1)[want]))
    nbytes_local = 3 * (hi - lo) * 2 * words_for(n) * 4
    return {"config": f"C4 root slot: {rows} candidates, a2 in [100, 4000] (Zipf, n={n}) AND a3 = {v_star}; "
                      f"Case II fetch of compact 128-bit records; rows sharded x{world}",
            "metric": "root_slot_ms", "ms": med["total_ms"], "unit": "ms", "n_gpus": world,
            "phases_ms": {k: med[k] for k in ("secEval_ms", "combine_ms", "fetch_ms")},
            "matches": int(want.sum()), "kept": int(recs.count),
            "rank0_secEval_hbm_frac": nbytes_local / (med["secEval_ms"] * 1e-3) / 1e9 / HBM_PEAK,
            "fetch": "flag + 128-bit compact record (vertex index, a2, a3), replicated table; the reference "
                     "layout's one-hot id row is 500 GB per component at this size (SURVEY Appendix B)",
            "gate": {"opened_count_equals_plaintext": ok_open and int(recs.count) == int(want.sum()),
                     "records_are_the_matches": ok_recs}}


def c4_sec_eval(rows: int, seed: int, steps: int, warmup: int, rank: int, world: int) -> dict:
    """C4 (BASELINE configs[3]) root-slot secEval, row-sharded over `world`
    ranks (an initialised NCCL group when world > 1): 2M candidates of one
    vertex type (16M vertices / 8 types), Zipf(1.1) attribute over 10^4
    values, an interval predicate (2 DCF passes, folded into one parity pass
    over XORed indicators with both zero shares XORed in -- the co-resident
    trio's secEval, same result shares) for all three parties, match bits
    all-gathered.  Strong scaling; device time max over ranks.

    Shares are drawn by GLOBAL row (workloads.shared_one_hot row0), so every
    world size shares the same table; rank 0 then gates the all-gathered
    result bit for bit against the oracle port on rows taken from EVERY
    rank's shard (regenerated from the same streams)."""
    import torch.distributed as dist

    from paper_2209_03526_b200.sharding import ShardPlan, fold_indicators, sharded_sec_eval_trio

    n = 10_000
    plan = ShardPlan(rows, world)
    lo, hi = plan.bounds(rank)
    rng = np.random.default_rng(seed)
    ranks = np.arange(1, n + 1)
    p = 1.0 / ranks ** 1.1
    vals_all = rng.choice(n, size=rows, p=p / p.sum()).astype(np.int32)
    vals = torch.from_numpy(vals_all[lo:hi]).cuda()
    comps = list(workloads.shared_one_hot(vals, n, seed, 40, row0=lo))
    w = words_for(n)
    krng = np.random.default_rng(seed + 1)  # identical keys on every rank
    pairs = [fss.ic_gen(100, 4000, n, krng) for _ in range(3)]
    (k11, k21), (k12, k22), (k13, k23) = pairs
    keys = [(k11, k12), (k22, k13), (k23, k21)]
    inds = [[(fss.full_domain(fss.KeyBatch.from_keys([fss.key_parts_for_engine(keys[q][0])[ps]]), n)[0],
              fss.full_domain(fss.KeyBatch.from_keys([fss.key_parts_for_engine(keys[q][1])[ps]]), n)[0])
             for q in range(3)] for ps in range(2)]
    cfg = make_session_configs(b"\x44" * 16)
    zk = [(c.zero_key_own, c.zero_key_prev) for c in cfg]
    # the two passes folded into one parity pass (the co-resident trio's secEval, ShardedTrio.sec_eval)
    folded = fold_indicators(inds)
    step = lambda: sharded_sec_eval_trio(comps, w, plan, rank, folded, zk, [0, 1], fold=True)  # noqa: E731
    # warm up with the timed loop's reference pattern (the previous result alive while the next
    # is allocated), so the caching allocator holds both buffers and the timed loop never calls
    # cudaMalloc: a driver allocation right after the previous leg's empty_cache stalled the
    # host-driven launches (1.08 -> 2.6-8 ms per step seen, intermittently)
    res = None
    for _ in range(max(warmup, 2)):
        res = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = events(steps + 1)
    host_ms = []
    ev[0].record()
    for i in range(steps):
        h0 = time.perf_counter()
        res = step()
        host_ms.append(1e3 * (time.perf_counter() - h0))
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[steps]) / steps
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    nbytes_local = 3 * (hi - lo) * w * 4
    cpu = gate = None
    if rank == 0:
        import oracle

        zero = {(p_, ps): oracle.zero_share(zk[p_][0], zk[p_][1], ps, rows) for p_ in range(3) for ps in range(2)}

        def gpu_bits(p_, ps=None):  # undo the re-share blinding: additive bits = result ^ both zero shares
            return res[0][p_].cpu().numpy().view(np.uint32) ^ zero[(p_, 0)] ^ zero[(p_, 1)]

        if world == 1:
            cpu = cpu_port_sec_eval(comps, w, lambda p_, ps: inds[ps][p_], gpu_bits, 20000, folded=True)
        # N-rank parity gate: 2048 rows from the start of every shard, shares regenerated by global row
        per = 2048
        checked, equal = 0, True
        full = {p_: oracle.unpack_bits(gpu_bits(p_), rows) for p_ in range(3)}
        for r in range(world):
            r_lo, r_hi = plan.bounds(r)
            m = min(per, r_hi - r_lo)
            if m <= 0:
                continue
            sub = torch.from_numpy(vals_all[r_lo:r_lo + m]).cuda()
            sc = [c.cpu().numpy().view(np.uint32) for c in workloads.shared_one_hot(sub, n, seed, 40, row0=r_lo)]
            for p_ in range(3):
                want = 0
                for ps in range(2):
                    ia = inds[ps][p_][0].cpu().numpy().view(np.uint32)[:w]
                    ib = inds[ps][p_][1].cpu().numpy().view(np.uint32)[:w]
                    want = want ^ oracle.masked_parity(sc[p_], sc[(p_ + 1) % 3], ia, ib)
                equal = equal and bool(np.array_equal(want, full[p_][r_lo:r_lo + m]))
            checked += m
        gate = {"rows_checked": checked, "shards_checked": world, "equal_to_oracle": equal,
                "how": "all-gathered re-shared bits ^ both passes' zero shares == the XOR of the two passes' "
                       f"oracle.masked_parity on the first {per} rows of every rank's shard (shares drawn by "
                       "global row)"}
        if not equal:
            raise SystemExit("C4 sharded secEval differs from the oracle port")
    return {"config": f"C4 root secEval, {rows} candidates (Zipf attr n={n}, w={w}), interval, "
                      f"rows sharded x{world}", "metric": "secEval_candidates_per_s",
            "value": rows / (ms * 1e-3), "unit": "candidates/s", "ms_per_step": ms, "n_gpus": world,
            "scaling": "strong", "rank0_hbm_GBps": nbytes_local / (ms * 1e-3) / 1e9,
            "rank0_hbm_frac": nbytes_local / (ms * 1e-3) / 1e9 / HBM_PEAK,
            "collective": "NCCL all_gather of packed blinded match bits" if world > 1 else "none",
            "result_words": int(res[0][0].numel()), "cpu_baseline": cpu, "parity_gate": gate,
            "rank0_step_ms": [round(x, 4) for x in step_ms], "rank0_host_enqueue_ms": [round(x, 4) for x in host_ms]}


def run_c4(args):
    import os

    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    line = c4_sec_eval(args.c4_rows, args.seed, args.steps, args.warmup, rank, world)
    if rank == 0:
        emit(line)
    if world > 1:
        dist.destroy_process_group()


def run_c5_sharded(args):
    """C5 under torchrun: rows sharded across ranks, each online step = local
    pack + NCCL all_to_all + local unpack (sharding.ShardedTrioShuffle)."""
    import os

    import torch.distributed as dist

    from paper_2209_03526_b200.sharding import ShardedTrioShuffle, ShardPlan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                            **({} if "MASTER_ADDR" in os.environ else
                               {"init_method": "tcp://127.0.0.1:29555", "rank": 0, "world_size": 1}))
    cfg = make_session_configs(b"\x77" * 16)
    seeds = (cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next)
    width = 128
    for lg in range(args.min_log, args.max_log + 1, args.log_step):
        rows = 1 << lg
        plan = ShardPlan(rows, world, align=1)
        lo, hi = plan.bounds(rank)
        comps = [workloads.device_random_words(rows * 4, args.seed, 20 + c).reshape(rows, 4)[lo:hi].clone()
                 for c in range(3)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sh = ShardedTrioShuffle(seeds, 0, rows, width, plan, rank)
        torch.cuda.synchronize()
        t_off = time.perf_counter() - t0
        for _ in range(args.warmup):
            out = sh.online(comps)
        torch.cuda.synchronize()
        dist.barrier()
        ev = events(2)
        ev[0].record()
        for _ in range(args.steps):
            out = sh.online(comps)
        ev[1].record()
        torch.cuda.synchronize()
        ms = torch.tensor([ev[0].elapsed_time(ev[1]) / args.steps], device="cuda")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        ms = float(ms.item())
        nbytes = rows * (14 * 16 + 4 * 4)
        if rank == 0:
            emit({"config": f"C5 shuffle 2^{lg} rows x 128-bit, rows sharded x{world}", "metric": "shuffle_online_GBps",
                  "value": nbytes / (ms * 1e-3) / 1e9, "unit": "GB/s", "ms": ms, "n_gpus": world,
                  "hbm_frac_per_gpu": nbytes / world / (ms * 1e-3) / 1e9 / HBM_PEAK,
                  "offline_s": t_off, "cross_gpu_bytes_per_rank": int(4 * rows * 16 * (world - 1) / world / world),
                  "path": "ShardedTrioShuffle: pack + all_to_all + unpack per step"})
        del comps, sh, out
        torch.cuda.empty_cache()
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["c1", "c3", "c3p", "c4", "c5", "c5d", "access", "funcs", "all"])
    ap.add_argument("--access-rows", type=int, default=20_000)
    ap.add_argument("--c4-rows", type=int, default=2_000_000)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--rows", type=int, default=200_000)
    ap.add_argument("--min-log", type=int, default=16)
    ap.add_argument("--max-log", type=int, default=28)
    ap.add_argument("--log-step", type=int, default=2)
    args = ap.parse_args()
    _lib.check(_lib.load().ogm_init())
    if args.which in ("c1", "all"):
        run_c1(args)
    if args.which in ("c3", "all"):
        run_c3(args)
    if args.which in ("c5", "all"):
        run_c5(args)
    if args.which == "c4":
        run_c4(args)
    if args.which == "c3p":
        run_c3_pipeline(args)
    if args.which == "c5d":
        run_c5_sharded(args)
    if args.which in ("access", "all"):
        run_access(args)
    if args.which in ("funcs", "all"):
        run_funcs(args)


if __name__ == "__main__":
    main()
