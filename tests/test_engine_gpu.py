"""GPU parity of the protocol layer against the live reference's recorded runs.

Every case re-runs the reference's three-party protocol on the B200 (three
party threads, one CUDA stream each, device-resident messages) from the same
inputs and session master, and requires bit-identical output shares, opened
values and per-party transcript digests (SHA-256 over every frame, in the
reference's encoding, src/net.py:288-295) -- so every message byte matches.
"""

import json

import numpy as np
import pytest
import torch

from paper_2209_03526_b200 import fss, rss
from paper_2209_03526_b200.bits import BitVector, words_for
from paper_2209_03526_b200.engine import (CandidateGroup, EngineConfig, _OpenLabels, combine_predicates,
                                          open_results, sec_eval, sec_fetch_multi, sec_fetch_unique, sec_match)
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph, parse_graph_text
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
from paper_2209_03526_b200.query import gen_token, load_query, serialize_token
from paper_2209_03526_b200.rss import DBits, SharedBitVector
from paper_2209_03526_b200.shuffle import MatchTable, sec_shuffle

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32).copy()).cuda()


def host(t):
    return t.detach().cpu().numpy().view(np.uint32)


def digest(g, key):
    return bytes(g[key]).hex()


def make_groups(g, tag, count, domain, with_ids=True, padded=False):
    from paper_2209_03526_b200.graphs import padded_device_matrix
    attr = [padded_device_matrix(g[f"{tag}_attr{c}"]) if padded else dev(g[f"{tag}_attr{c}"]) for c in range(3)]
    if with_ids and f"{tag}_id0" in g:
        ids = [dev(g[f"{tag}_id{c}"]) for c in range(3)]
    else:
        w = (count + 31) // 32
        ids = [torch.zeros((count, w), dtype=torch.int32, device="cuda") for _ in range(3)]
    return [CandidateGroup(None, None, count, count, ids[p], ids[(p + 1) % 3],
                           {"a": (attr[p], attr[(p + 1) % 3])}, {"a": domain}) for p in range(3)]


@pytest.mark.parametrize("padded", [False, True])
def test_sec_eval_matches_reference(golden, padded):
    g = golden("engine")
    for tag in g["ev_cases"]:
        count, domain = int(g[f"{tag}_count"]), int(g[f"{tag}_domain"])
        groups = make_groups(g, tag, count, domain, with_ids=False, padded=padded)
        keys = [(fss.parse_key(g[f"{tag}_key{p}_0"].tobytes()), fss.parse_key(g[f"{tag}_key{p}_1"].tobytes()))
                for p in range(3)]
        rts = local_runtimes(make_session_configs(g[f"{tag}_master"].tobytes()), transcript=True)
        res = run_trio(lambda rt: sec_eval(rt, groups[rt.index - 1], keys[rt.index - 1], "a", domain), rts)
        for p in range(3):
            assert np.array_equal(host(res[p].share_a.words), g[f"{tag}_out{p}_a"]), tag
            assert np.array_equal(host(res[p].share_b.words), g[f"{tag}_out{p}_b"]), tag
            assert rts[p].transcript_digest() == digest(g, f"{tag}_digest{p}"), tag
            assert rts[p].meter.total.logical_bits == int(g[f"{tag}_bits{p}"])
            assert rts[p].meter.total.bytes_sent == int(g[f"{tag}_bytes{p}"])
        assert np.array_equal(rss.reconstruct(res).to_bits(), g[f"{tag}_plain"])


@pytest.mark.parametrize("fold", [True, False])
@pytest.mark.parametrize("padded", [False, True])
def test_trio_sec_eval_matches_reference(golden, fold, padded, monkeypatch):
    """Trio.sec_eval (all three parties at once; an interval's two passes
    folded into one parity pass, or not) returns exactly the reference's
    per-party output shares: party p holds components (p, p + 1) -- every
    recorded case, including intervals on the TMA-staged parity path."""
    from paper_2209_03526_b200.graphs import padded_device_matrix
    from paper_2209_03526_b200.trio import Trio, TrioGroup

    monkeypatch.setattr(Trio, "FOLD_PASSES", fold)
    g = golden("engine")
    for tag in g["ev_cases"]:
        count, domain = int(g[f"{tag}_count"]), int(g[f"{tag}_domain"])
        attr = [padded_device_matrix(g[f"{tag}_attr{c}"]) if padded else dev(g[f"{tag}_attr{c}"]) for c in range(3)]
        ids = [torch.zeros((count, (count + 31) // 32), dtype=torch.int32, device="cuda") for _ in range(3)]
        group = TrioGroup(None, None, count, count, ids, {"a": attr}, {"a": domain})
        keys = [(fss.parse_key(g[f"{tag}_key{p}_0"].tobytes()), fss.parse_key(g[f"{tag}_key{p}_1"].tobytes()))
                for p in range(3)]
        res = Trio(g[f"{tag}_master"].tobytes()).sec_eval(group, keys, "a", domain, {})
        for p in range(3):
            assert np.array_equal(host(res[p]), g[f"{tag}_out{p}_a"]), (tag, p)
            assert np.array_equal(host(res[(p + 1) % 3]), g[f"{tag}_out{p}_b"]), (tag, p)


def test_combine_matches_reference(golden):
    g = golden("engine")
    for tag in g["cb_cases"]:
        n = int(g[f"{tag}_n"])
        comps = g[f"{tag}_comps"]
        per_party = [[], [], []]
        for col in comps:
            d = [DBits(dev(col[c]), n) for c in range(3)]
            for p in range(3):
                per_party[p].append(SharedBitVector(p + 1, d[p], d[(p + 1) % 3]))
        combiner, mode = str(g[f"{tag}_combiner"]), str(g[f"{tag}_mode"])
        rts = local_runtimes(make_session_configs(g[f"{tag}_master"].tobytes()), transcript=True)
        res = run_trio(lambda rt: combine_predicates(rt, per_party[rt.index - 1], combiner, mode), rts)
        for p in range(3):
            assert np.array_equal(host(res[p].share_a.words), g[f"{tag}_out{p}_a"]), tag
            assert np.array_equal(host(res[p].share_b.words), g[f"{tag}_out{p}_b"]), tag
            assert rts[p].transcript_digest() == digest(g, f"{tag}_digest{p}"), tag


def test_fetch_matches_reference(golden):
    g = golden("engine")
    for tag in g["fe_cases"]:
        count, domain = int(g[f"{tag}_count"]), int(g[f"{tag}_domain"])
        unique = bool(g[f"{tag}_unique"])
        groups = make_groups(g, tag, count, domain)
        fl = [DBits(dev(g[f"{tag}_flag{c}"]), count) for c in range(3)]
        flags = [SharedBitVector(p + 1, fl[p], fl[(p + 1) % 3]) for p in range(3)]
        rts = local_runtimes(make_session_configs(g[f"{tag}_master"].tobytes()), transcript=True)

        def worker(rt):
            grp, f = groups[rt.index - 1], flags[rt.index - 1]
            if unique:
                return [sec_fetch_unique(rt, grp, f)], []
            audit = []
            return sec_fetch_multi(rt, grp, f, _OpenLabels(), audit), audit

        res = run_trio(worker, rts)
        for p in range(3):
            recs, audit = res[p]
            assert len(recs) == int(g[f"{tag}_n{p}"]), tag
            for r, rec in enumerate(recs):
                base = f"{tag}_p{p}_r{r}"
                assert np.array_equal(host(rec.vertex_id.share_a.words), g[f"{base}_id_a"]), base
                assert np.array_equal(host(rec.vertex_id.share_b.words), g[f"{base}_id_b"]), base
                assert np.array_equal(host(rec.attrs["a"].share_a.words), g[f"{base}_at_a"]), base
                assert np.array_equal(host(rec.attrs["a"].share_b.words), g[f"{base}_at_b"]), base
            if f"{tag}_audit{p}" in g:
                assert np.array_equal(audit[0][1], g[f"{tag}_audit{p}"])
            assert rts[p].transcript_digest() == digest(g, f"{tag}_digest{p}"), tag
        if unique:
            assert all(not rt.opened for rt in rts)


def test_shuffle_matches_reference(golden):
    g = golden("shuffle")
    for tag in g["cases"]:
        rows, width, rounds = int(g[f"{tag}_rows"]), int(g[f"{tag}_width"]), int(g[f"{tag}_rounds"])
        comps = [dev(g[f"{tag}_in{c}"]) for c in range(3)]
        rts = local_runtimes(make_session_configs(g[f"{tag}_master"].tobytes()), transcript=True)

        def worker(rt):
            out = None
            for _ in range(rounds):
                i = rt.index - 1
                out = sec_shuffle(rt, MatchTable(rt.index, width, comps[i], comps[(i + 1) % 3]))
            return out

        res = run_trio(worker, rts)
        for p in range(3):
            assert np.array_equal(host(res[p].share_a), g[f"{tag}_out{p}_a"]), tag
            assert np.array_equal(host(res[p].share_b), g[f"{tag}_out{p}_b"]), tag
            assert rts[p].transcript_digest() == digest(g, f"{tag}_digest{p}"), tag
            assert rts[p].meter.total.bytes_sent == int(g[f"{tag}_bytes{p}"])


@pytest.mark.parametrize("name", ["campus", "unique-chain", "conj", "rand0", "rand1", "rand2", "c1"])
def test_sec_match_end_to_end_matches_reference(golden, name):
    g = golden("match")
    rec = json.loads(str(g[f"{name}_json"]))
    graph = parse_graph_text(rec["graph"])
    rng = np.random.default_rng(rec["seed"])
    schema, shares = encrypt_graph(graph, rec["k"], rng)
    assert schema.digest().hex() == rec["schema_digest"]
    query = load_query(rec["query"], schema)
    tokens = gen_token(query, schema, rng)
    assert [serialize_token(t).hex() for t in tokens] == rec["tokens"]  # rng-compatible keygen
    dshares = device_trio(shares)
    rts = local_runtimes(make_session_configs(bytes.fromhex(rec["master"])), transcript=True)
    results = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], dshares[rt.index - 1],
                                            EngineConfig(any_mode=rec["mode"])), rts)
    matches, _ = open_results(results[:2], schema)
    assert sorted(list(m) for m in set(matches)) == rec["matches"]
    assert [list(sg) for sg in results[0].subgraphs] == rec["subgraphs"]
    for p, res in enumerate(results):
        for s, recs in enumerate(res.records):
            for ri, r in enumerate(recs):
                base = f"{name}_p{p}_s{s}_r{ri}"
                assert np.array_equal(host(r.vertex_id.share_a.words), g[f"{base}_id_a"]), base
                assert np.array_equal(host(r.vertex_id.share_b.words), g[f"{base}_id_b"]), base
                for a in sorted(r.attrs):
                    assert np.array_equal(host(r.attrs[a].share_a.words), g[f"{base}_{a}_a"]), base
                    assert np.array_equal(host(r.attrs[a].share_b.words), g[f"{base}_{a}_b"]), base
        for j, (_phase, bits) in enumerate(res.opened_flags):
            assert np.array_equal(bits, g[f"{name}_p{p}_open{j}"])
    assert [rt.transcript_digest() for rt in rts] == rec["digests"]
    assert [rt.meter.total.bytes_sent for rt in rts] == rec["bytes"]


@pytest.mark.parametrize("native", [True, False])
def test_c1_config_matches_reference(golden, native):
    """BASELINE configs[0] (C1: 1000 vertices, 3 types, 3-vertex path, k = 2)
    share by share: the golden is the live reference's sec_match on exactly
    the graph, query, seeds and session master bench.py's query_latency leg
    uses; the per-party drop-in path and the trio path (native executor or
    Python schedule) reproduce every record share, opened vector, subgraph,
    transcript digest and byte count."""
    from paper_2209_03526_b200 import workloads
    rec = json.loads(str(golden("match")["c1_json"]))
    assert rec["graph"] == workloads.tiny_graph_text(1)
    assert rec["query"] == workloads.tiny_query(workloads.tiny_graph(1), 1)
    assert (rec["k"], rec["seed"], rec["master"]) == (2, 1, (b"\x5a" * 16).hex())
    if native:
        test_sec_match_end_to_end_matches_reference(golden, "c1")
    test_trio_fast_path_matches_reference(golden, "c1", native)


@pytest.mark.parametrize("name", ["campus", "c1", "rand1", "rand2"])
def test_co_resident_sec_match_matches_reference(golden, name):
    """The drop-in per-party API without transcripts: the three party
    threads meet and run the native trio executor once (engine.
    _meet_and_match).  Record shares, opened vectors and subgraphs equal
    the reference's run; each runtime's zero-share counter, table counter
    and opened values advance exactly as the per-party protocol's, so a
    second sec_match on the same runtimes matches the per-party path too."""
    g = golden("match")
    rec = json.loads(str(g[f"{name}_json"]))
    rng = np.random.default_rng(rec["seed"])
    schema, shares = encrypt_graph(parse_graph_text(rec["graph"]), rec["k"], rng)
    tokens = gen_token(load_query(rec["query"], schema), schema, rng)
    dshares = device_trio(shares)
    cfg = EngineConfig(any_mode=rec["mode"])
    fast = local_runtimes(make_session_configs(bytes.fromhex(rec["master"])))
    slow = local_runtimes(make_session_configs(bytes.fromhex(rec["master"])), transcript=True)
    for rnd in range(2):
        got = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], dshares[rt.index - 1], cfg), fast)
        want = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], dshares[rt.index - 1], cfg), slow)
        for a, b in zip(got, want):
            assert a.subgraphs == b.subgraphs
            assert [len(r) for r in a.records] == [len(r) for r in b.records]
            for ra, rb in zip(a.records, b.records):
                for x, y in zip(ra, rb):
                    assert torch.equal(x.vertex_id.share_a.words, y.vertex_id.share_a.words)
                    assert torch.equal(x.vertex_id.share_b.words, y.vertex_id.share_b.words)
                    for n in x.attrs:
                        assert torch.equal(x.attrs[n].share_a.words, y.attrs[n].share_a.words)
            assert [(p, list(map(int, v))) for p, v in a.opened_flags] == \
                [(p, list(map(int, v))) for p, v in b.opened_flags]
        for f, s in zip(fast, slow):
            assert (f.zs.counter, f._table_counter) == (s.zs.counter, s._table_counter)
            assert [(lab, v.to_bits().tolist()) for lab, v in f.opened] == \
                [(lab, (v if isinstance(v, BitVector) else BitVector(v.words, v.logical_len)).to_bits().tolist())
                 for lab, v in s.opened]
        if rnd == 0:
            assert sorted(list(m) for m in set(open_results(got[:2], schema)[0])) == rec["matches"]
            for p, r in enumerate(got):
                for j, (_phase, bits) in enumerate(r.opened_flags):
                    assert np.array_equal(bits, g[f"{name}_p{p}_open{j}"])


def test_open_label_guard_and_and_gate():
    from paper_2209_03526_b200.errors import ProtocolError
    rng = np.random.default_rng(9)
    x = BitVector.from_bits([0, 1, 1, 0])
    sx = rss.share(x, rng)
    out = run_trio(lambda rt: rss.open_shared(rt, sx[rt.index - 1], label=5),
                   local_runtimes(make_session_configs(b"\x01" * 16)))
    assert all(o.to_host() == x for o in out)
    with pytest.raises(ProtocolError, match="label"):
        run_trio(lambda rt: rss.open_shared(rt, sx[rt.index - 1], label=rt.index),
                 local_runtimes(make_session_configs(b"\x01" * 16)))
    a, b = BitVector.random(1000, rng), BitVector.random(1000, rng)
    sa, sb = rss.share(a, rng), rss.share(b, rng)
    z = run_trio(lambda rt: rss.and_gate(rt, sa[rt.index - 1], sb[rt.index - 1]),
                 local_runtimes(make_session_configs(b"\x02" * 16)))
    assert rss.reconstruct(z) == (a & b)


@pytest.mark.parametrize("words,rows", [(11, 70), (64, 1000), (100, 333), (5691, 2048), (313, 2013), (129, 4097),
                                        (1024, 77), (1025, 100)])
@pytest.mark.parametrize("npass", [1, 2])
def test_masked_parity_kernels_vs_oracle(words, rows, npass):
    """Every kernel path (unaligned G-lane; aligned TMA-staged rows up to 1024
    words, with ragged stages and any warp-column count; aligned
    register-indicator beyond) for per-party and trio launches against the
    oracle's src/engine.py:76-80."""
    import oracle
    from paper_2209_03526_b200 import _lib
    from paper_2209_03526_b200.graphs import padded_device_matrix
    rng = np.random.default_rng(words * 7 + rows + npass)
    comps_h = [rng.integers(0, 1 << 32, (rows, words), dtype=np.uint32) for _ in range(3)]
    inds_h = [[rng.integers(0, 1 << 32, words, dtype=np.uint32) for _ in range(2)] for _ in range(3 * npass)]
    A = _lib.ptr_array
    for padded in (False, True):
        comps = [padded_device_matrix(c) if padded else dev(c) for c in comps_h]
        inds = [[dev(x) for x in pair] for pair in inds_h]
        pitch = comps[0].stride(0)
        # trio: j = pass*3 + party
        outs = [torch.empty(((rows + 31) // 32,), dtype=torch.int32, device="cuda") for _ in range(3 * npass)]
        _lib.call("ogm_masked_parity", rows, words, pitch, 3, A(comps), 3, _lib.int_array([0, 1, 2]),
                  _lib.int_array([1, 2, 0]), npass, A([t for pair in inds for t in pair]), A(outs), _lib.stream_ptr())
        for ps in range(npass):
            for q in range(3):
                j = ps * 3 + q
                want = oracle.masked_parity(comps_h[q], comps_h[(q + 1) % 3], inds_h[j][0], inds_h[j][1])
                got = np.unpackbits(host(outs[j]).view(np.uint8), bitorder="little")[:rows]
                assert np.array_equal(got, want), (words, rows, npass, padded, j)
                # per-party launch of the same party/pass
                o1 = torch.empty_like(outs[j])
                _lib.call("ogm_masked_parity", rows, words, pitch, 2, A([comps[q], comps[(q + 1) % 3]]), 1,
                          _lib.int_array([0]), _lib.int_array([1]), 1, A(inds[j]), A([o1]), _lib.stream_ptr())
                assert torch.equal(o1, outs[j])


@pytest.mark.parametrize("words,rows", [(11, 70), (313, 2013), (5691, 300)])
def test_masked_parity_acc_xors_into_out(words, rows):
    """ogm_masked_parity_acc (every kernel path) XORs the parities into the
    caller's buffer: prefill ^ ogm_masked_parity's output."""
    from paper_2209_03526_b200 import _lib
    from paper_2209_03526_b200.graphs import padded_device_matrix
    rng = np.random.default_rng(words + rows)
    comps = [padded_device_matrix(rng.integers(0, 1 << 32, (rows, words), dtype=np.uint32)) for _ in range(3)]
    inds = [dev(rng.integers(0, 1 << 32, words, dtype=np.uint32)) for _ in range(12)]
    nw = (rows + 31) // 32
    A = _lib.ptr_array
    args = (rows, words, comps[0].stride(0), 3, A(comps), 3, _lib.int_array([0, 1, 2]), _lib.int_array([1, 2, 0]), 2,
            A(inds))
    plain = [torch.empty((nw,), dtype=torch.int32, device="cuda") for _ in range(6)]
    _lib.call("ogm_masked_parity", *args, A(plain), _lib.stream_ptr())
    pre = [dev(rng.integers(0, 1 << 32, nw, dtype=np.uint32)) for _ in range(6)]
    acc = [p.clone() for p in pre]
    _lib.call("ogm_masked_parity_acc", *args, A(acc), _lib.stream_ptr())
    for a, p, q in zip(acc, pre, plain):
        assert torch.equal(a, p ^ q)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_sec_eval_slices_equal_unsharded(world):
    """Per-rank shards (masked parity on the row slice + zero-share slice by
    CTR-block offset), concatenated in rank order, equal the single-GPU
    blinded vectors -- what sharded_sec_eval_trio all-gathers."""
    import oracle
    from paper_2209_03526_b200 import _lib
    from paper_2209_03526_b200.graphs import padded_device_matrix
    from paper_2209_03526_b200.sharding import (ShardPlan, assemble_many, sec_eval_local_packed,
                                                sharded_sec_eval_trio)
    rows, words, counters = 5000, 70, [7, 8]
    rng = np.random.default_rng(world)
    comps_h = [rng.integers(0, 1 << 32, (rows, words), dtype=np.uint32) for _ in range(3)]
    inds_h = [[(rng.integers(0, 1 << 32, words, dtype=np.uint32), rng.integers(0, 1 << 32, words, dtype=np.uint32))
               for _ in range(3)] for _ in range(2)]
    keys = [bytes([9 + i]) * 16 for i in range(3)]
    zk = [(keys[0], keys[2]), (keys[1], keys[0]), (keys[2], keys[1])]
    comps = [padded_device_matrix(c) for c in comps_h]
    inds = [[(dev(a), dev(b)) for a, b in ps] for ps in inds_h]
    plan = ShardPlan(rows, world)
    if world == 1:
        res = sharded_sec_eval_trio(comps, words, plan, 0, inds, zk, counters)
        full = [res[j // 3][j % 3] for j in range(6)]
    else:
        # every rank's packed buffer, then the product's assembly of the all-gather
        packs = []
        for r in range(world):
            lo, hi = plan.bounds(r)
            packs.append(sec_eval_local_packed([c[lo:hi] for c in comps], words, plan, r, inds, zk, counters))
        full = assemble_many(torch.stack(packs), plan)
    for ps in range(2):
        for q in range(3):
            want = oracle.pack_bits(oracle.masked_parity(comps_h[q], comps_h[(q + 1) % 3], *inds_h[ps][q]))
            want = want ^ oracle.zero_share(*zk[q], counters[ps], rows)
            assert np.array_equal(host(full[ps * 3 + q]), want), (world, ps, q)


@pytest.mark.parametrize("world", [1, 3])
def test_folded_sec_eval_equals_two_passes(world):
    """A two-pass predicate folded (fold_indicators + fold=True: one parity
    pass over XORed indicators, both zero shares XORed in) gives the XOR of
    the two passes' re-shared vectors -- what ShardedTrio / Trio combine."""
    from paper_2209_03526_b200.graphs import padded_device_matrix
    from paper_2209_03526_b200.sharding import (ShardPlan, assemble_many, fold_indicators, sec_eval_local_packed,
                                                sharded_sec_eval_trio)
    rows, words, counters = 70_000, 313, [3, 4]
    rng = np.random.default_rng(40 + world)
    comps_h = [rng.integers(0, 1 << 32, (rows, words), dtype=np.uint32) for _ in range(3)]
    inds_h = [[(rng.integers(0, 1 << 32, words, dtype=np.uint32), rng.integers(0, 1 << 32, words, dtype=np.uint32))
               for _ in range(3)] for _ in range(2)]
    keys = [bytes([19 + i]) * 16 for i in range(3)]
    zk = [(keys[0], keys[2]), (keys[1], keys[0]), (keys[2], keys[1])]
    comps = [padded_device_matrix(c) for c in comps_h]
    inds = [[(dev(a), dev(b)) for a, b in ps] for ps in inds_h]
    plan = ShardPlan(rows, world)
    two = sharded_sec_eval_trio(comps, words, ShardPlan(rows, 1), 0, inds, zk, counters)
    folded = fold_indicators(inds)
    if world == 1:
        got = sharded_sec_eval_trio(comps, words, plan, 0, folded, zk, counters, fold=True)[0]
    else:
        packs = [sec_eval_local_packed([c[lo:hi] for c in comps], words, plan, r, folded, zk, counters, fold=True)
                 for r, (lo, hi) in enumerate(plan.bounds(r) for r in range(world))]
        got = assemble_many(torch.stack(packs), plan)
    for q in range(3):
        assert torch.equal(got[q], two[0][q] ^ two[1][q]), q


@pytest.mark.parametrize("rows,width", [(1, 128), (1000, 128), (70_001, 129), (300_000, 45), (50_000, 700)])
@pytest.mark.parametrize("window_bytes,tile_rows", [(None, None), (64 << 10, 100)])
def test_planned_gather_equals_direct(rows, width, window_bytes, tile_rows):
    """Two-pass L2-window planned gather == direct gather, bit for bit, incl.
    ragged last windows, 5-word rows, wide rows and many small windows."""
    from paper_2209_03526_b200.prf import seeded_permutation_device
    from paper_2209_03526_b200.shuffle import GatherPlan, gather
    from paper_2209_03526_b200.bits import words_for
    w = words_for(width)
    g = torch.Generator(device="cuda").manual_seed(rows)
    mk = lambda: torch.randint(-2**31, 2**31 - 1, (rows, w), dtype=torch.int32, device="cuda", generator=g)  # noqa: E731
    m1, m2, m3, r = mk(), mk(), mk(), mk()
    idx = seeded_permutation_device(b"\x05" * 16, b"SHPI", 3, rows)
    want = gather(rows, width, torch.empty_like(m1), inner=idx, m1=m1, m2=m2, m3=m3, r=r)
    plan = GatherPlan(idx, w, window_bytes=window_bytes, tile_rows=tile_rows)
    got = plan.run(torch.empty_like(m1), m1=m1, m2=m2, m3=m3, r=r)
    assert torch.equal(got, want)


def test_shuffle_planned_path_matches_reference(golden, monkeypatch):
    """The golden shuffle cases again with the planned two-pass gathers forced on."""
    from paper_2209_03526_b200 import shuffle as shmod
    monkeypatch.setattr(shmod, "PLAN_MIN_BYTES", 0)
    test_shuffle_matches_reference(golden)


@pytest.mark.parametrize("native", [True, False])
@pytest.mark.parametrize("name", ["campus", "unique-chain", "conj", "rand0", "rand1", "rand2", "c1"])
def test_trio_fast_path_matches_reference(golden, name, native):
    """The single-thread trio path (one launch per step for all three parties)
    reproduces the reference's record shares, opened flags and subgraphs --
    both the native executor (ogm_trio_match) and the Python schedule."""
    from paper_2209_03526_b200.trio import Trio
    g = golden("match")
    rec = json.loads(str(g[f"{name}_json"]))
    graph = parse_graph_text(rec["graph"])
    rng = np.random.default_rng(rec["seed"])
    schema, shares = encrypt_graph(graph, rec["k"], rng)
    query = load_query(rec["query"], schema)
    tokens = gen_token(query, schema, rng)
    dshares = device_trio(shares)
    res = Trio(bytes.fromhex(rec["master"])).match(list(tokens), list(dshares), any_mode=rec["mode"], native=native)
    results = res.party_results()
    for r in results:
        r._trio = None   # open_results' per-record reconstruction, not the batched shortcut
    matches, details = open_results(results[:2], schema)
    assert sorted(list(m) for m in set(matches)) == rec["matches"]
    assert res.open(schema) == (matches, details)  # the batched reconstruction
    assert [list(sg) for sg in res.subgraphs] == rec["subgraphs"]
    for p, r in enumerate(results):
        for s, recs in enumerate(r.records):
            for ri, mr in enumerate(recs):
                base = f"{name}_p{p}_s{s}_r{ri}"
                assert np.array_equal(host(mr.vertex_id.share_a.words), g[f"{base}_id_a"]), base
                assert np.array_equal(host(mr.vertex_id.share_b.words), g[f"{base}_id_b"]), base
                for a in sorted(mr.attrs):
                    assert np.array_equal(host(mr.attrs[a].share_a.words), g[f"{base}_{a}_a"]), base
                    assert np.array_equal(host(mr.attrs[a].share_b.words), g[f"{base}_{a}_b"]), base
        for j, (_phase, bits) in enumerate(r.opened_flags):
            assert np.array_equal(bits, g[f"{name}_p{p}_open{j}"])


@pytest.mark.parametrize("world,rows,width", [(1, 1000, 128), (2, 1000, 129), (3, 7001, 70), (8, 50_000, 128),
                                              (1, 1 << 23, 128), (1, 300_000, 129), (2, (1 << 24) + 96, 128)])
def test_sharded_shuffle_equals_trio_shuffle(world, rows, width):
    """Row-sharded shuffle emulated for `world` ranks on one GPU (ThreadComm:
    one thread per rank, all-to-all at a barrier) equals the single-GPU trio
    shuffle.  Covers the one-rank path (the single-GPU chained / per-step
    planned shuffle) and planned pack/unpack gathers (2 x 2^23 rows)."""
    import paper_2209_03526_b200.sharding as sh
    from paper_2209_03526_b200.bits import words_for
    from paper_2209_03526_b200.sharded_trio import run_emulated
    from paper_2209_03526_b200.trio import Trio
    w = words_for(width)
    g = torch.Generator(device="cuda").manual_seed(rows + world)
    comps = [torch.randint(-2**31, 2**31 - 1, (rows, w), dtype=torch.int32, device="cuda", generator=g)
             for _ in range(3)]
    if width % 32:
        for c in comps:
            c[:, -1] &= (1 << (width % 32)) - 1
    trio = Trio(b"\x66" * 16)
    want = [c[:, :w] for c in trio.shuffle(comps, width, online_blinds=False)]
    seeds = (trio.s12, trio.s23, trio.s31)
    plan = sh.ShardPlan(rows, world, align=1)

    def rank_fn(comm):
        lo, hi = plan.bounds(comm.rank)
        shuf = sh.ShardedTrioShuffle(seeds, 0, rows, width, plan, comm.rank)
        return shuf.online([c[lo:hi].contiguous() for c in comps], comm)

    outs = run_emulated(world, rank_fn)
    for j in range(3):
        assert torch.equal(torch.cat([o[j] for o in outs]), want[j]), j


def _np_pack(rows, flag_bits, fields, width, sets):
    """Plain bit-level packing (src/engine.py:227-233) of components `sets`."""
    acc = np.zeros((rows, width), np.uint8)
    for s in sets:
        cols = []
        if flag_bits is not None:
            fb = np.unpackbits(flag_bits[s].cpu().numpy().view(np.uint8), bitorder="little")[:rows]
            cols.append(fb[:, None])
        for mats, wd in fields:
            m = mats[s].cpu().numpy()
            cols.append(np.unpackbits(np.ascontiguousarray(m).view(np.uint8), axis=1, bitorder="little")[:, :wd])
        acc ^= np.concatenate(cols, axis=1)
    pad = (-width) % 32
    packed = np.packbits(np.pad(acc, ((0, 0), (0, pad))), axis=1, bitorder="little").view(np.int32)
    return torch.from_numpy(packed.copy())


@pytest.mark.parametrize("widths,aligned,flag", [([45, 129], True, True), ([45, 129], False, True),
                                                  ([3001, 70000, 129, 5], True, True),
                                                  ([3001, 70000, 129, 5], False, False),
                                                  ([200000, 8969], True, True), ([31, 1, 64], True, False)])
def test_pack_gather_vs_bit_reference(widths, aligned, flag):
    from paper_2209_03526_b200.trio import PackedRows, Trio, _pitch

    rows = 23
    g = torch.Generator(device="cuda").manual_seed(sum(widths))

    def mat(wd):
        w = words_for(wd)
        pitch = (w + 3) // 4 * 4 if aligned else w
        m = torch.randint(-2**31, 2**31 - 1, (rows, pitch), dtype=torch.int32, device="cuda", generator=g)
        return m[:, :w]

    fields = [([mat(wd) for _ in range(3)], wd) for wd in widths]
    flags = [torch.randint(-2**31, 2**31 - 1, (words_for(rows),), dtype=torch.int32, device="cuda", generator=g)
             for _ in range(3)] if flag else None
    width = (1 if flag else 0) + sum(widths)
    pr = PackedRows(rows, width, flags, fields)
    t = Trio(b"\x02" * 16)
    idx = torch.randperm(rows, device="cuda", generator=g).to(torch.int32)
    r = torch.randint(-2**31, 2**31 - 1, (rows, _pitch(width)), dtype=torch.int32, device="cuda", generator=g)
    w = words_for(width)
    for sets in ((0,), (0, 1), (2,), (0, 1, 2)):
        want = _np_pack(rows, flags, fields, width, sets)
        got = t.pack_gather(pr, sets).cpu()
        assert torch.equal(got[:, :w], want), (sets, widths)
        assert bool((got[:, w:] == 0).all())
        got = t.pack_gather(pr, sets, idx=idx, r=r).cpu()
        assert torch.equal(got[:, :w], want[idx.cpu().long()] ^ r.cpu()[:, :w]), (sets, widths)


@pytest.mark.parametrize("rows,width,pad", [(1, 1, 0), (37, 31, 3), (37, 32, 0), (19, 33, 2), (23, 129, 3),
                                           (5, 391053, 3), (300, 2000, 4)])
def test_prf_rows_vs_oracle(rows, width, pad):
    import oracle
    from paper_2209_03526_b200.shuffle import blind_table

    seed = bytes(range(16, 32))
    w = words_for(width)
    got = blind_table(seed, b"SHTB", 7, rows, width, pitch=w + pad).cpu().numpy().view(np.uint32)
    want = oracle.blind_table(seed, b"SHTB", 7, rows, width)
    assert np.array_equal(got[:, :w], want)
    assert not got[:, w:].any()


@pytest.mark.parametrize("rows,words,window", [(70000, 4, 256 << 10), (50001, 5, 200 << 10), (3000, 4, 1 << 20)])
def test_window_planned_gather_equals_direct(rows, words, window):
    from paper_2209_03526_b200.shuffle import GatherPlan, gather

    g = torch.Generator(device="cuda").manual_seed(rows)
    M = torch.randint(-2**31, 2**31 - 1, (rows, words), dtype=torch.int32, device="cuda", generator=g)
    R = torch.randint(-2**31, 2**31 - 1, (rows, words), dtype=torch.int32, device="cuda", generator=g)
    idx = torch.randperm(rows, device="cuda", generator=g).to(torch.int32)
    want = gather(rows, 32 * words, torch.empty_like(M), inner=idx, m1=M, r=R)
    plan = GatherPlan(idx, words, window_bytes=window)
    assert plan.window == max(1, window // (4 * words))
    got = plan.run(torch.empty_like(M), m1=M, r=R)
    assert torch.equal(got, want)


@pytest.mark.parametrize("rows,words,pitch", [(40001, 5, 8), (30000, 4, 8), (20000, 3, 4)])
def test_planned_gather_pitched_rows(rows, words, pitch):
    """Planned gather over 16-B-pitched tables (padding words ride along)."""
    from paper_2209_03526_b200.shuffle import GatherPlan, gather

    g = torch.Generator(device="cuda").manual_seed(rows + pitch)
    full = lambda: torch.randint(-2**31, 2**31 - 1, (rows, pitch), dtype=torch.int32, device="cuda", generator=g)  # noqa: E731
    M, R = full(), full()
    M[:, words:] = 0
    R[:, words:] = 0
    idx = torch.randperm(rows, device="cuda", generator=g).to(torch.int32)
    want = gather(rows, 32 * words, torch.empty_like(M), inner=idx, m1=M, r=R)
    plan = GatherPlan(idx, pitch, window_bytes=32 << 10, tile_rows=333)
    got = plan.run(torch.empty_like(M), m1=M, r=R)
    assert torch.equal(got[:, :words], want[:, :words])


@pytest.mark.parametrize("rows", [1, 999, 1 << 16, 300_001])
def test_shuffle_online_fused_equals_party_steps(rows):
    """The one-launch online shuffle (ogm_shuffle_online_fused) writes the same
    messages x1, y1, c1 and the same new component R3 as the four
    ShuffleOffline party steps."""
    from paper_2209_03526_b200 import workloads
    from paper_2209_03526_b200.net import make_session_configs
    from paper_2209_03526_b200.shuffle import ShuffleOffline, shuffle_online_fused

    cfg = make_session_configs(b"\x3c" * 16)
    comps = [workloads.device_random_words(rows * 4, 5, 80 + c).reshape(rows, 4) for c in range(3)]
    off = [ShuffleOffline(p + 1, cfg[p].seed_with_next, cfg[p].seed_with_prev, 2, rows, 128, plan=False)
           for p in range(3)]
    e = lambda: torch.empty_like(comps[0])  # noqa: E731
    want = [e() for _ in range(4)]
    off[0].step_x1(comps[0], comps[1], want[0])
    off[1].step_y1(comps[2], want[1])
    off[1].step_c1(want[0], want[2])
    off[2].step_r3(want[1], want[2], want[3])
    got = [e() for _ in range(4)]
    shuffle_online_fused(off, comps[0], comps[1], comps[2], *got)
    r3_only = torch.empty_like(got[3])
    shuffle_online_fused(off, comps[0], comps[1], comps[2], got[0], got[1], None, r3_only)
    assert torch.equal(r3_only, want[3])
    for g_, w_ in zip(got, want):
        assert torch.equal(g_, w_)


def test_c5_planned_shuffle_matches_oracle_at_scale():
    """C5 at 2^23 rows x 128 bits (128 MB tables: the planned two-pass gathers
    with source-order blinds and the L2-window pass): the four party steps'
    new components equal the oracle's numpy restatement of
    src/shuffle.py:80-144 bit for bit."""
    import oracle
    from paper_2209_03526_b200 import workloads
    from paper_2209_03526_b200.net import make_session_configs
    from paper_2209_03526_b200.shuffle import ShuffleOffline

    rows = 1 << 23
    cfg = make_session_configs(b"\x5c" * 16)
    s12, s23, s31 = cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next
    comps = [workloads.device_random_words(rows * 4, 9, 90 + c).reshape(rows, 4) for c in range(3)]
    off = [ShuffleOffline(p + 1, cfg[p].seed_with_next, cfg[p].seed_with_prev, 4, rows, 128) for p in range(3)]
    assert off[0].plan_x1 is not None and off[2].plan_r3 is not None
    e = lambda: torch.empty_like(comps[0])  # noqa: E731
    x1, y1, c1, r3 = e(), e(), e(), e()
    off[0].step_x1(comps[0], comps[1], x1)
    off[1].step_y1(comps[2], y1)
    off[1].step_c1(x1, c1)
    off[2].step_r3(y1, c1, r3)
    host = [c.cpu().numpy().view(np.uint32) for c in comps]
    (o1, o2, o3), (m_x1, m_y1, m_c1, _) = oracle.shuffle_trio(s12, s23, s31, 4, host, 128)
    assert np.array_equal(x1.cpu().numpy().view(np.uint32), m_x1)
    assert np.array_equal(y1.cpu().numpy().view(np.uint32), m_y1)
    assert np.array_equal(c1.cpu().numpy().view(np.uint32), m_c1)
    assert np.array_equal(r3.cpu().numpy().view(np.uint32), o3)
    assert np.array_equal(off[0].out_a.cpu().numpy().view(np.uint32), o1)
    assert np.array_equal(off[0].out_b.cpu().numpy().view(np.uint32), o2)
    # the chained online shuffle (messages handed over in shared memory): same messages, same R3
    from paper_2209_03526_b200.shuffle import shuffle_online_planned
    msgs = [e(), e(), e()]
    r3c = shuffle_online_planned(off, comps[0], comps[1], comps[2], e(), msgs=msgs)
    for got, want in zip(msgs + [r3c], (m_x1, m_y1, m_c1, o3)):
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
    r3n = shuffle_online_planned(off, comps[0], comps[1], comps[2], e())
    assert torch.equal(r3n, r3c)


@pytest.mark.parametrize("rows", [4096, 3 * 4096 + 77, 148 * 4096 + 4095, 1 << 20, (1 << 24) + 3 * 4096 + 5])
def test_chained_online_shuffle_equals_party_steps(rows, monkeypatch):
    """ogm_shuffle_online_planned (each message handed from sender to
    receiver tile by tile in shared memory; ragged last tiles; the dual
    window pass) gives the four per-party planned steps' messages and R3;
    so does the flat hand-over, in the receiving partition's I-row or slot
    order, with partition destinations from the run tables or from gdst."""
    from paper_2209_03526_b200 import shuffle, workloads
    from paper_2209_03526_b200.net import make_session_configs
    from paper_2209_03526_b200.shuffle import ShuffleOffline, shuffle_online_planned

    cfg = make_session_configs(b"\x3a" * 16)
    comps = [workloads.device_random_words(rows * 4, 5, 50 + c).reshape(rows, 4) for c in range(3)]
    off = [ShuffleOffline(p + 1, cfg[p].seed_with_next, cfg[p].seed_with_prev, 2, rows, 128, plan=True)
           for p in range(3)]
    e = lambda: torch.empty_like(comps[0])  # noqa: E731
    want = [e() for _ in range(4)]
    off[0].step_x1(comps[0], comps[1], want[0])
    off[1].step_y1(comps[2], want[1])
    off[1].step_c1(want[0], want[2])
    off[2].step_r3(want[1], want[2], want[3])
    msgs = [e(), e(), e()]
    r3 = shuffle_online_planned(off, comps[0], comps[1], comps[2], e(), msgs=msgs)
    for got, w in zip(msgs + [r3], want):
        assert torch.equal(got, w)
    for order in ("inter", "slot"):
        for runs in (True, False):
            monkeypatch.setattr(shuffle, "FLAT_ORDER", order)
            monkeypatch.setattr(shuffle, "USE_RUN_TABLES", runs)
            assert torch.equal(shuffle_online_planned(off, comps[0], comps[1], comps[2], e()), want[3]), (order, runs)


@pytest.mark.parametrize("rows,window", [(1, 1), (4096, 1 << 20), (3 * 4096 + 77, 1000), (1 << 20, 1 << 16),
                                         (123457, 4099), (5 * 4096, 7)])
def test_plan_run_table_reconstructs_gdst(rows, window):
    """ogm_gather_plan_runs: for every slot s of tile t, off[t][d] + s = gdst[s]
    with d the run holding s (the last run starting at or before it), runs
    ordered by window, start[t][nwin] = the tile's row count (ragged tiles,
    empty runs, one row per window)."""
    from paper_2209_03526_b200.shuffle import GatherPlan

    g = torch.Generator(device="cuda").manual_seed(rows)
    idx = torch.randperm(rows, device="cuda", generator=g).to(torch.int32)
    plan = GatherPlan(idx, 4, window_bytes=window * 16)
    start, off, nwin = plan.runs()
    T, ntiles = plan.tile, -(-rows // plan.tile)
    assert nwin == -(-rows // window)
    st = start.cpu().numpy().view(np.uint16)[:ntiles * ((nwin + 8) & ~7)].reshape(ntiles, -1)
    of = off.cpu().numpy()[:ntiles * ((nwin + 3) & ~3)].reshape(ntiles, -1)
    gd = plan.gdst.cpu().numpy()
    for t in range(ntiles):
        n_t = min(T, rows - t * T)
        assert st[t, nwin] == n_t and st[t, 0] == 0 and np.all(np.diff(st[t, :nwin + 1].astype(np.int64)) >= 0)
        s = np.arange(t * T, t * T + n_t)
        d = np.searchsorted(st[t, :nwin], s - t * T, side="right") - 1
        assert np.array_equal(of[t, d].astype(np.int64) + s, gd[s]), t
        assert np.array_equal(d, gd[s] // window), t


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_fold_and_keep_slices_on_device(world):
    """The device side of the sharded fold and keep: each rank's
    fold of its row slice (flag bits sliced at its first row) XORed over the
    ranks equals the unsharded fold; each rank's device compaction of its
    opened slice, offset by the exclusive scan, gives the global kept rows."""
    from paper_2209_03526_b200 import sharding as sh

    rows, words = 5000, 13
    g = torch.Generator(device="cuda").manual_seed(world)
    mats = [torch.randint(-2**31, 2**31 - 1, (rows, 16), dtype=torch.int32, device="cuda", generator=g)[:, :words]
            for _ in range(3)]
    flags = [torch.randint(-2**31, 2**31 - 1, ((rows + 31) // 32,), dtype=torch.int32, device="cuda", generator=g)
             for _ in range(3)]
    want = sh._fold_local(rows, words, mats, flags)
    plan = sh.ShardPlan(rows, world)
    acc = [torch.zeros_like(w) for w in want]
    kept = []
    bits = np.unpackbits(flags[0].cpu().numpy().view(np.uint8), bitorder="little")[:rows]
    for r in range(world):
        lo, hi = plan.bounds(r)
        part = sh._fold_local(hi - lo, words, [m[lo:hi] for m in mats], [f[lo // 32:] for f in flags])
        acc = [a ^ p_ for a, p_ in zip(acc, part)]
        k = int(bits[lo:hi].sum())
        local = sh._compact(flags[0][lo // 32:], hi - lo, k)
        kept += (local.cpu().numpy() + lo).tolist()
    for a, w_ in zip(acc, want):
        assert torch.equal(a, w_)
    assert kept == np.nonzero(bits)[0].tolist()


def test_run_trio_party_threads_nested_and_errors():
    """run_trio on the long-lived party threads: a run_trio from inside a
    party (the threads are busy) falls back to fresh threads instead of
    deadlocking, a party's failure is re-raised, and the threads serve the
    next call afterwards."""
    from paper_2209_03526_b200 import net

    cfg = net.make_session_configs(b"\x11" * 16)

    def outer(rt):
        inner = net.run_trio(lambda r: r.index * 10, net.local_runtimes(net.make_session_configs(b"\x12" * 16)))
        return rt.index, inner

    res = net.run_trio(outer, net.local_runtimes(cfg))
    assert [r[0] for r in res] == [1, 2, 3] and all(r[1] == [10, 20, 30] for r in res)

    def bad(rt):
        if rt.index == 2:
            raise ValueError("boom")
        return rt.index

    with pytest.raises(ValueError, match="boom"):
        net.run_trio(bad, net.local_runtimes(cfg))
    assert net.run_trio(lambda rt: rt.index, net.local_runtimes(cfg)) == [1, 2, 3]


@pytest.mark.parametrize("n,window,tile", [(1, 1, 1), (100, 7, 16), (5000, 333, 100), (70_001, 4096, 1024),
                                           (1 << 20, 1 << 17, 4096), ((1 << 20) + 77, 1 << 18, 16384),
                                           (123457, 1, 4096)])
def test_gather_plan_matches_stable_sorts(n, window, tile):
    """ogm_gather_plan (per-tile shared-memory sorts + per-window scans, no
    library sort) equals its definition: I rows = the sources stably sorted
    by destination window, slots = each tile's sources stably sorted by
    window, q2 = the I row of idx[i] (numpy stable argsorts)."""
    from paper_2209_03526_b200.shuffle import GatherPlan

    g = torch.Generator(device="cuda").manual_seed(n + window)
    idx = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
    plan = GatherPlan(idx, 4, window_bytes=window * 16, tile_rows=tile)
    ih = idx.cpu().numpy().astype(np.int64)
    inv = np.empty(n, np.int64)
    inv[ih] = np.arange(n)
    d = inv // window
    order = np.argsort(d, kind="stable")            # sources in I order
    P = np.empty(n, np.int64)
    P[order] = np.arange(n)
    t = np.arange(n) // tile
    slots = np.lexsort((np.arange(n), d, t))       # by tile, then window, then source
    assert np.array_equal(plan.q2.cpu().numpy(), P[ih])
    assert np.array_equal(plan.gdst.cpu().numpy(), P[slots])
    assert np.array_equal(plan.srow.cpu().numpy().view(np.uint16).astype(np.int64), slots % tile)
