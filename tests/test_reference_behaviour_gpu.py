"""The reference's behavioural tests, re-run against the B200 package.

Mirrors /root/reference/pkg/tests/test_rss.py, test_shuffle.py,
test_fss.py and test_engine.py (cited per test) so the drop-in's semantics,
error types and messages are checked the way the reference checks its own.
Randomness is drawn the same way, but outputs are compared against
brute-force / plaintext truths as the reference does (no reference import:
this runs on the GPU box).
"""

import numpy as np
import torch
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2209_03526_b200 import fss, rss
from paper_2209_03526_b200.bits import BitVector
from paper_2209_03526_b200.engine import EngineConfig, open_results, sec_match
from paper_2209_03526_b200.errors import ProtocolError
from paper_2209_03526_b200.graphs import device_trio, encrypt_graph, parse_graph_text
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_local_trio, run_trio
from paper_2209_03526_b200.query import gen_token, load_query
from paper_2209_03526_b200.shuffle import MatchTable, composed_permutation, sec_shuffle, simulate_shuffle

pytestmark = pytest.mark.gpu


def bv(bits):
    return BitVector.from_bits(bits)


# ---------------------------------------------------------------- rss (tests/test_rss.py)


def test_share_reconstruct_small_exhaustive():
    """tests/test_rss.py:21-33 (first part)."""
    rng = np.random.default_rng(0)
    for n in range(1, 7):
        for value in range(1 << n):
            x = BitVector.from_int(value, n)
            assert rss.reconstruct(rss.share(x, rng)) == x


def test_reconstruct_pairs_and_errors():
    """tests/test_rss.py:36-78."""
    rng = np.random.default_rng(7)
    x = BitVector.random(257, rng)
    sh = rss.share(x, rng)
    for pair in ((0, 1), (1, 2), (0, 2)):
        assert rss.reconstruct([sh[pair[0]], sh[pair[1]]]) == x
    with pytest.raises(ValueError, match="cover"):
        rss.reconstruct([sh[0]])
    other = rss.share(bv([1, 0]), rng)
    with pytest.raises(ValueError, match="length"):
        rss.reconstruct([rss.share(bv([1, 0, 1]), rng)[0], other[1]])
    s1, s2, s3 = rss.share(bv([1, 0, 1, 1]), rng)
    bad = rss.SharedBitVector(2, s2.share_a ^ rss.DBits.from_host(bv([1, 0, 0, 0])), s2.share_b)
    with pytest.raises(ValueError, match="inconsistent"):
        rss.reconstruct([s1, bad, s3])
    with pytest.raises(ValueError):
        rss.share(BitVector.zeros(0), rng)


def test_xor_local_and_public():
    """tests/test_rss.py:81-108, :145-150."""
    rng = np.random.default_rng(4)
    x, y, c = (BitVector.random(130, rng) for _ in range(3))
    sx, sy = rss.share(x, rng), rss.share(y, rng)
    assert rss.reconstruct([a.xor(b) for a, b in zip(sx, sy)]) == (x ^ y)
    assert rss.reconstruct([s.xor_public(c) for s in sx]) == (x ^ c)
    with pytest.raises(ValueError, match="different parties"):
        sx[0].xor(sx[1])


def test_and_gate_truth_and_accounting():
    """tests/test_rss.py:111-124."""
    rng = np.random.default_rng(6)
    for xb, yb, want in (([0], [1], [0]), ([1], [1], [1]), ([1, 0, 1, 1], [1, 1, 0, 1], [1, 0, 0, 1])):
        sx, sy = rss.share(bv(xb), rng), rss.share(bv(yb), rng)
        out = run_local_trio(lambda rt: rss.and_gate(rt, sx[rt.index - 1], sy[rt.index - 1]))
        assert rss.reconstruct(out) == bv(want)
    x, y = BitVector.random(64, rng), BitVector.random(64, rng)
    sx, sy = rss.share(x, rng), rss.share(y, rng)
    out = run_local_trio(lambda rt: (rss.and_gate(rt, sx[rt.index - 1], sy[rt.index - 1]),
                                     rt.meter.total.logical_bits))
    assert rss.reconstruct([o[0] for o in out]) == (x & y)
    assert all(o[1] == 64 for o in out)


def test_zero_shares_cancel_and_count():
    """tests/test_rss.py:153-175."""
    keys = [bytes([i + 1]) * 16 for i in range(3)]
    ctxs = [rss.ZeroShareContext(keys[0], keys[2]), rss.ZeroShareContext(keys[1], keys[0]),
            rss.ZeroShareContext(keys[2], keys[1])]
    for _ in range(20):
        outs = [c.next_share(77).to_host() for c in ctxs]
        assert (outs[0] ^ outs[1] ^ outs[2]).is_zero()
    assert all(c.counter == 20 for c in ctxs)
    a = ctxs[0].peek(256, 7).to_host()
    assert ctxs[0].peek(256, 7).to_host() == a and ctxs[0].peek(256, 8).to_host() != a


# ---------------------------------------------------------------- shuffle (tests/test_shuffle.py)


def run_shuffle(plain_rows, master=b"\x07" * 16, rounds=1, transcript=False):
    rng = np.random.default_rng(1234)
    shares = [rss.share(r, rng) for r in plain_rows]
    configs = make_session_configs(master)

    def worker(rt):
        out = None
        for _ in range(rounds):
            out = sec_shuffle(rt, MatchTable.from_rows([shares[i][rt.index - 1] for i in range(len(plain_rows))]))
        return out

    rts = local_runtimes(configs, transcript=transcript)
    outs = run_trio(worker, rts)
    rebuilt = [rss.reconstruct([outs[0].row(i), outs[1].row(i), outs[2].row(i)]) for i in range(len(plain_rows))]
    return rebuilt, outs, configs, rts


def test_single_row_and_multiset_vs_simulator():
    """tests/test_shuffle.py:33-48."""
    row = bv([1, 0, 1, 1, 0])
    assert run_shuffle([row])[0] == [row]
    rng = np.random.default_rng(5)
    for n in (2, 3, 8, 17, 32):
        rows = [BitVector.random(45, rng) for _ in range(n)]
        rebuilt, _, cfg, _ = run_shuffle(rows)
        want = simulate_shuffle(cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next, 0, rows)
        assert rebuilt == want
        assert sorted(r.words.tobytes() for r in rebuilt) == sorted(r.words.tobytes() for r in rows)


def test_output_is_valid_replicated_sharing():
    """tests/test_shuffle.py:51-61."""
    rng = np.random.default_rng(6)
    rows = [BitVector.random(70, rng) for _ in range(9)]
    _, outs, _, _ = run_shuffle(rows)
    for i in range(9):
        for p in range(3):
            assert np.array_equal(outs[p].share_b[i].cpu().numpy(), outs[(p + 1) % 3].share_a[i].cpu().numpy())
            assert not (outs[p].row(i).share_a.to_host().words[-1] >> 6)  # clean 70-bit tail


def test_seeds_and_table_ids_change_order():
    """tests/test_shuffle.py:64-82."""
    rows = [BitVector.from_int(i + 1, 32) for i in range(8)]
    first = run_shuffle(rows, master=b"\x01" * 16)[0]
    second = run_shuffle(rows, master=b"\x02" * 16)[0]
    assert sorted(r.to_int() for r in first) == sorted(r.to_int() for r in second)
    assert [r.to_int() for r in first] != [r.to_int() for r in second]
    rows16 = [BitVector.from_int(i + 1, 16) for i in range(8)]
    once, _, cfg, _ = run_shuffle(rows16, rounds=1)
    twice = run_shuffle(rows16, rounds=2)[0]
    s = (cfg[0].seed_with_next, cfg[1].seed_with_next, cfg[2].seed_with_next)
    assert [r.to_int() for r in once] == [rows16[i].to_int() for i in composed_permutation(*s, 0, 8)]
    assert [r.to_int() for r in twice] == [rows16[i].to_int() for i in composed_permutation(*s, 1, 8)]


def test_single_party_obliviousness_structure():
    """tests/test_shuffle.py:85-117: party 1's transcript does not depend on s23."""
    base = make_session_configs(b"\x21" * 16)
    variant = make_session_configs(b"\x21" * 16)
    variant[1].seed_with_next = b"\xee" * 16
    variant[2].seed_with_prev = b"\xee" * 16

    def transcripts(configs):
        rng = np.random.default_rng(99)
        rows = [BitVector.random(33, rng) for _ in range(12)]
        rts = local_runtimes(configs, transcript=True)

        def worker(rt):
            table = MatchTable.from_rows([rss.share(r, np.random.default_rng(50 + i))[rt.index - 1]
                                          for i, r in enumerate(rows)])
            sec_shuffle(rt, table)
            return rt.transcript_digest()

        return run_trio(worker, rts)

    tb, tv = transcripts(base), transcripts(variant)
    assert tb[0] == tv[0] and tb[1] != tv[1] and tb[2] != tv[2]


def test_table_width_mismatch():
    """tests/test_shuffle.py:120-125."""
    rng = np.random.default_rng(3)
    rows = [rss.share(BitVector.random(16, rng), rng)[0], rss.share(BitVector.random(24, rng), rng)[0]]
    with pytest.raises(ValueError, match="width"):
        MatchTable.from_rows(rows)


# ---------------------------------------------------------------- fss (tests/test_fss.py)


def indicator(pair, n):
    return (fss.full_domain_eval(pair[0], n) ^ fss.full_domain_eval(pair[1], n)).to_bits()


def brute(kind, ops, n):
    xs = np.arange(n)
    return {"eq": xs == ops[0], "lt": xs < ops[0], "le": xs <= ops[0], "gt": xs > ops[0],
            "ge": xs >= ops[0]}.get(kind, (xs >= ops[0]) & (xs <= ops[-1])).astype(np.uint8)


@given(st.integers(2, 512), st.data())
@settings(max_examples=25, deadline=None)
def test_comparison_variants_random(n, data):
    """tests/test_fss.py:75-82."""
    alpha = data.draw(st.integers(0, n - 1))
    kind = data.draw(st.sampled_from(["lt", "le", "gt", "ge"]))
    rng = np.random.default_rng(data.draw(st.integers(0, 2**32 - 1)))
    assert indicator(fss.cmp_gen(kind, alpha, n, rng), n).tolist() == brute(kind, (alpha,), n).tolist()


@given(st.integers(2, 300), st.data())
@settings(max_examples=25, deadline=None)
def test_interval_random(n, data):
    """tests/test_fss.py:85-92."""
    lo = data.draw(st.integers(0, n - 1))
    hi = data.draw(st.integers(lo, n - 1))
    rng = np.random.default_rng(data.draw(st.integers(0, 2**32 - 1)))
    assert indicator(fss.ic_gen(lo, hi, n, rng), n).tolist() == brute("iv", (lo, hi), n).tolist()


def test_interval_spec_and_open_variants():
    """tests/test_fss.py:95-113."""
    rng = np.random.default_rng(5)
    assert indicator(fss.ic_gen(0, 127, 128, rng), 128).tolist() == [1] * 128
    assert indicator(fss.ic_gen(5, 5, 64, rng), 64).tolist() == indicator(fss.dpf_gen(5, 64, rng), 64).tolist()
    xs = np.arange(32)
    for cl, ch in ((True, True), (True, False), (False, True), (False, False)):
        pair = fss.ic_gen(7, 13, 32, rng, closed_low=cl, closed_high=ch)
        want = ((xs >= 7) if cl else (xs > 7)) & ((xs <= 13) if ch else (xs < 13))
        assert indicator(pair, 32).tolist() == want.astype(int).tolist()
    with pytest.raises(fss.DomainError):
        fss.ic_gen(9, 3, 16, rng)


def test_key_sizes_equal_and_serde_errors():
    """tests/test_fss.py:138-164."""
    rng = np.random.default_rng(10)
    for n in (2, 64, 1000):
        sizes = {len(fss.serialize_key(fss.dpf_gen(0, n, rng)[0])),
                 len(fss.serialize_key(fss.cmp_gen("lt", 0, n, rng)[0])),
                 len(fss.serialize_key(fss.cmp_gen("ge", n - 1, n, rng)[1]))}
        assert len(sizes) == 1
    with pytest.raises(ValueError):
        fss.parse_key(fss.serialize_key(fss.dpf_gen(1, 4, rng)[0])[:-3])
    with pytest.raises(ValueError):
        fss.parse_key(b"")


# ---------------------------------------------------------------- engine (tests/test_engine.py)

CAMPUS = """V U u1 place=Harbin
V U u2 place=Beijing
V P p1 age=35
V P p2 age=31
V P p3 age=40
V P p4 age=52
V C c1 field=software
V C c2 field=Internet
E u1 p1
E u1 p2
E u1 p3
E u2 p4
E p1 c1
E p2 c1
E p3 c2
E p4 c2
E p1 p2
"""


def run_query(text, qtext, k=2, seed=1, master=b"\x11" * 16, mode="or"):
    graph = parse_graph_text(text)
    rng = np.random.default_rng(seed)
    schema, shares = encrypt_graph(graph, k, rng)
    tokens = gen_token(load_query(qtext, schema), schema, rng)
    d = device_trio(shares)
    rts = local_runtimes(make_session_configs(master))
    # co_resident=False: the per-party protocol threads (the trio paths are compared against it)
    res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1],
                                        EngineConfig(any_mode=mode, co_resident=False)), rts)
    return set(open_results(res[:2], schema)[0]), rts, res, schema, tokens


def test_unsatisfiable_root_and_conjunction():
    """tests/test_engine.py:373-383."""
    assert run_query(CAMPUS, "Q u U place = Beijing\nQ p P age > 100\nQE u p\n")[0] == set()
    got = run_query(CAMPUS, "Q u U place = Harbin\nQ p P age >= 35\nQ p P age <= 40\nQE u p\n")[0]
    assert got == {("u1", "p1"), ("u1", "p3")}


def test_all_dummy_posting_list_and_access_counts():
    """tests/test_engine.py:270-308."""
    text = "V P p1 a=1\nV P p2 a=2\nV C c1 z=10\nV C c2 z=20\nE p2 c1\nE p2 c2\n"
    assert run_query(text, "Q root P a = 1\nQ leaf C z >= 10\nQE root leaf\n")[0] == set()
    text = "V P p1 a=1\nV P p2 a=2\nV C c1 z=10\nV C c2 z=20\nV C c3 z=30\nE p1 c1\nE p1 c2\nE p1 c3\nE p2 c2\n"
    got, rts, _, _, _ = run_query(text, "Q root P a = 1\nQ leaf C z >= 10\nQE root leaf\n")
    assert got == {("p1", "c1"), ("p1", "c2"), ("p1", "c3")}
    assert sorted(int(v.popcount()) for _, v in rts[0].opened)[-1] == 3


def test_any_modes_and_unique_route():
    """tests/test_engine.py:320-356."""
    text = "V P p1 a=1 b=1\nV P p2 a=1 b=5\nV P p3 a=3 b=1\nV P p4 a=3 b=5\nE p1 p2\nE p3 p4\n"
    q = "Q root P a = 1\nQ root P b = 1\nQC root ANY\n"
    assert ("p1",) in run_query(text, q, mode="or")[0]
    assert ("p1",) not in run_query(text, q, mode="xor")[0]
    rep = "V P p1 a=1\nV P p2 a=1\nV P p3 a=2\nV P p4 a=2\nE p1 p2\nE p3 p4\n"
    got, rts, _, _, _ = run_query(rep, "Q root P a = 1\n")
    assert got == {("p1",), ("p2",)} and all(len(rt.opened) == 1 for rt in rts)
    got, rts, _, _, _ = run_query(CAMPUS, "Q root P age = 35\n")
    assert got == {("p1",)} and all(not rt.opened for rt in rts)


def test_results_consistent_across_party_pairs_and_schema_guard():
    """tests/test_engine.py:455-478."""
    got, _, res, schema, tokens = run_query(CAMPUS, "Q a P age = 35\n")
    for pair in ((0, 1), (1, 2), (0, 2)):
        assert set(open_results([res[pair[0]], res[pair[1]]], schema)[0]) == got
    other = encrypt_graph(parse_graph_text(CAMPUS + "V U u3 place=Xian\nV C c3 field=retail\nV P p5 age=29\n"
                                           "E u3 p5\nE p5 c3\n"), 3, np.random.default_rng(2))[1]
    d = device_trio(other)
    rts = local_runtimes(make_session_configs(b"\x40" * 16))
    with pytest.raises(ValueError, match="different schemas"):
        run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1], EngineConfig()), rts)


def test_open_label_guard():
    """tests/test_rss.py:127-142."""
    rng = np.random.default_rng(9)
    sx = rss.share(bv([0, 1, 1, 0]), rng)
    with pytest.raises(ProtocolError, match="label"):
        run_local_trio(lambda rt: rss.open_shared(rt, sx[rt.index - 1], label=rt.index))


@pytest.mark.parametrize("text,qtext,mode", [
    (CAMPUS, "Q u U place = Beijing\nQ p P age > 100\nQE u p\n", "or"),
    (CAMPUS, "Q u U place = Harbin\nQ p P age >= 35\nQ p P age <= 40\nQE u p\n", "or"),
    ("V P p1 a=1\nV P p2 a=2\nV C c1 z=10\nV C c2 z=20\nE p2 c1\nE p2 c2\n",
     "Q root P a = 1\nQ leaf C z >= 10\nQE root leaf\n", "or"),
    ("V P p1 a=1\nV P p2 a=2\nV C c1 z=10\nV C c2 z=20\nV C c3 z=30\nE p1 c1\nE p1 c2\nE p1 c3\nE p2 c2\n",
     "Q root P a = 1\nQ leaf C z >= 10\nQE root leaf\n", "or"),
    ("V P p1 a=1 b=1\nV P p2 a=1 b=5\nV P p3 a=3 b=1\nV P p4 a=3 b=5\nE p1 p2\nE p3 p4\n",
     "Q root P a = 1\nQ root P b = 1\nQC root ANY\n", "or"),
    ("V P p1 a=1 b=1\nV P p2 a=1 b=5\nV P p3 a=3 b=1\nV P p4 a=3 b=5\nE p1 p2\nE p3 p4\n",
     "Q root P a = 1\nQ root P b = 1\nQC root ANY\n", "xor"),
    ("V P p1 a=1\nV P p2 a=1\nV P p3 a=2\nV P p4 a=2\nE p1 p2\nE p3 p4\n", "Q root P a = 1\n", "or"),
    (CAMPUS, "Q root P age = 35\n", "or"),
])
def test_trio_path_equals_per_party_on_edge_cases(text, qtext, mode):
    """The same edge cases (empty root, all-dummy posting lists, ANY modes,
    unique route) through the trio fast path: identical matches, identical
    record shares, and identical opened vectors with identical labels."""
    from paper_2209_03526_b200.trio import Trio

    got, rts, res, schema, tokens = run_query(text, qtext, mode=mode)
    graph = parse_graph_text(text)
    rng = np.random.default_rng(1)
    schema2, shares = encrypt_graph(graph, 2, rng)
    tokens2 = gen_token(load_query(qtext, schema2), schema2, rng)
    tr = Trio(b"\x11" * 16)
    tres = tr.match(list(tokens2), list(device_trio(shares)), any_mode=mode)
    views = tres.party_results()
    assert set(open_results(views[:2], schema2)[0]) == got
    assert tres.open(schema2) == open_results(views[:2], schema2)
    assert [(lbl, v.to_bits().tolist()) for lbl, v in tr.opened] == \
        [(lbl, v.to_bits().tolist()) for lbl, v in rts[0].opened]
    for q in range(3):
        for s_, (a_recs, b_recs) in enumerate(zip(res[q].records, views[q].records)):
            assert len(a_recs) == len(b_recs), s_
            for ra, rb in zip(a_recs, b_recs):
                assert np.array_equal(np.asarray(ra.vertex_id.share_a.to_bits()), np.asarray(rb.vertex_id.share_a.to_bits()))


def _random_graph_text(rng):
    n = int(rng.integers(60, 161))
    types = "ABC"[: int(rng.integers(2, 4))]
    doms = {(t, a): int(rng.integers(8, 65)) for t in types for a in ("a0", "a1")}
    lines, vt = [], []
    for i in range(n):
        t = types[int(rng.integers(0, len(types)))]
        vt.append(t)
        lines.append(f"V {t} v{i} a0={int(rng.integers(0, doms[(t, 'a0')]))} a1={int(rng.integers(0, doms[(t, 'a1')]))}")
    seen = set()
    for _ in range(2 * n):
        a, b = int(rng.integers(0, n)), int(rng.integers(0, n))
        if a == b or (a, b) in seen or (b, a) in seen:
            continue
        seen.add((a, b))
        lines.append(f"E v{a} v{b}")
    return "\n".join(lines) + "\n"


def _random_query_text(rng, schema):
    types = sorted(schema.types)
    m = int(rng.integers(2, 5))
    qv = [types[int(rng.integers(0, len(types)))]]
    edges = []
    for i in range(1, m):
        p = int(rng.integers(0, i))
        opts = sorted(schema.types[qv[p]].posting_types)
        if not opts:
            break
        qv.append(opts[int(rng.integers(0, len(opts)))])
        edges.append((p, i))
    lines = []
    for i, t in enumerate(qv):
        for _ in range(int(rng.integers(1, 3))):
            a = ("a0", "a1")[int(rng.integers(0, 2))]
            vals = sorted(schema.types[t].attrs[a].values, key=float)
            op = ("=", "<", "<=", ">", ">=", "in")[int(rng.integers(0, 6))]
            if op == "in":
                lo, hi = sorted(int(rng.integers(0, len(vals))) for _ in range(2))
                lines.append(f"Q q{i} {t} {a} in {vals[lo]} {vals[hi]}")
            else:
                lines.append(f"Q q{i} {t} {a} {op} {vals[int(rng.integers(0, len(vals)))]}")
    lines += [f"QE q{p} q{c}" for p, c in edges]
    return "\n".join(lines) + "\n"


def test_random_corpus_equals_oracle_both_paths():
    """Acceptance criterion 1 of the reference (tests/test_acceptance.py:26-55)
    restated on our own seeded random graphs/queries: 30 graph/query pairs,
    the per-party drop-in path and the trio fast path both return exactly the
    plaintext matcher's subgraphs, and the same opened vectors."""
    import oracle.matcher as om
    from paper_2209_03526_b200.trio import Trio

    nonempty = 0
    for trial in range(30):
        rng = np.random.default_rng(5000 + trial)
        text = _random_graph_text(rng)
        graph = parse_graph_text(text)
        schema, shares = encrypt_graph(graph, 2, np.random.default_rng(trial))
        qtext = _random_query_text(rng, schema)
        query = load_query(qtext, schema)
        tokens = gen_token(query, schema, np.random.default_rng(100 + trial))
        want = om.oracle_match(graph, query, schema)
        d = device_trio(shares)
        master = bytes([trial]) * 16
        rts = local_runtimes(make_session_configs(master))
        res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], d[rt.index - 1],
                                            EngineConfig(co_resident=False)), rts)
        assert set(open_results(res[:2], schema)[0]) == want, (trial, qtext)
        tr = Trio(master)
        tres = tr.match(list(tokens), list(d))
        opened = open_results(tres.party_results()[:2], schema)
        assert set(opened[0]) == want, (trial, qtext)
        assert tres.open(schema) == opened, (trial, qtext)
        assert [v.to_bits().tolist() for _, v in tr.opened] == [v.to_bits().tolist() for _, v in rts[0].opened]
        nonempty += bool(want)
    assert nonempty >= 5


def test_fss_exhaustive_600_checks():
    """Acceptance criterion 3 (tests/test_acceptance.py:83-113): 100 random
    parameter sets x {DPF, <, <=, >, >=, interval}, domains 2..4096, each key
    pair's full-domain XOR equal to the brute-force indicator."""
    rng = np.random.default_rng(7)
    checked = 0
    for _ in range(100):
        n = int(rng.integers(2, 4097))
        alpha = int(rng.integers(0, n))
        assert indicator(fss.dpf_gen(alpha, n, rng), n).tolist() == brute("eq", (alpha,), n).tolist()
        checked += 1
        for kind in ("lt", "le", "gt", "ge"):
            a = int(rng.integers(0, n))
            assert indicator(fss.cmp_gen(kind, a, n, rng), n).tolist() == brute(kind, (a,), n).tolist()
            checked += 1
        lo = int(rng.integers(0, n))
        hi = int(rng.integers(lo, n))
        assert indicator(fss.ic_gen(lo, hi, n, rng), n).tolist() == brute("iv", (lo, hi), n).tolist()
        checked += 1
    assert checked == 600


def test_shuffle_exhaustive_sizes_both_paths():
    """Acceptance criterion 5 (tests/test_acceptance.py:153-195): table sizes
    1..64, the reconstructed order equals the seeded composed permutation and
    the multiset is preserved -- through the per-party sec_shuffle and the
    trio shuffle (one ogm_trio_shuffle call), which must agree share for share."""
    from paper_2209_03526_b200.trio import Trio

    rng = np.random.default_rng(12)
    master = b"\x55" * 16
    configs = make_session_configs(master)
    s12, s23, s31 = (configs[0].seed_with_next, configs[1].seed_with_next, configs[2].seed_with_next)
    for size in range(1, 65):
        rows = [BitVector.random(40, rng) for _ in range(size)]
        shares = [rss.share(r, rng) for r in rows]
        outs = run_trio(lambda rt: sec_shuffle(rt, MatchTable.from_rows([shares[i][rt.index - 1] for i in range(size)])),
                        local_runtimes(make_session_configs(master)))
        got = [rss.reconstruct([outs[0].row(i), outs[1].row(i), outs[2].row(i)]) for i in range(size)]
        perm = composed_permutation(s12, s23, s31, 0, size)
        assert got == [rows[int(i)] for i in perm], size
        # the trio path: components x_j = party j's share_a
        comps = [torch.stack([torch.as_tensor(shares[i][c].share_a.words).cuda() for i in range(size)]) for c in range(3)]
        tr = Trio(master)
        new = tr.shuffle(comps, 40)
        for c in range(3):
            want_c = outs[c].share_a.cpu().numpy().view(np.uint32)
            assert np.array_equal(new[c][:, : want_c.shape[1]].cpu().numpy().view(np.uint32), want_c), (size, c)
