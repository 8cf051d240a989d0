"""Host-side data preparation either side of the hot path: graph ingest,
schema/dictionaries, k-padding and share generation restated from
src/graphs.py must give byte-identical schemas and shares for the same rng."""

import json

import numpy as np

from paper_2209_03526_b200.graphs import build_schema, encrypt_graph, parse_graph_text


def test_schema_digests_match_recorded_reference(golden):
    g = golden("match")
    for name in g["names"]:
        rec = json.loads(str(g[f"{name}_json"]))
        graph = parse_graph_text(rec["graph"])
        schema, _ = encrypt_graph(graph, rec["k"], np.random.default_rng(rec["seed"]))
        assert schema.digest().hex() == rec["schema_digest"], name


def test_encrypt_graph_shares_match_live_reference(reference, golden):
    from oblivgm.graphs import encrypt_graph as ref_encrypt
    from oblivgm.graphs import parse_graph_text as ref_parse

    g = golden("match")
    for name in g["names"]:
        rec = json.loads(str(g[f"{name}_json"]))
        _, mine = encrypt_graph(parse_graph_text(rec["graph"]), rec["k"], np.random.default_rng(rec["seed"]))
        _, theirs = ref_encrypt(ref_parse(rec["graph"]), rec["k"], np.random.default_rng(rec["seed"]))
        for a, b in zip(mine, theirs):
            for t in a.types:
                assert np.array_equal(a.types[t].id_a, b.types[t].id_a)
                assert np.array_equal(a.types[t].id_b, b.types[t].id_b)
                for n in a.types[t].attrs:
                    assert np.array_equal(a.types[t].attrs[n][0], b.types[t].attrs[n][0])
                for n in a.types[t].posting:
                    assert np.array_equal(a.types[t].posting[n][1], b.types[t].posting[n][1])


def test_schema_json_round_trip(golden):
    from paper_2209_03526_b200.graphs import GraphSchema
    rec = json.loads(str(golden("match")["campus_json"]))
    schema = build_schema(parse_graph_text(rec["graph"]), 2)
    back = GraphSchema.from_json(schema.to_json())
    assert back.digest() == schema.digest()


def _resolved(q):
    return ([(v.name, v.vtype, v.combiner, [(p.attr, p.kind, tuple(p.operands), tuple(p.closed))
                                            for p in v.predicates]) for v in q.vertices],
            [list(c) for c in q.children], list(q.parent))


def test_query_resolution_matches_live_reference(reference, golden):
    """Random queries over the recorded graphs (the reference's own query
    generator, every operator) and hand-written edge cases resolve to the
    same slots, predicates (kind, index-space operands, closedness) and tree
    as the reference's load_query (src/query.py:88-256)."""
    from oblivgm.datagen import random_query_text
    from oblivgm.graphs import build_schema as ref_schema
    from oblivgm.graphs import parse_graph_text as ref_parse
    from oblivgm.query import load_query as ref_load

    from paper_2209_03526_b200.query import load_query

    g = golden("match")
    for name in g["names"]:
        rec = json.loads(str(g[f"{name}_json"]))
        mine = build_schema(parse_graph_text(rec["graph"]), rec["k"])
        theirs = ref_schema(ref_parse(rec["graph"]), rec["k"])
        rng = np.random.default_rng(5)
        texts = [rec["query"]]
        for _ in range(40 if name.startswith("rand") else 0):   # the generator needs ordinal attributes
            texts.append(random_query_text(rng, theirs, n_targets=int(rng.integers(1, 5)),
                                           kinds=("eq", "lt", "le", "gt", "ge", "iv"), multi_pred_prob=0.5))
        for t in texts:
            assert _resolved(load_query(t, mine)) == _resolved(ref_load(t, theirs)), t


def test_query_errors_match_reference(reference, golden):
    from oblivgm.graphs import build_schema as ref_schema
    from oblivgm.graphs import parse_graph_text as ref_parse
    from oblivgm.query import QueryFormatError as RefError
    from oblivgm.query import load_query as ref_load

    from paper_2209_03526_b200.query import QueryFormatError, load_query

    rec = json.loads(str(golden("match")["campus_json"]))
    mine, theirs = build_schema(parse_graph_text(rec["graph"]), 2), ref_schema(ref_parse(rec["graph"]), 2)
    cases = ["Q a Z age = 5\n", "Q a P size = 5\n", "Q a P age = 33\n", "Q a U place < 5\n",
             "Q a P age = 31\nQ b P age = 31\nQE a b\nQE a b\n", "Q a P age = 31\nQ b P age = 31\n",
             "Q a P age = 31\nQ b C field = software\nQE a b\nQE b a\n",
             "Q a U place = Harbin\nQ b C field = software\nQE a b\n", "", "Q a P age ? 31\n",
             "Q a P age in 31\n", "Q a P age < 31 32\n", "QC a ALL\n", "Q a P age = 31\nQC a SOME\n",
             "Q a P age = 31\nQS b\n", "Q a P age = 31\nQX a\n", "Q a P age = 31\nQ a U place = Harbin\n",
             "# c\n\nQ a P age = 31\nQE a\n", "Q a P\n", "Q a P age < x\n"]
    for text in cases:
        try:
            ref_load(text, theirs)
            want = None
        except RefError as exc:
            want = str(exc)
        except ValueError as exc:   # float() of a bad interval operand
            want = ("ValueError", type(exc).__name__)
        try:
            load_query(text, mine)
            got = None
        except QueryFormatError as exc:
            got = str(exc)
        except ValueError as exc:
            got = ("ValueError", type(exc).__name__)
        assert got == want, text


def test_graph_parse_errors_match_reference(reference):
    from oblivgm.graphs import GraphFormatError as RefError
    from oblivgm.graphs import parse_graph_text as ref_parse

    from paper_2209_03526_b200.graphs import GraphFormatError

    cases = ["V P p1", "V P p1 age", "V P p1 age=5\nV P p1 age=6", "V P p1 age=5\nE p1 p9",
             "V P p1 age=5\nE p1 p1", "V P p1 age=5\nV P p2 age=6\nE p1 p2\nE p2 p1", "X P p1",
             "V P p1 age=5\nV P p2 size=6", "V P p1 a=1 a=2", "V P p1 =3", "# x\n\nE a", "V P p1 a=1\nE p1 p1 p1"]
    for text in cases:
        with_ref = with_mine = None
        try:
            ref_parse(text)
        except RefError as exc:
            with_ref = str(exc)
        try:
            parse_graph_text(text)
        except GraphFormatError as exc:
            with_mine = str(exc)
        assert with_mine == with_ref, text


def test_one_hot_rows_matches_hot_index():
    """TrioResult.open's batched decoding (trio.one_hot_rows) equals
    BitVector.hot_index (src/bits.py) row by row: random one-hot and all-zero
    rows over fields of different widths, empty fields included, and the
    weight > 1 error names the first offending row's weight."""
    import pytest

    from paper_2209_03526_b200.bits import BitVector
    from paper_2209_03526_b200.trio import one_hot_rows

    rng = np.random.default_rng(7)
    shapes = [(5, 1), (0, 3), (17, 4), (1, 33), (0, 0), (9, 2)]
    mats = []
    for rows, w in shapes:
        m = np.zeros((rows, w), np.uint32)
        for r in range(rows):
            if w and rng.random() < 0.8:
                b = int(rng.integers(0, 32 * w))
                m[r, b // 32] = np.uint32(1) << np.uint32(b % 32)
        mats.append(m)
    x = np.concatenate([m.reshape(-1) for m in mats])
    got = one_hot_rows(x, shapes)
    want = [[BitVector(m[r], 32 * m.shape[1]).hot_index() if m.shape[1] else None for r in range(m.shape[0])]
            for m in mats]
    assert got == want
    assert one_hot_rows(np.zeros(0, np.uint32), []) == []
    bad = [m.copy() for m in mats]
    bad[2][3] = 0
    bad[2][3, 0] = 0b1011
    bad[5][0, 1] = 0b11
    with pytest.raises(ValueError, match="expected Hamming weight <= 1, got 3"):
        one_hot_rows(np.concatenate([m.reshape(-1) for m in bad]), shapes)
