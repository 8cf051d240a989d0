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
