"""File formats (src/storage.py) against files written by the live reference."""

import io
import json
import tempfile

import numpy as np
import pytest

from paper_2209_03526_b200.graphs import GraphSchema, encrypt_graph, parse_graph_text
from paper_2209_03526_b200.storage import StorageError, load_graph_share, save_graph_share


def _campus():
    from __graft_entry__ import SMOKE_GRAPH
    return parse_graph_text(SMOKE_GRAPH)


def test_graph_share_files_byte_identical_and_loadable(golden, tmp_path):
    g = golden("storage")
    schema = GraphSchema.from_json(g["schema_json"].tobytes().decode())
    mine_schema, shares = encrypt_graph(_campus(), 2, np.random.default_rng(1))
    assert mine_schema.digest() == schema.digest()
    for p in range(3):
        save_graph_share(tmp_path / f"g{p}.ogmg", shares[p])
        assert (tmp_path / f"g{p}.ogmg").read_bytes() == g[f"ogmg{p}"].tobytes()
        (tmp_path / f"ref{p}.ogmg").write_bytes(g[f"ogmg{p}"].tobytes())
        loaded = load_graph_share(tmp_path / f"ref{p}.ogmg", schema, device=None)
        for t in shares[p].types:
            a, b = shares[p].types[t], loaded.types[t]
            x = schema.types[t].population
            eq = lambda m, n, width: np.array_equal(masked(m, width), n)  # noqa: E731
            assert eq(a.id_a, b.id_a, x) and eq(a.id_b, b.id_b, x)
            for n in a.attrs:
                d = schema.types[t].attrs[n].domain_size
                assert eq(a.attrs[n][0], b.attrs[n][0], d) and eq(a.attrs[n][1], b.attrs[n][1], d)
            for n in a.posting:
                x2 = schema.types[n].population
                assert eq(a.posting[n][0], b.posting[n][0], x2) and eq(a.posting[n][1], b.posting[n][1], x2)


def masked(m, width):
    """Share rows as the reference stores them: BitVector(words, width) masks tails."""
    m = np.array(m, np.uint32)
    if width % 32 and m.size:
        m[..., -1] &= np.uint32((1 << (width % 32)) - 1)
    return m


def test_graph_share_corruption_is_rejected(golden, tmp_path):
    g = golden("storage")
    schema = GraphSchema.from_json(g["schema_json"].tobytes().decode())
    raw = bytearray(g["ogmg0"].tobytes())
    path = tmp_path / "bad.ogmg"
    path.write_bytes(bytes(raw[:-3]))
    with pytest.raises(StorageError, match="truncated"):
        load_graph_share(path, schema, device=None)
    raw2 = bytearray(raw)
    raw2[_first_record(raw2) + 6] ^= 3   # party byte of the first record
    path.write_bytes(bytes(raw2))
    with pytest.raises(StorageError, match="party"):
        load_graph_share(path, schema, device=None)
    raw3 = bytearray(raw)
    raw3[0] = ord("X")
    path.write_bytes(bytes(raw3))
    with pytest.raises(StorageError, match="not a graph share"):
        load_graph_share(path, schema, device=None)


def _first_record(raw):
    return 4 + 2 + 1 + 32
