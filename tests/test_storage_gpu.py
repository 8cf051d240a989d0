"""Reference-written graph shares loaded straight into HBM serve the query and
reproduce the reference's own result files byte for byte."""

import numpy as np
import pytest

from paper_2209_03526_b200.engine import EngineConfig, open_results, sec_match
from paper_2209_03526_b200.graphs import GraphSchema, parse_graph_text
from paper_2209_03526_b200.net import local_runtimes, make_session_configs, run_trio
from paper_2209_03526_b200.query import gen_token, load_query
from paper_2209_03526_b200.storage import load_graph_share, load_results, save_results

pytestmark = pytest.mark.gpu


def test_device_loaded_reference_files_serve_query_and_round_trip_results(golden, tmp_path):
    from __graft_entry__ import SMOKE_GRAPH, SMOKE_QUERY
    from paper_2209_03526_b200.graphs import encrypt_graph
    g = golden("storage")
    schema = GraphSchema.from_json(g["schema_json"].tobytes().decode())
    dev_shares = []
    for p in range(3):
        (tmp_path / f"g{p}.ogmg").write_bytes(g[f"ogmg{p}"].tobytes())
        dev_shares.append(load_graph_share(tmp_path / f"g{p}.ogmg", schema))   # -> HBM via ogm_unpack_records
    rng = np.random.default_rng(1)
    encrypt_graph(parse_graph_text(SMOKE_GRAPH), 2, rng)          # advance rng exactly as the reference did
    tokens = gen_token(load_query(SMOKE_QUERY, schema), schema, rng)
    rts = local_runtimes(make_session_configs(b"\x11" * 16))
    res = run_trio(lambda rt: sec_match(rt, tokens[rt.index - 1], dev_shares[rt.index - 1], EngineConfig()), rts)
    assert set(open_results(res[:2], schema)[0]) == {("u1", "p1", "p3", "c1", "c2"), ("u1", "p2", "p3", "c1", "c2")}
    for p in range(3):
        save_results(tmp_path / f"r{p}.ogmr", res[p], schema)
        assert (tmp_path / f"r{p}.ogmr").read_bytes() == g[f"ogmr{p}"].tobytes()
        (tmp_path / f"ref{p}.ogmr").write_bytes(g[f"ogmr{p}"].tobytes())
    back = [load_results(tmp_path / f"ref{p}.ogmr", schema) for p in range(3)]
    assert set(open_results(back, schema)[0]) == {("u1", "p1", "p3", "c1", "c2"), ("u1", "p2", "p3", "c1", "c2")}
