"""Multi-GPU sec_match (sharded_trio.ShardedTrio): every type table
row-sharded over W ranks, collectives for the exchanges.

Emulated ranks (ThreadComm, W threads on one GPU) at W = 1, 2, 3 and 8, and
two real processes over torch.distributed (gloo), must reproduce the live
reference's recorded sec_match runs (tests/golden/match.npz) bit for bit on
every rank: matches, subgraphs, every record share and every opened vector.
"""

import json
import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

NAMES = ["campus", "unique-chain", "conj", "c1", "rand0", "rand1", "rand2"]


def _setup(g, name):
    from paper_2209_03526_b200.graphs import device_trio, encrypt_graph, parse_graph_text
    from paper_2209_03526_b200.query import gen_token, load_query

    rec = json.loads(str(g[f"{name}_json"]))
    rng = np.random.default_rng(rec["seed"])
    schema, shares = encrypt_graph(parse_graph_text(rec["graph"]), rec["k"], rng)
    tokens = gen_token(load_query(rec["query"], schema), schema, rng)
    return rec, schema, tokens, device_trio(shares)


def _check(g, name, rec, schema, res):
    from paper_2209_03526_b200.engine import open_results

    host = lambda t: t.detach().cpu().numpy().view(np.uint32)  # noqa: E731
    results = res.party_results()
    matches, _ = open_results(results[:2], schema)
    assert sorted(list(m) for m in set(matches)) == rec["matches"], name
    assert [list(sg) for sg in res.subgraphs] == rec["subgraphs"], name
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
            assert np.array_equal(bits, g[f"{name}_p{p}_open{j}"]), (name, j)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("name", NAMES)
def test_sharded_match_emulated_ranks(golden, name, world):
    from paper_2209_03526_b200.sharded_trio import ShardedTrio, local_shards, run_emulated

    g = golden("match")
    rec, schema, tokens, dshares = _setup(g, name)
    master = bytes.fromhex(rec["master"])

    def rank_fn(comm):
        mine = local_shards(list(dshares), world, comm.rank)
        return ShardedTrio(master, comm).match(list(tokens), mine, any_mode=rec["mode"])

    for res in run_emulated(world, rank_fn):
        _check(g, name, rec, schema, res)


def _gloo_worker(rank, world, port, name, out_dir):
    import torch.distributed as dist

    from paper_2209_03526_b200.sharded_trio import ShardedTrio, local_shards
    from tests.conftest import GOLDEN

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = np.load(GOLDEN / "match.npz", allow_pickle=False)
    rec, schema, tokens, dshares = _setup(g, name)
    res = ShardedTrio(bytes.fromhex(rec["master"]), None).match(list(tokens), local_shards(list(dshares), world, rank),
                                                                any_mode=rec["mode"])
    _check(g, name, rec, schema, res)
    with open(os.path.join(out_dir, f"ok{rank}"), "w") as f:
        f.write("ok")
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["campus", "c1", "rand1"])
def test_sharded_match_two_gloo_processes(name, tmp_path):
    """Two processes, torch.distributed over gloo (the NCCL code path's
    collectives staged through the host), one GPU: both ranks reproduce the
    reference run."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.spawn(_gloo_worker, args=(2, port, name, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok0").exists() and (tmp_path / "ok1").exists()
