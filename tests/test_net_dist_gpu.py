"""Three server processes (one party each) on the GPU, talking over the
distributed transport: the campus query reproduces the reference's records,
opened flags and per-party transcript digests (tests/golden/match.npz)."""

import json
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _party(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=3)
    torch.cuda.set_device(0)
    from paper_2209_03526_b200.engine import EngineConfig, sec_match
    from paper_2209_03526_b200.graphs import encrypt_graph, parse_graph_text
    from paper_2209_03526_b200.net import make_session_configs
    from paper_2209_03526_b200.net_dist import DistPartyRuntime
    from paper_2209_03526_b200.query import gen_token, load_query
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "match.npz"))
    rec = json.loads(str(g["campus_json"]))
    rng = np.random.default_rng(rec["seed"])
    schema, shares = encrypt_graph(parse_graph_text(rec["graph"]), rec["k"], rng)
    tokens = gen_token(load_query(rec["query"], schema), schema, rng)
    cfg = make_session_configs(bytes.fromhex(rec["master"]))[rank]
    rt = DistPartyRuntime(cfg, transcript=True)
    res = sec_match(rt, tokens[rank], shares[rank].to_device(), EngineConfig())
    rt.flush()
    torch.cuda.synchronize()
    q.put((rank, rt.transcript_digest(), [list(sg) for sg in res.subgraphs],
           [[r.vertex_id.share_a.words.cpu().numpy().tobytes() for r in recs] for recs in res.records]))
    dist.barrier()
    dist.destroy_process_group()


def test_three_party_processes_match_reference(golden):
    g = golden("match")
    rec = json.loads(str(g["campus_json"]))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + os.getpid() % 500
    procs = [ctx.Process(target=_party, args=(r, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    out = dict((r[0], r) for r in (q.get(timeout=300) for _ in range(3)))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for p in range(3):
        assert out[p][1] == rec["digests"][p]
        assert out[p][2] == rec["subgraphs"]
        for s, recs in enumerate(out[p][3]):
            for ri, words in enumerate(recs):
                assert np.frombuffer(words, np.uint32).tolist() == g[f"campus_p{p}_s{s}_r{ri}_id_a"].tolist()
