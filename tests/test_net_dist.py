"""Party transport across processes (torch.distributed, gloo on CPU):
framing, round counters and transcript digests equal the co-resident
runtime's for the same message sequence (src/net.py:131-165, 288-295)."""

import os

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_03526_b200.net import OP_OPEN, OP_RESHARE, Message, make_session_configs


def _script(rt):
    """A fixed message pattern touching every op and direction."""
    got = []
    for k in range(3):
        rt.send_next(OP_RESHARE, Message(b"", torch.arange(5 + k, dtype=torch.int32) * rt.index), logical_bits=7)
        got.append(rt.recv_prev(OP_RESHARE).tensor.tolist())
    rt.send_next(OP_OPEN, Message((7).to_bytes(4, "little"), torch.full((3,), rt.index, dtype=torch.int32)))
    m = rt.recv_prev(OP_OPEN)
    got.append((m.head, m.tensor.tolist()))
    rt.send_prev(OP_RESHARE, Message(b"xy", None))
    got.append(rt.recv_next(OP_RESHARE).head)
    return got


def _worker(rank, port, q, skew):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=3)
    from paper_2209_03526_b200.net_dist import DistPartyRuntime
    from paper_2209_03526_b200.errors import ProtocolError
    cfg = make_session_configs(b"\x09" * 16)[rank]
    rt = DistPartyRuntime(cfg, transcript=True, device="cpu")
    try:
        if skew and rank == 1:
            rt.links[rt._next]._tx[OP_RESHARE] = 5   # party 2 skips rounds on its link to party 3
        out = _script(rt)
        rt.flush()
        q.put((rank, out, rt.transcript_digest(), rt.meter.total.bytes_sent, None))
    except ProtocolError as exc:
        q.put((rank, None, None, None, str(exc)))
    dist.barrier() if not skew else None
    dist.destroy_process_group()


def _run(skew=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + (7 if skew else 0) + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, port, q, skew)) for r in range(3)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(3):
        try:
            r = q.get(timeout=90 if not res else (5 if skew else 60))
            res[r[0]] = r
            if skew and r[4]:
                break  # the peers of a failing party block in recv; stop here
        except Exception:
            break
    for p in procs:
        p.join(30)
        if p.is_alive():
            p.kill()
    return res


def test_dist_runtime_matches_co_resident_runtime():
    import paper_2209_03526_b200.net as net
    res = _run()
    assert len(res) == 3 and all(r[4] is None for r in res.values())
    # the same script on the co-resident (thread) runtime, CPU tensors
    cfgs = make_session_configs(b"\x09" * 16)
    trs = [net._new_transcript(c) for c in cfgs]
    q = {(i, j): net.DeviceChannel() for i in (1, 2, 3) for j in (1, 2, 3) if i != j}

    class CpuRt(net.PartyRuntime):  # thread runtime without CUDA streams
        def __init__(self, cfg, links, tr):
            from paper_2209_03526_b200.rss import ZeroShareContext
            self.index, self.session, self.links, self._transcript = cfg.party_index, cfg.session, links, tr
            self.meter, self.opened, self.recv_timeout = net.Meter(), [], 30.0
            self._next, self._prev = net.next_party(self.index), net.prev_party(self.index)

    rts = []
    for c, tr in zip(cfgs, trs):
        i = c.party_index
        links = {j: net.PeerLink(q[(i, j)], q[(j, i)], c.session, tr) for j in (1, 2, 3) if j != i}
        rts.append(CpuRt(c, links, tr))
    import threading
    outs = [None] * 3
    ths = [threading.Thread(target=lambda k=k: outs.__setitem__(k, _script(rts[k]))) for k in range(3)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for k in range(3):
        assert res[k][1] == outs[k]
        assert res[k][2] == rts[k].transcript_digest()
        assert res[k][3] == rts[k].meter.total.bytes_sent


def test_dist_runtime_detects_round_skew():
    res = _run(skew=True)
    errs = [r[4] for r in res.values() if r[4]]
    assert any("round skew" in e for e in errs)
