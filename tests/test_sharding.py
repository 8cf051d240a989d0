"""Multi-rank secEval host logic on CPU: world_size-2 gloo all-gather of
row-sharded, zero-share-blinded match bits must equal the unsharded result
bit for bit.  The per-shard arithmetic is the CPU oracle
(tests may call it); the shard plan, CTR-block-aligned slicing, padding and
assembly are the product's (paper_2209_03526_b200.sharding)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2209_03526_b200.sharding import ALIGN_ROWS, ShardPlan, all_gather_bits

ROWS, WORDS, COUNTER = 1000, 9, 5
KEYS = [bytes([i + 1]) * 16 for i in range(3)]
PAIRS = [(KEYS[0], KEYS[2]), (KEYS[1], KEYS[0]), (KEYS[2], KEYS[1])]


def _inputs():
    rng = np.random.default_rng(42)
    comps = [rng.integers(0, 1 << 32, (ROWS, WORDS), dtype=np.uint32) for _ in range(3)]
    inds = [(rng.integers(0, 1 << 32, WORDS, dtype=np.uint32), rng.integers(0, 1 << 32, WORDS, dtype=np.uint32))
            for _ in range(3)]
    return comps, inds


def _blinded_reference():
    comps, inds = _inputs()
    out = []
    for q in range(3):
        bits = oracle.masked_parity(comps[q], comps[(q + 1) % 3], *inds[q])
        out.append(oracle.pack_bits(bits) ^ oracle.zero_share(*PAIRS[q], COUNTER, ROWS))
    return out


def _zero_share_slice(q, w0, nwords):
    """Words [w0, w0+nwords) of the share via CTR block offsets (oracle)."""
    blk0 = w0 // 4
    raw = [np.frombuffer(oracle.prf_stream(k, b"ZSHR", COUNTER, 16 * (-(-nwords // 4)), block_offset=blk0),
                         np.uint32) for k in PAIRS[q]]
    w = (raw[0] ^ raw[1])[:nwords].copy()
    total = -(-ROWS // 32)
    if ROWS % 32 and w0 + nwords == total:
        w[-1] &= np.uint32((1 << (ROWS % 32)) - 1)
    return w


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comps, inds = _inputs()
    plan = ShardPlan(ROWS, world)
    lo, hi = plan.bounds(rank)
    w0, w1 = plan.word_bounds(rank)
    outs = []
    for party in range(3):
        bits = oracle.masked_parity(comps[party][lo:hi], comps[(party + 1) % 3][lo:hi], *inds[party])
        local = oracle.pack_bits(bits) if hi > lo else np.zeros(0, np.uint32)
        local = local ^ _zero_share_slice(party, w0, w1 - w0)
        full = all_gather_bits(torch.from_numpy(local.view(np.int32).copy()), plan)
        outs.append(full.numpy().view(np.uint32).copy())
    q.put((rank, outs))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sec_eval_equals_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 7 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    want = _blinded_reference()
    for r in range(world):
        for party in range(3):
            assert np.array_equal(got[r][party], want[party]), (world, r, party)


def test_plan_alignment_and_coverage():
    for rows in (1, 31, 128, 1000, 200_000, 2_000_001):
        for world in (1, 2, 4, 8):
            plan = ShardPlan(rows, world)
            covered = []
            for r in range(world):
                lo, hi = plan.bounds(r)
                assert lo % ALIGN_ROWS == 0 or lo == rows
                covered.extend(range(lo, hi)) if rows < 5000 else None
            if rows < 5000:
                assert covered == list(range(rows))
            assert plan.bounds(world - 1)[1] == rows


# ---------------------------------------------------------------------------
# row-sharded shuffle: exchange plans + all_to_all (gloo, CPU)
# ---------------------------------------------------------------------------

SH_ROWS, SH_W = 1000, 5


def _numpy_take(rows, width, src, idx, r=None, m3=None):
    out = src[idx.long()].clone() if rows else torch.zeros((0, src.shape[1]), dtype=src.dtype)
    if r is not None:
        out ^= r
    if m3 is not None:
        out ^= m3
    return out


def _xworker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2209_03526_b200.sharding as sh
    sh._take = _numpy_take   # test-only CPU data movement; plans + collective are the product's
    g = torch.Generator().manual_seed(11)
    M = torch.randint(-2**31, 2**31 - 1, (SH_ROWS, SH_W), dtype=torch.int32, generator=g)
    k = torch.randperm(SH_ROWS, generator=g).to(torch.int32)
    plan = sh.ShardPlan(SH_ROWS, world, align=1)
    lo, hi = plan.bounds(rank)
    xp = sh.exchange_plan(k, plan, rank)
    out = sh.exchange_gather(M[lo:hi], xp, 32 * SH_W)
    q.put((rank, out.numpy().copy(), M[k.long()][lo:hi].numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_exchange_gather_all_to_all(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 11 + os.getpid() % 1000
    procs = [ctx.Process(target=_xworker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank, out, want in got:
        assert np.array_equal(out, want), rank


# ---------------------------------------------------------------------------
# sharded folds (XOR all-reduce) and sharded open + compaction (gloo, CPU)
# ---------------------------------------------------------------------------

F_ROWS, F_WORDS = 700, 6


def _fold_inputs():
    rng = np.random.default_rng(77)
    mats = [rng.integers(0, 1 << 32, (F_ROWS, F_WORDS), dtype=np.uint32) for _ in range(3)]
    flags = [rng.integers(0, 1 << 32, -(-F_ROWS // 32), dtype=np.uint32) for _ in range(3)]
    return mats, flags


def _numpy_fold(rows, words, mats, flags):
    """src/engine.py:95-102 for the three parties (test-only CPU stand-in for the kernel)."""
    out = []
    for q in range(3):
        a, b = mats[q].numpy().view(np.uint32)[:rows], mats[(q + 1) % 3].numpy().view(np.uint32)[:rows]
        fa = np.unpackbits(flags[q].numpy().view(np.uint8), bitorder="little")[:rows].astype(bool)
        fb = np.unpackbits(flags[(q + 1) % 3].numpy().view(np.uint8), bitorder="little")[:rows].astype(bool)
        acc = np.bitwise_xor.reduce(a[fa] ^ b[fa], axis=0) if fa.any() else np.zeros(words, np.uint32)
        acc = acc ^ (np.bitwise_xor.reduce(a[fb], axis=0) if fb.any() else np.zeros(words, np.uint32))
        out.append(torch.from_numpy(np.asarray(acc, np.uint32).view(np.int32).copy()))
    return out


def _numpy_compact(bits, n, k):
    b = np.unpackbits(bits.numpy().view(np.uint8), bitorder="little")[:n]
    return torch.from_numpy(np.nonzero(b)[0].astype(np.int32))[:k]


def _fworker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2209_03526_b200.sharding as sh
    sh._fold_local = _numpy_fold     # test-only CPU arithmetic; slicing + collectives are the product's
    sh._compact = _numpy_compact
    mats, flags = _fold_inputs()
    plan = sh.ShardPlan(F_ROWS, world, align=32)
    lo, hi = plan.bounds(rank)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32).copy())  # noqa: E731
    folds = sh.sharded_fold_trio([t(m[lo:hi]) for m in mats], [t(f) for f in flags], plan, rank)
    plain = np.unpackbits(flags[0].view(np.uint8), bitorder="little")[:F_ROWS]
    local_bits = np.packbits(np.concatenate([plain[lo:hi], np.zeros((-(hi - lo)) % 32, np.uint8)]),
                             bitorder="little").view(np.uint32)
    host, local, first, total = sh.sharded_keep(t(local_bits), plan, rank)
    q.put((rank, [f.numpy().view(np.uint32).copy() for f in folds], host.copy(), (local.numpy() + lo).tolist(),
           first, total))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fold_and_keep(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + world * 13 + os.getpid() % 1000
    procs = [ctx.Process(target=_fworker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=120) for _ in range(world)), key=lambda x: x[0])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    mats, flags = _fold_inputs()
    want = _numpy_fold(F_ROWS, F_WORDS, [torch.from_numpy(m.view(np.int32)) for m in mats],
                       [torch.from_numpy(f.view(np.int32)) for f in flags])
    plain = np.unpackbits(flags[0].view(np.uint8), bitorder="little")[:F_ROWS]
    kept = np.nonzero(plain)[0].tolist()
    order = []
    for rank, folds, host, local, first, total in got:
        for party in range(3):
            assert np.array_equal(folds[party], want[party].numpy().view(np.uint32)), (world, rank, party)
        assert np.array_equal(np.unpackbits(host.view(np.uint8), bitorder="little")[:F_ROWS], plain)
        assert total == len(kept) and first == len(order)
        order += local
    assert order == kept


def _pworker(rank, world, port, q):
    """sharded_sec_eval_trio's exchange: one all-gather of the packed
    (pass, party) buffer + assembly; the per-rank arithmetic is the oracle."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2209_03526_b200.sharding as sh
    comps, inds = _inputs()
    plan = ShardPlan(ROWS, world)
    lo, hi = plan.bounds(rank)
    w0, w1 = plan.word_bounds(rank)

    def local_packed(*_a, **_k):
        packed = torch.zeros((3, plan.words_per_rank), dtype=torch.int32)
        for party in range(3):
            bits = oracle.masked_parity(comps[party][lo:hi], comps[(party + 1) % 3][lo:hi], *inds[party])
            local = oracle.pack_bits(bits) if hi > lo else np.zeros(0, np.uint32)
            local = local ^ _zero_share_slice(party, w0, w1 - w0)
            packed[party, : local.size] = torch.from_numpy(local.view(np.int32).copy())
        return packed

    sh.sec_eval_local_packed = local_packed   # test-only CPU arithmetic; exchange + assembly are the product's
    res = sh.sharded_sec_eval_trio(None, WORDS, plan, rank, [None], None, [COUNTER])
    q.put((rank, [t.numpy().view(np.uint32).copy() for t in res[0]]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sec_eval_single_all_gather(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30100 + world * 17 + os.getpid() % 1000
    procs = [ctx.Process(target=_pworker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    want = _blinded_reference()
    for r in range(world):
        for party in range(3):
            assert np.array_equal(got[r][party], want[party]), (world, r, party)
