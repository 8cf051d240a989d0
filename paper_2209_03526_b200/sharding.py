"""Row sharding across GPUs: one process per GPU.

secEval shards naturally: candidate rows are independent.  Vertex tables are
partitioned by vertex-id ranges whose sizes are multiples of 128 rows, so
every shard's packed output starts on a 16-byte CTR block of the zero-share
stream (128 rows = 4 words = 1 AES block).  Each rank evaluates its rows for
all three co-resident parties, blinds them with *its slice* of the
zero-share stream (random access by CTR block, ogm_zero_share_slice), and
the one exchange -- an all-gather of the packed blinded bits -- rebuilds the
full re-shared vector on every rank, bit-identical to the single-GPU run.
Party messages never cross NVLink: the three servers live on every GPU.

The plan / assembly logic is device-agnostic (covered by gloo tests on CPU);
:func:`sharded_sec_eval_trio` is the CUDA path (NCCL all-gather).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, fss
from .bits import words_for

ALIGN_ROWS = 128  # one AES-CTR block of packed bits


class Comm:
    """The two collectives the sharded stages need, over ``world`` ranks.
    ``group`` arguments below accept a Comm or a torch.distributed process
    group (None = the default group)."""

    rank: int = 0
    world: int = 1

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        """Every rank's ``t`` (same shape on all), concatenated flat in rank order."""
        raise NotImplementedError

    def all_to_all(self, recv: torch.Tensor, send: torch.Tensor, recv_splits: list, send_splits: list) -> None:
        """Rows send[sum(send_splits[:r]) : ...] go to rank r; recv holds
        every rank's rows for this one, in rank order."""
        raise NotImplementedError


class DistComm(Comm):
    """torch.distributed: NCCL on device tensors (over NVLink); gloo stages
    device tensors through the host."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host = dist.get_backend(group) == "gloo"

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        flat = t.reshape(-1).contiguous()
        src = flat.cpu() if self.host else flat
        out = torch.empty((self.world * flat.numel(),), dtype=flat.dtype, device=src.device)
        self.dist.all_gather_into_tensor(out, src, group=self.group)
        return out.to(flat.device)

    def all_to_all(self, recv, send, recv_splits, send_splits) -> None:
        if not self.host:
            self.dist.all_to_all_single(recv, send, recv_splits, send_splits, group=self.group)
            return
        r = torch.empty(recv.shape, dtype=recv.dtype)
        self.dist.all_to_all_single(r, send.cpu(), recv_splits, send_splits, group=self.group)
        recv.copy_(r)


class ThreadComm:
    """``world`` emulated ranks in one process, one thread each, sharing a
    device (tests): collectives meet at a barrier.  ``comm.rank_view(r)`` is
    rank r's Comm."""

    def __init__(self, world: int):
        import threading
        self.world = world
        self._barrier = threading.Barrier(world)
        self._slots: list = [None] * world

    def rank_view(self, rank: int) -> "Comm":
        return _ThreadRank(self, rank)


class _ThreadRank(Comm):
    def __init__(self, hub: ThreadComm, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def _exchange(self, item):
        if item is not None and isinstance(item[0], torch.Tensor) and item[0].is_cuda:
            torch.cuda.current_stream(item[0].device).synchronize()   # the deposit is complete
        self.hub._slots[self.rank] = item
        self.hub._barrier.wait()
        got = list(self.hub._slots)
        self.hub._barrier.wait()   # every rank has read the slots before they are reused
        return got

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        got = self._exchange((t.reshape(-1).contiguous(),))
        return torch.cat([g[0].to(t.device) for g in got])

    def all_to_all(self, recv, send, recv_splits, send_splits) -> None:
        got = self._exchange((send, list(send_splits)))
        parts = []
        for src_send, src_splits in got:
            off = sum(src_splits[: self.rank])
            parts.append(src_send[off: off + src_splits[self.rank]].to(recv.device))
        if parts and recv.numel():
            recv.copy_(torch.cat(parts))


def as_comm(group) -> Comm:
    return group if isinstance(group, Comm) else DistComm(group)


@dataclass(frozen=True)
class ShardPlan:
    rows: int
    world: int
    align: int = ALIGN_ROWS

    @property
    def per_rank(self) -> int:
        per = -(-self.rows // self.world)
        return -(-per // self.align) * self.align

    def bounds(self, rank: int) -> tuple[int, int]:
        lo = min(rank * self.per_rank, self.rows)
        return lo, min(lo + self.per_rank, self.rows)

    def word_bounds(self, rank: int) -> tuple[int, int]:
        lo, hi = self.bounds(rank)
        return lo // 32, words_for(hi) if hi > lo else lo // 32

    @property
    def words_per_rank(self) -> int:
        return self.per_rank // 32

    @property
    def total_words(self) -> int:
        return words_for(self.rows)


def pad_slice(local: torch.Tensor, plan: ShardPlan) -> torch.Tensor:
    """Local packed words -> fixed-size all-gather chunk (zero padded)."""
    out = torch.zeros((plan.words_per_rank,), dtype=local.dtype, device=local.device)
    out[: local.numel()] = local
    return out


def assemble(gathered: torch.Tensor, plan: ShardPlan) -> torch.Tensor:
    """All-gathered chunks (world * words_per_rank) -> the full packed vector."""
    parts = []
    for r in range(plan.world):
        lo, hi = plan.word_bounds(r)
        parts.append(gathered[r * plan.words_per_rank: r * plan.words_per_rank + (hi - lo)])
    return torch.cat(parts)[: plan.total_words]


def all_gather_bits(local: torch.Tensor, plan: ShardPlan, group=None) -> torch.Tensor:
    return assemble(as_comm(group).all_gather(pad_slice(local, plan)), plan)


def fold_indicators(inds) -> list:
    """[pass][party] -> (ind_a, ind_b) of a two-pass predicate folded into ONE
    pass: per party (a0 ^ a1, b0 ^ b1).  Parity is linear, so one masked
    parity over the folded indicators is the XOR of the two passes'
    (sec_eval_local_packed(fold=True))."""
    def x(a, b):
        o = torch.empty_like(a)
        _lib.call("ogm_xor_words", a.numel(), _lib.ptr(a), _lib.ptr(b), None, _lib.ptr(o), _lib.stream_ptr())
        return o
    return [[(x(inds[0][q][0], inds[1][q][0]), x(inds[0][q][1], inds[1][q][1])) for q in range(3)]]


def sec_eval_local_packed(comps, words: int, plan: ShardPlan, rank: int, inds, zero_keys, counters,
                          fold: bool = False) -> torch.Tensor:
    """This rank's share of a row-sharded secEval for all three parties: the
    blinded packed bits of its rows for every (pass, party), as one
    zero-padded (3*npass, words_per_rank) buffer ready for ONE all-gather
    (at 8 GPUs the per-call collective latency, not the kernel, bounds the
    strong scaling).  Row j = pass j // 3, party j % 3.

    fold=True (a two-pass predicate, co-resident trio): ``inds`` holds the
    ONE folded pass (fold_indicators) and ``counters`` both passes' zero-share
    counters; the buffer then holds 3 rows, each the XOR of the two passes'
    re-shared bits (both zero shares XORed in) -- the same result shares from
    one parity pass and half the all-gather."""
    if plan.per_rank % 32:
        raise ValueError("secEval shards need row counts that are multiples of 32 (default ShardPlan alignment)")
    if fold and (len(inds) != 1 or len(counters) != 2):
        raise ValueError("a folded secEval takes one folded pass of indicators and two counters")
    lo, hi = plan.bounds(rank)
    nloc = hi - lo
    npass = len(inds)
    nvec = 3 * npass
    w0, w1 = plan.word_bounds(rank)
    wpr = max(plan.words_per_rank, 1)
    # the zero shares are written first (they initialise the words), then the parities are
    # XORed in: no zeroing launches; only a short last shard's padding is cleared
    packed = torch.empty((nvec, wpr), dtype=torch.int32, device=comps[0].device)
    if w1 - w0 < wpr:
        packed[:, w1 - w0:].zero_()
    outs = [packed[j] for j in range(nvec)]
    A = _lib.ptr_array
    adds = [[outs[ps * 3 + q][: w1 - w0] for q in range(3)] for ps in range(npass)]
    k = (zero_keys[0][0], zero_keys[1][0], zero_keys[2][0])
    none3 = A([None, None, None])
    if w1 > w0 and fold:
        # both passes' zero shares in one output (F(c0) ^ F(c1) per key)
        _lib.call("ogm_zero_share_trio_fold2", *k, counters[0], counters[1], plan.rows, w0, w1 - w0, none3,
                  A(adds[0]), _lib.stream_ptr())
    elif w1 > w0 and npass == 2:
        # both passes, all three parties: one launch (3 AES per block and pass, not 6)
        _lib.call("ogm_zero_share_trio_slice2", *k, counters[0], counters[1], plan.rows, w0, w1 - w0,
                  none3, A(adds[0]), none3, A(adds[1]), _lib.stream_ptr())
    elif w1 > w0:
        _lib.call("ogm_zero_share_trio_slice", *k, counters[0], plan.rows, w0, w1 - w0, none3, A(adds[0]),
                  _lib.stream_ptr())
    if nloc:
        flat = [t for ps in range(npass) for q in range(3) for t in inds[ps][q]]
        _lib.call("ogm_masked_parity_acc", nloc, words, comps[0].stride(0), 3, A(comps), 3,
                  _lib.int_array([0, 1, 2]), _lib.int_array([1, 2, 0]), npass, A(flat), A(outs),
                  _lib.stream_ptr())
    return packed


def assemble_many(gathered: torch.Tensor, plan: ShardPlan) -> list:
    """(world, nvec, words_per_rank) all-gathered buffers -> nvec full vectors.
    Every rank but the trailing ones holds exactly words_per_rank words (the
    plan gives each per_rank rows, a multiple of 32), so all padding sits at
    the end: one transposing copy, then a slice."""
    world, nvec, wpr = gathered.shape
    flat = gathered.permute(1, 0, 2).reshape(nvec, world * wpr)
    return [flat[j, : plan.total_words] for j in range(nvec)]


def sharded_sec_eval_trio(comps, words: int, plan: ShardPlan, rank: int, inds, zero_keys, counters,
                          group=None, fold: bool = False) -> list:
    """One secEval for all three parties on this rank's row shard.

    comps: the three (rows_local, pitch) share components of this shard.
    inds:  [pass][party] -> (ind_a, ind_b) full-domain indicator words.
    zero_keys: [(k_own, k_prev)] per party (src/net.py:229-232).
    counters: zero-share counter per pass (identical across parties).
    Returns per pass the three parties' full blinded vectors (all ranks),
    i.e. the re-share messages; component j of the result is blinded_{j-1}.
    fold: as sec_eval_local_packed (one folded pass, two counters).
    """
    packed = sec_eval_local_packed(comps, words, plan, rank, inds, zero_keys, counters, fold=fold)
    nvec, wpr = packed.shape
    if plan.world == 1:
        full = [packed[j][: plan.total_words] for j in range(nvec)]
    else:
        out = as_comm(group).all_gather(packed)
        full = assemble_many(out.view(plan.world, nvec, wpr), plan)
    return [[full[ps * 3 + q] for q in range(3)] for ps in range(nvec // 3)]


# ---------------------------------------------------------------------------
# Sharded folds (Case I fetch, sec_access posting fold) and the
# sharded open + compaction
# ---------------------------------------------------------------------------
#
# A fold XOR-reduces over candidate rows, so a row shard folds its own rows
# and one exchange combines the partials.  NCCL has no XOR reduction: the
# exchange is an all-gather of the per-rank partials followed by a local XOR
# fold -- w(width) words per rank per party, tiny next to the fold's read.


def xor_allreduce(t: torch.Tensor, group=None) -> torch.Tensor:
    """XOR of `t` over all ranks (same shape everywhere): all-gather + fold."""
    comm = as_comm(group)
    flat = t.reshape(-1).contiguous()
    out = comm.all_gather(flat).view(comm.world, flat.numel())
    world = comm.world
    acc = out[0].clone()
    for r in range(1, world):
        acc ^= out[r]
    return acc.reshape(t.shape)


def _fold_local(rows: int, words: int, mats: list, flags: list) -> list:
    """The three parties' partial folds of this rank's rows (one trio launch)."""
    outs = [torch.empty((max(words, 1),), dtype=torch.int32, device=mats[0].device)[:words] for _ in range(3)]
    A = _lib.ptr_array
    _lib.call("ogm_select_fold", rows, words, mats[0].stride(0) if rows else words, 3, A(mats),
              A([mats[(q + 1) % 3] for q in range(3)]), A(flags), A([flags[(q + 1) % 3] for q in range(3)]),
              A(outs), _lib.stream_ptr())
    return outs


def sharded_fold_trio(mats_local: list, flags_full: list, plan: ShardPlan, rank: int, group=None) -> list:
    """src/engine.py:95-102 (_select_one_additive) over row-sharded matrices
    for the three co-resident parties: mats_local[c] holds this rank's rows
    [lo, hi) of component c (rows x pitch), flags_full[c] the full selection
    bit vector of component c (replicated: C/8 bytes).  Returns every
    party's additive fold, identical on all ranks to the unsharded fold."""
    lo, hi = plan.bounds(rank)
    if hi > lo and lo % 32:
        raise ValueError("fold shards must start on a 32-row word boundary")
    words = mats_local[0].shape[1] if mats_local[0].dim() == 2 else 0
    w0 = lo // 32
    flags = [f[w0:] for f in flags_full]  # bit 0 of word 0 = this shard's first row
    parts = _fold_local(hi - lo, words, mats_local, flags)
    if plan.world == 1:
        return parts
    return [xor_allreduce(p_, group) for p_ in parts]


def _compact(bits: torch.Tensor, n: int, k: int) -> torch.Tensor:
    """Indices of the set bits among the first n (device compaction, order kept)."""
    idx = torch.empty((max(n, 1),), dtype=torch.int32, device=bits.device)
    cnt = torch.empty((1,), dtype=torch.int64, device=bits.device)
    nb = int(_lib.load().ogm_compact_workspace_bytes(n))
    ws = torch.empty((nb,), dtype=torch.uint8, device=bits.device)
    _lib.call("ogm_compact_bits", n, _lib.ptr(bits), _lib.ptr(idx), _lib.ptr(cnt), _lib.ptr(ws), nb,
              _lib.stream_ptr())
    return idx[:k]


def sharded_keep(plain_local: torch.Tensor, plan: ShardPlan, rank: int, group=None):
    """Open + compaction over a row-sharded table (src/engine.py:243-252).

    plain_local = this rank's opened flag bits (packed, rows [lo, hi)).  The
    one exchange is the all-gather of the opened bits -- every party notes
    the whole opened vector anyway (src/rss.py:184-206) -- so each rank
    derives all shards' kept counts from it and the exclusive scan needs no
    further collective.  Kept rows keep the global shuffled order: shards
    are contiguous row ranges, so rank r's kept rows follow ranks < r.
    Returns (full opened vector on the host, this rank's kept local rows on
    the device, global position of its first kept row, global kept count)."""
    lo, hi = plan.bounds(rank)
    if any(b[0] % 32 and b[1] > b[0] for b in (plan.bounds(r) for r in range(plan.world))):
        raise ValueError("keep shards must start on 32-row word boundaries")
    full = all_gather_bits(plain_local, plan, group) if plan.world > 1 else plain_local
    host = full.cpu().numpy().view(np.uint32)
    bits = np.unpackbits(host.view(np.uint8), bitorder="little")[: plan.rows]
    counts = [int(bits[a:b].sum()) for a, b in (plan.bounds(r) for r in range(plan.world))]
    local = _compact(plain_local, hi - lo, counts[rank])
    return host, local, sum(counts[:rank]), sum(counts)


# ---------------------------------------------------------------------------
# Row-sharded 3-party shuffle ("global permutation -> all-to-all")
# ---------------------------------------------------------------------------
#
# Every online step of the shuffle is out[i] = M[k(i)] ^ B[i] (^ m3[i]) with
# k a permutation fixed offline (shuffle.ShuffleOffline).  Rows of M and out
# are sharded by ShardPlan.  All three parties live on every GPU, so every
# rank knows k and plans the exchange locally:
#   pack    send = M_local[send_idx]          (rows other ranks need from me,
#                                              grouped by destination rank)
#   a2a     recv = all_to_all(send)           (the step's only collective)
#   unpack  out  = recv[recv_pos] ^ B ^ m3    (B = this shard's combined blinds)
# pack/unpack are ogm_shuffle_gather launches; blinds for the shard come from
# the PRF with the shard's global row offset, so no blinding data moves.


@dataclass
class ExchangePlan:
    send_idx: torch.Tensor     # local source rows, grouped by destination rank
    send_splits: list
    recv_splits: list
    recv_pos: torch.Tensor     # position of out row i's source in the recv buffer


def exchange_plan(k_full: torch.Tensor, plan: ShardPlan, rank: int) -> ExchangePlan:
    """Offline index planning for out[i] = M[k_full[i]] on this rank's rows."""
    dev = k_full.device
    per = plan.per_rank
    lo, hi = plan.bounds(rank)

    def owner(x):
        return torch.clamp(x // per, max=plan.world - 1)

    src = k_full[lo:hi].long()
    own = owner(src)
    order = torch.argsort(own, stable=True)             # recv buffer order: by sender, then by i
    recv_pos = torch.empty_like(order)
    recv_pos[order] = torch.arange(order.numel(), device=dev)
    recv_splits = torch.bincount(own, minlength=plan.world).tolist() if order.numel() else [0] * plan.world
    sends, send_splits = [], []
    for s in range(plan.world):
        l2, h2 = plan.bounds(s)
        srcs = k_full[l2:h2].long()
        mine = srcs[owner(srcs) == rank] - lo
        sends.append(mine)
        send_splits.append(int(mine.numel()))
    send_idx = torch.cat(sends) if sends else torch.zeros(0, dtype=torch.long, device=dev)
    return ExchangePlan(send_idx.to(torch.int32), send_splits, recv_splits, recv_pos.to(torch.int32))


def _take(rows: int, width: int, src: torch.Tensor, idx: torch.Tensor, r=None, m3=None) -> torch.Tensor:
    """out[i] = src[idx[i]] ^ r[i] ^ m3[i] on the device (ogm_shuffle_gather)."""
    from .shuffle import gather
    out = torch.empty((rows, words_for(width)), dtype=torch.int32, device=src.device)
    if rows:
        gather(rows, width, out, inner=idx, m1=src, r=r, m3=m3)
    return out


def exchange_gather(m_local: torch.Tensor, xp: ExchangePlan, width: int, r=None, m3=None, group=None):
    send = _take(xp.send_idx.numel(), width, m_local, xp.send_idx)
    recv = torch.empty((sum(xp.recv_splits), send.shape[1]), dtype=send.dtype, device=send.device)
    as_comm(group).all_to_all(recv, send, xp.recv_splits, xp.send_splits)
    return _take(xp.recv_pos.numel(), width, recv, xp.recv_pos, r=r, m3=m3)


class ShardedTrioShuffle:
    """Offline material + online steps of one shuffle (table id ``tid``) for
    this rank's rows; the concatenation over ranks equals the single-GPU
    trio shuffle (trio.Trio.shuffle) bit for bit.

    At one rank the exchange is the identity, so the online phase IS the
    single-GPU one (shuffle.ShuffleOffline: the chained planned gathers for
    16-byte rows, planned gathers per step otherwise).  With more ranks each
    step is pack -> all-to-all -> unpack; when a rank's table is past
    PLAN_MIN_BYTES the pack and unpack gathers run planned (partition pass +
    window pass) like the single-GPU shuffle."""

    def __init__(self, seeds: tuple, tid: int, rows: int, width: int, plan: ShardPlan, rank: int, device=None):
        from .prf import seeded_permutation_device
        from .shuffle import (LABEL_BLIND, LABEL_PERM, LABEL_RAND, PLAN_MIN_BYTES, GatherPlan, ShuffleOffline,
                              compose, gather)
        s12, s23, s31 = seeds
        self.width, self.plan, self.rank = width, plan, rank
        dev = device or torch.device("cuda")
        pi12, pi23, pi31 = (seeded_permutation_device(s, LABEL_PERM, tid, rows, device=dev) for s in (s12, s23, s31))
        lo, hi = plan.bounds(rank)
        n = hi - lo
        self.lo, self.n = lo, n
        self.single = None
        if plan.world == 1:
            pc = {(s12, tid, rows): pi12, (s23, tid, rows): pi23, (s31, tid, rows): pi31}
            pairs = [(s12, s31), (s23, s12), (s31, s23)]
            self.single = [ShuffleOffline(p + 1, *pairs[p], tid, rows, width, device=dev, perm_cache=pc)
                           for p in range(3)]
            self.fast = words_for(width) == 4 and rows > 0
            if self.fast and self.single[0].plan_x1 is not None:
                for o in self.single:
                    o.chain_blinds()
            return
        k1, k3 = compose(pi31, pi12), compose(pi23, pi31)
        bt = (LABEL_BLIND, tid)

        def tab():
            return torch.empty((n, words_for(width)), dtype=torch.int32, device=dev)

        # this shard's combined blinds (destination-indexed), PRF at global rows
        self.u = gather(n, width, tab(), outer=pi31[lo:hi], inner=pi12, t1=(s12, *bt), t2=(s31, *bt))
        self.v = gather(n, width, tab(), inner=pi12[lo:hi], t1=(s12, *bt))
        self.w = gather(n, width, tab(), inner=pi23[lo:hi], t1=(s23, *bt), r=(s12, LABEL_RAND, tid), row0=lo)
        self.z = gather(n, width, tab(), outer=pi23[lo:hi], inner=pi31, t1=(s31, *bt), t2=(s23, *bt),
                        r=(s31, LABEL_RAND, tid), row0=lo)
        self.r1 = gather(n, width, tab(), r=(s31, LABEL_RAND, tid), row0=lo)
        self.r2 = gather(n, width, tab(), r=(s12, LABEL_RAND, tid), row0=lo)
        self.xp = {"x1": exchange_plan(k1, plan, rank), "y1": exchange_plan(pi12, plan, rank),
                   "c1": exchange_plan(pi23, plan, rank), "r3": exchange_plan(k3, plan, rank)}
        big = n * words_for(width) * 4 >= PLAN_MIN_BYTES
        self.plans = {}
        if big:   # local gathers over tables past L2: planned (partition + window passes)
            for k_, xp in self.xp.items():
                self.plans[k_] = (GatherPlan(xp.send_idx, words_for(width)) if xp.send_idx.numel() else None,
                                  GatherPlan(xp.recv_pos, words_for(width)) if xp.recv_pos.numel() else None)

    def _step(self, name: str, m_local, r=None, m3=None, group=None):
        xp = self.xp[name]
        pack, unpack = self.plans.get(name, (None, None))
        w = self.width
        if pack is None and unpack is None:
            return exchange_gather(m_local, xp, w, r=r, m3=m3, group=group)
        nw = words_for(w)
        send = torch.empty((xp.send_idx.numel(), nw), dtype=torch.int32, device=m_local.device)
        if pack is not None:
            pack.run(send, m1=m_local)
        recv = torch.empty((sum(xp.recv_splits), nw), dtype=torch.int32, device=m_local.device)
        as_comm(group).all_to_all(recv, send, xp.recv_splits, xp.send_splits)
        out = torch.empty((xp.recv_pos.numel(), nw), dtype=torch.int32, device=m_local.device)
        if unpack is not None:
            unpack.run(out, m1=recv, r=r, m3=m3)
        return out

    def online(self, comps: list, group=None) -> list:
        """comps: this rank's rows of the three components -> new components."""
        if self.single is not None:
            return self._online_single(comps)
        ab = torch.empty_like(comps[0])
        if ab.numel():
            _lib.call("ogm_xor_words", ab.numel(), _lib.ptr(comps[0]), _lib.ptr(comps[1]), None, _lib.ptr(ab),
                      _lib.stream_ptr())
        x1 = self._step("x1", ab, r=self.u, group=group)            # P1
        y1 = self._step("y1", comps[2], r=self.v, group=group)      # P2
        c1 = self._step("c1", x1, r=self.w, group=group)            # P2
        r3 = self._step("r3", y1, r=self.z, m3=c1, group=group)     # P3
        return [self.r1, self.r2, r3]

    def _online_single(self, comps: list) -> list:
        from .shuffle import shuffle_online_fused, shuffle_online_planned
        p1, p2, p3 = self.single
        a, b, c = comps
        r3 = torch.empty_like(a)
        if self.n == 0:
            return [p1.out_a, p1.out_b, r3]
        if self.fast and p1.plan_x1 is not None:
            shuffle_online_planned(self.single, a, b, c, r3)
        elif self.fast:
            shuffle_online_fused(self.single, a, b, c, torch.empty_like(a), torch.empty_like(a), None, r3)
        else:
            x1, y1, c1 = torch.empty_like(a), torch.empty_like(a), torch.empty_like(a)
            p1.step_x1(a, b, x1)
            p2.step_y1(c, y1)
            p2.step_c1(x1, c1)
            p3.step_r3(y1, c1, r3)
        return [p1.out_a, p1.out_b, r3]


__all__ = ["Comm", "DistComm", "ThreadComm", "as_comm", "ShardPlan", "pad_slice", "assemble", "all_gather_bits", "sharded_sec_eval_trio", "fold_indicators", "ExchangePlan",
           "exchange_plan", "exchange_gather", "ShardedTrioShuffle", "fss"]
