"""Multi-GPU sec_match: the trio fast path over row-sharded type tables
(src/engine.py:352-417 orchestrated across ranks).

Every type's tables -- one-hot ids, attribute one-hots, posting tensors --
are partitioned by vertex-id ranges (``ShardPlan``, multiples of 128 rows so
every shard's packed bits start on an AES-CTR block of the zero-share
stream).  All three logical servers live on every rank, so party messages
never cross NVLink; the only exchanges are the collectives below.  Every
rank runs the same schedule and consumes zero-share counters, table ids and
open labels exactly like the single-GPU ``Trio`` -- results are
bit-identical to it (and to the reference), on every rank:

  step                              touches             exchange
  root secEval (per predicate)      root rows (shard)   one all-gather of the packed blinded bits
  combine                           match bits (full)   none (every rank computes it)
  Case I fold (unique route)        root rows (shard)   XOR all-reduce of the partial folds
  Case II fetch: shuffle            root rows (shard)   one all-to-all per shuffle step
                 open + keep        shuffled rows       all-gather of the opened bits; kept records all-gathered
  sec_access posting fold           parent rows (shard) XOR all-reduce (L_max x w(X_ne) words)
  child groups (secEval, fetch)     the group (small)   none (replicated)
  GF(2) attribute select-many       child rows (shard)  XOR all-reduce (K x w(n) words)

``local_shards`` cuts this rank's views out of full device shares (tests and
single-host runs); a deployment loads only its rows.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .bits import BitVector, rows2d, words_for
from .graphs import GraphShare, TypePartyShare
from .sharding import (Comm, ShardedTrioShuffle, ShardPlan, as_comm, sec_eval_local_packed, assemble_many,
                       sharded_fold_trio, sharded_keep, xor_allreduce)
from .trio import PackedRows, Trio, TrioGroup, TrioRecords, _nxt

A = _lib.ptr_array


def type_plans(schema, world: int) -> dict:
    """One ShardPlan per vertex type (rows = the type's population)."""
    return {t: ShardPlan(ts.population, world) for t, ts in schema.types.items()}


def local_shards(gshares: list, world: int, rank: int) -> list:
    """This rank's rows of every type table of the three party shares (views)."""
    plans = type_plans(gshares[0].schema, world)
    out = []
    for gs in gshares:
        types = {}
        for t, s in gs.types.items():
            lo, hi = plans[t].bounds(rank)
            types[t] = TypePartyShare(s.id_a[lo:hi], s.id_b[lo:hi],
                                      {n: (p[0][lo:hi], p[1][lo:hi]) for n, p in s.attrs.items()},
                                      {n: (p[0][lo:hi], p[1][lo:hi]) for n, p in s.posting.items()})
        out.append(GraphShare(gs.party_index, gs.schema, types))
    return out


@dataclass
class ShardedGroup(TrioGroup):
    """A candidate group whose rows are this rank's shard of a type table."""

    plan: ShardPlan = field(default=None)
    rank: int = 0


class ShardedTrio(Trio):
    """Trio over row-sharded tables; ``comm`` is a sharding.Comm (or a
    torch.distributed process group / None for the default group)."""

    def __init__(self, master: bytes | None = None, comm: Comm | None = None, configs=None, device=None):
        super().__init__(master, configs, device)
        self.comm = as_comm(comm)
        self.world, self.rank = self.comm.world, self.comm.rank

    # -- root group ---------------------------------------------------------
    def _root_group(self, gshares: list, vtype: str, ts, needed: list) -> TrioGroup:
        tps = [gs.types[vtype] for gs in gshares]
        plan = ShardPlan(ts.population, self.world)
        return ShardedGroup(None, None, ts.population, ts.population, [t.id_a for t in tps],
                            {a: [t.attrs[a][0] for t in tps] for a in needed},
                            {a: ts.attrs[a].domain_size for a in needed}, plan=plan, rank=self.rank)

    # -- secEval: local rows, one all-gather --------------------------------
    def sec_eval(self, group: TrioGroup, key_pairs: list, attr: str, domain: int, cache: dict) -> list:
        if not isinstance(group, ShardedGroup):
            return super().sec_eval(group, key_pairs, attr, domain, cache)
        rows6 = self._pass_indicators(key_pairs, domain, cache)
        npass = len(rows6)
        fold = npass == 2   # one parity pass over the folded indicators (Trio._folded_indicators)
        if fold:
            rows6 = [self._folded_indicators(key_pairs, domain, cache)]
        inds = [[(r[2 * q], r[2 * q + 1]) for q in range(3)] for r in rows6]
        comps = group.attrs[attr]
        zk = [(k, None) for k in self.k]
        counters = [self.counter + ps for ps in range(npass)]
        packed = sec_eval_local_packed(comps, comps[0].shape[1], group.plan, self.rank, inds, zk, counters,
                                       fold=fold)
        self.counter += npass
        nvec, wpr = packed.shape
        if self.world == 1:
            full = [packed[j][: group.plan.total_words] for j in range(nvec)]
        else:
            full = assemble_many(self.comm.all_gather(packed).view(self.world, nvec, wpr), group.plan)
        result = None
        for ps in range(nvec // 3):
            b = full[3 * ps: 3 * ps + 3]
            shared = [b[2].contiguous(), b[0].contiguous(), b[1].contiguous()]   # comp j := blinded_{j-1}
            result = shared if result is None else self.xor(result, shared)
        return result

    # -- Case I: local fold, XOR all-reduce, re-share ------------------------
    def fetch_unique(self, group: TrioGroup, flags: list) -> TrioRecords:
        if not isinstance(group, ShardedGroup):
            return super().fetch_unique(group, flags)

        def fold(mats, width):
            parts = sharded_fold_trio([rows2d(m) for m in mats], flags, group.plan, self.rank, self.comm)
            return self.reshare(parts, width)

        ids = fold(group.ids, group.id_width)
        attrs = {n: fold(group.attrs[n], group.attr_widths[n]) for n in sorted(group.attrs)}
        return TrioRecords(group.parent_slot, group.parent_record, 1, group.id_width, [c[None] for c in ids],
                           {a: [c[None] for c in v] for a, v in attrs.items()}, dict(group.attr_widths))

    # -- Case II: sharded shuffle, open, keep, records all-gathered ----------
    def fetch_multi(self, group: TrioGroup, flags: list, audit: list, online_blinds=None) -> TrioRecords:
        if not isinstance(group, ShardedGroup):
            return super().fetch_multi(group, flags, audit, online_blinds)
        plan, rank = group.plan, self.rank
        lo, hi = plan.bounds(rank)
        n = hi - lo
        names = sorted(group.attrs)
        widths = [group.attr_widths[a] for a in names]
        row_width = 1 + group.id_width + sum(widths)
        w = words_for(row_width)
        fl = [f[lo // 32:] for f in flags]   # bit 0 = this shard's first row (lo is 128-aligned)
        pr = PackedRows(n, row_width, fl, [(group.ids, group.id_width)] + [(group.attrs[a], wd)
                                                                        for a, wd in zip(names, widths)])
        comps = [self.pack_gather(pr, (c,))[:, :w].contiguous() for c in range(3)]
        tid = self.table_id
        self.table_id += 1
        sh = ShardedTrioShuffle((self.s12, self.s23, self.s31), tid, plan.rows, row_width, plan, rank,
                                device=self.dev)
        new = sh.online(comps, self.comm)
        # open the flag column (bit 0 of word 0): plain = R1 ^ R2 ^ R3 on this shard's rows
        self.label += 1
        x = torch.empty_like(new[0])
        plain = self._empty(words_for(n))
        if n:
            _lib.call("ogm_xor_words", x.numel(), _lib.ptr(new[0]), _lib.ptr(new[1]), _lib.ptr(new[2]),
                      _lib.ptr(x), _lib.stream_ptr())
            _lib.call("ogm_column_bits", _lib.ptr(x), w, n, _lib.ptr(plain), _lib.stream_ptr())
        host, local_idx, first, total = sharded_keep(plain, plan, rank, self.comm)
        opened = BitVector(host[: words_for(plan.rows)], plan.rows)
        self.opened.append((self.label, opened))
        bits = opened.to_bits()
        audit.append(("fetch", bits))
        # this shard's kept rows, sliced into fields, then every shard's kept records in shard order
        k_local = local_idx.numel()
        fields = [(1, group.id_width)]
        off = 1 + group.id_width
        for wd in widths:
            fields.append((off, wd))
            off += wd
        counts = [int(bits[a:b].sum()) for a, b in (plan.bounds(r) for r in range(self.world))]
        kmax = max(counts) if counts else 0
        got = []
        for bo, fw in fields:
            fwd = words_for(fw)
            per = []
            for c in range(3):
                if total == 0:   # every rank knows the count: no collective
                    per.append(torch.zeros((0, fwd), dtype=torch.int32, device=self.dev))
                    continue
                mine = torch.zeros((kmax, fwd), dtype=torch.int32, device=self.dev)
                if k_local:
                    _lib.call("ogm_extract_field", _lib.ptr(new[c]), w, _lib.ptr(local_idx), k_local, bo, fw,
                              _lib.ptr(mine), fwd, _lib.stream_ptr())
                allr = (self.comm.all_gather(mine).view(self.world, kmax, fwd) if self.world > 1
                        else mine.view(1, kmax, fwd))
                per.append(torch.cat([allr[r, : counts[r]] for r in range(self.world)]))
            got.append(per)
        return TrioRecords(group.parent_slot, group.parent_record, total, group.id_width, got[0],
                           dict(zip(names, got[1:])), dict(zip(names, widths)))

    # -- sec_access: posting fold and select-many over sharded tables --------
    def access(self, rec: TrioRecords, i: int, parent_type: str, child_type: str, needed: list, gshares: list,
               provenance: tuple, audit: list) -> TrioGroup:
        schema = gshares[0].schema
        parent_slot, parent_rec = provenance
        x_ne = schema.types[child_type].population
        w_ne = words_for(x_ne)
        widths = {a: schema.types[child_type].attrs[a].domain_size for a in needed}
        lists = [gs.types[parent_type].posting[child_type][0] for gs in gshares]
        l_max = lists[0].shape[1]

        def empty():
            z = lambda wd: torch.zeros((0, wd), dtype=torch.int32, device=self.dev)  # noqa: E731
            return TrioGroup(parent_slot, parent_rec, 0, x_ne, [z(w_ne)] * 3,
                             {a: [z(words_for(widths[a]))] * 3 for a in needed}, widths)

        if l_max == 0:
            return empty()
        pplan = ShardPlan(schema.types[parent_type].population, self.world)
        sel = [c[i].contiguous() for c in rec.ids]
        parts = sharded_fold_trio([rows2d(m) for m in lists], sel, pplan, self.rank, self.comm)
        fetched = self.reshare_matrix([p_.reshape(l_max, w_ne) for p_ in parts], x_ne)
        rows = PackedRows(l_max, 1 + x_ne, self._parity_rows(fetched, w_ne), [(fetched, x_ne)])
        sh = self.shuffle(rows, 1 + x_ne)
        k, got = self._open_keep(sh, l_max, "access", audit, [(1, x_ne)])
        if k == 0:
            return empty()
        ids = got[0]
        cplan = ShardPlan(x_ne, self.world)
        lo, hi = cplan.bounds(self.rank)
        attrs = {}
        for a in needed:
            va = [gs.types[child_type].attrs[a][0] for gs in gshares]   # this rank's child rows
            wd = va[0].shape[1]
            adds = []
            for q in range(3):
                out = torch.zeros((k, wd), dtype=torch.int32, device=self.dev)
                nloc = hi - lo
                if nloc:
                    ws = torch.empty((2 * nloc,), dtype=torch.int32, device=self.dev)
                    sa, sb = ids[q][:, lo // 32:], ids[_nxt(q)][:, lo // 32:]
                    _lib.call("ogm_select_many", k, nloc, wd, va[q].stride(0), _lib.ptr(sa), _lib.ptr(sb),
                              ids[q].stride(0), _lib.ptr(va[q]), _lib.ptr(va[_nxt(q)]), _lib.ptr(out), wd,
                              _lib.ptr(ws), _lib.stream_ptr())
                adds.append(xor_allreduce(out, self.comm) if self.world > 1 else out)
            attrs[a] = self.reshare_matrix(adds, widths[a])
        return TrioGroup(parent_slot, parent_rec, k, x_ne, ids, attrs, widths)

    def match(self, tokens: list, gshares: list, any_mode: str = "or", native: bool = False):
        """src/engine.py:352-417 over this rank's shards (``gshares`` from
        local_shards); the Python schedule with the sharded steps above."""
        return super().match(tokens, gshares, any_mode, native=False)


def run_emulated(world: int, fn, device=None) -> list:
    """Run ``fn(comm)`` for ``world`` emulated ranks on one device (threads,
    ThreadComm); returns the per-rank results.  For tests."""
    import threading

    from .sharding import ThreadComm

    hub = ThreadComm(world)
    results: list = [None] * world
    errors: list = [None] * world
    dev = torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())

    def run(r):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(torch.cuda.Stream(dev)):
                results[r] = fn(hub.rank_view(r))
                torch.cuda.current_stream().synchronize()
        except BaseException as exc:  # noqa: BLE001
            errors[r] = exc
            hub._barrier.abort()

    threads = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    real = [e for e in errors if e is not None and not isinstance(e, threading.BrokenBarrierError)]
    if real or any(errors):
        raise (real or [e for e in errors if e is not None])[0]
    return results


__all__ = ["ShardedTrio", "ShardedGroup", "local_shards", "type_plans", "run_emulated", "np"]
