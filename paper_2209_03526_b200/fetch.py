"""Fetch of flagged 128-bit rows for the three co-resident parties
(src/engine.py:220-270, ``sec_fetch_multi`` with a 128-bit id and no
attributes -- the C5 fetch shape), in the flag-split layout.

The reference builds rows ``flag | id`` (129 bits, 5 words, src/engine.py:
227-237), shuffles them (src/shuffle.py:80-144), opens the flag column
(src/rss.py:184-206) and slices the kept rows' ids back out.  Here the rows
stay split -- the payload as aligned 16-byte rows, the flag as a bit column
-- because every shuffle step is a row permutation plus XORs of equally laid
out rows (csrc/ogm_fetch.cuh).  The blinds are drawn in the reference's
5-word layout and split offline (``ShuffleOffline(flag_split=True)``), so
the kept records are bit-identical to the reference's.

The flag column is composed across the parties' steps, as the payload's
flat hand-over composes them: each party's bit gather is folded into the
next party's (offline kc = k1 o pi23, kr = pi12 o k3 and the matching blind
columns), so the message bits x1f / y1f exist only in flight and the column
costs two random bit reads per row instead of four (ogm_flag_open_composed).

Online phase (what the C5 fetch bench times):
  1. up to 2^20 rows: ONE cooperative launch (ogm_fetch128_online_fused):
     the 16-byte three-party shuffle, whose second phase also gathers the
     composed flag column and writes the opened column; at 2^21 rows the
     cooperative shuffle, then the composed flag launch; from 2^22 rows: the
     chained planned payload shuffle, then the composed flag launch (plus
     f1 ^ f2, ogm_flag_open_composed); above
     256 MB tables ONE call (ogm_fetch128_online_planned): the payload
     shuffle whose split final window passes also compute the flag column
     and the opened column (they walk the rows in output order anyway);
  2. keep: hand-written compaction copying the kept payload rows of the
     three new components (ogm_keep_rows).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .bits import words_for
from .shuffle import (FLAG_ROW_BITS, FUSED_MAX_BYTES, ShuffleOffline, compose, flat_chain_args, run_table_args,
                      shuffle_online_fused, shuffle_online_planned)

# up to 16 MB tables the flag column rides the cooperative shuffle launch (measured 2^16 / 2^18 rows:
# 0.042 / 0.053 ms against 0.057 / 0.071 ms in two launches; even at 2^20, 2% slower at 2^21)
FUSED_FLAGS_MAX_BYTES = 16 << 20
FLAG_TAIL_MIN_BYTES = 256 << 20   # above: the flag column rides the split window passes


def bit_gather(col: torch.Tensor, idx: torch.Tensor, n: int) -> torch.Tensor:
    """Packed bit column out with bit i = bit idx[i] of ``col`` (little-endian
    int32 words; clean tail).  Offline only (chunked torch ops)."""
    nw = words_for(n)
    out = torch.zeros((max(nw, 1),), dtype=torch.int32, device=col.device)
    w64 = col.to(torch.int64) & 0xFFFFFFFF
    shifts = torch.arange(32, device=col.device, dtype=torch.int64)
    step = 1 << 22
    for s in range(0, n, step):
        j = idx[s:min(n, s + step)].to(torch.int64)
        b = (w64[j >> 5] >> (j & 31)) & 1
        b = torch.nn.functional.pad(b, (0, (-b.numel()) % 32))
        v = (b.view(-1, 32) << shifts).sum(1)
        out[s // 32:s // 32 + v.numel()] = torch.where(v >= 1 << 31, v - (1 << 32), v).to(torch.int32)
    return out


class FlaggedFetch:
    """Offline material and online phase of one fetch of ``rows`` flagged
    128-bit rows for table id ``tid``.  ``seeds`` = (s12, s23, s31), the
    pairwise seeds (party 1 holds s12 and s31, and so on)."""

    def __init__(self, seeds: tuple, tid: int, rows: int, device=None, perm_cache=None, plan: bool | None = None,
                 flag_tail: bool | None = None):
        s12, s23, s31 = seeds
        self.rows, self.tid = rows, tid
        self.dev = torch.device(device or "cuda")
        self.fused = rows * 16 <= FUSED_MAX_BYTES if plan is None else not plan
        pairs = [(s12, s31), (s23, s12), (s31, s23)]
        pc = {} if perm_cache is None else perm_cache
        self.off = [ShuffleOffline(p + 1, *pairs[p], tid, rows, FLAG_ROW_BITS, device=self.dev, perm_cache=pc,
                                   plan=not self.fused, flag_split=True) for p in range(3)]
        p1, p2, p3 = self.off
        if not self.fused:
            for o in self.off:
                o.chain_blinds()
            flat_chain_args(self.off)
            # the chained shuffle reads only its chain blinds (chain_blinds); the other copies go
            p1.u = p2.v = p3.z = None
            if not p2.w_output_order:
                p2.w = None
        # R1 / R2 are held once (P1's pair); P2's and P3's copies are the same tables
        p2.out_a = p3.out_b = None
        self.r1, self.r2 = p1.out_a, p1.out_b
        self.r1f, self.r2f = p1.flag["out_a"], p1.flag["out_b"]
        nw = words_for(rows)
        # the composed flag column (offline): c1 bits = f12[kc] ^ uwf, R3 bits = f3[kr] ^ vzf ^ c1 bits
        self.kc, self.kr = compose(p2.pi23, p1.k1), compose(p3.k3, p2.pi12)
        self.uwf = bit_gather(p1.flag["u"], p2.pi23, rows) ^ p2.flag["w"]
        self.vzf = bit_gather(p2.flag["v"], p3.k3, rows) ^ p3.flag["z"]

        def vec():
            return torch.empty((max(nw, 1),), dtype=torch.int32, device=self.dev)

        self.r3 = torch.empty((rows, 4), dtype=torch.int32, device=self.dev)
        self.f12, self.c1f, self.r3f, self.plain = vec(), vec(), vec(), vec()
        self.plans = None if self.fused else [p1.plan_x1, p2.plan_y1, p2.plan_c1, p3.plan_r3]
        # the flag column rides the final window passes only where they are split (> 256 MB)
        self.flag_tail = not self.fused and (rows * 16 > FLAG_TAIL_MIN_BYTES if flag_tail is None else flag_tail)
        self.inter = ([torch.empty_like(self.r3) for _ in range(3)] if not self.fused
                      else [torch.empty_like(self.r3) for _ in range(2)])
        self.outs = [torch.empty((max(rows, 1), 4), dtype=torch.int32, device=self.dev) for _ in range(3)]
        nb = int(_lib.load().ogm_keep_rows_workspace_bytes(rows))
        self.ws = torch.empty((nb,), dtype=torch.uint8, device=self.dev)
        self.count = torch.zeros((1,), dtype=torch.int64, device=self.dev)
        # the opened column's and the kept count's host copies (pinned: a pageable copy stages
        # through a bounce buffer and synchronises on its own)
        pin = self.dev.type == "cuda"
        self.plain_host = torch.empty((max(nw, 1),), dtype=torch.int32, pin_memory=pin)
        self.count_host = torch.zeros((1,), dtype=torch.int64, pin_memory=pin)

    def online(self, flags: list, payload: list) -> None:
        """The three parties' online fetch over component flags [f1, f2, f3]
        (packed bit vectors) and payloads [p1, p2, p3] ((rows, 4) int32):
        leaves the new components' flag column opened in ``plain``, the
        kept count in ``count`` (device) and the kept records' payload
        share components in ``outs`` (rows [0, count)).  No host sync."""
        rows = self.rows
        if rows == 0:
            self.count.zero_()
            return
        p1, p2, p3 = self.off
        a, b, c = payload
        for t in payload:
            if t.shape != (rows, 4) or not t.is_contiguous():
                raise ValueError("payload components must be contiguous (rows, 4) tables")
        P = _lib.ptr
        if self.fused and rows * 16 <= FUSED_FLAGS_MAX_BYTES:
            # one cooperative launch: the shuffle, the composed flag column and the open
            _lib.call("ogm_fetch128_online_fused", rows, P(p1.k1), P(p2.pi12), P(p2.pi23), P(p3.k3), P(a), P(b),
                      P(c), P(p1.u), P(p2.v), P(p2.w), P(p3.z), P(self.inter[0]), P(self.inter[1]), P(self.r3),
                      P(self.kc), P(self.kr), P(flags[0]), P(flags[1]), P(flags[2]), P(self.uwf), P(self.vzf),
                      P(self.r1f), P(self.r2f), P(self.f12), P(self.r3f), P(self.plain), _lib.stream_ptr())
        elif self.fused or not self.flag_tail:
            if self.fused:
                shuffle_online_fused(self.off, a, b, c, self.inter[0], self.inter[1], None, self.r3)
            else:
                shuffle_online_planned(self.off, a, b, c, self.r3, inter=self.inter)
            _lib.call("ogm_flag_open_composed", rows, P(self.kc), P(self.kr), P(flags[0]), P(flags[1]),
                      P(flags[2]), P(self.uwf), P(self.vzf), P(self.r1f), P(self.r2f), P(self.f12), None,
                      P(self.r3f), P(self.plain), _lib.stream_ptr())
        else:
            # one call: the chained payload shuffle whose final window passes also produce the
            # composed flag column and the opened column
            (u,), (v, _) = p1.chain_blinds(), p2.chain_blinds()
            arr = lambda xs: (ctypes.c_void_p * len(xs))(*[P(x) for x in xs])  # noqa: E731
            q2, gd, sr, it = (arr([pl.q2 for pl in self.plans]), arr([pl.gdst for pl in self.plans]),
                              arr([pl.srow for pl in self.plans]), arr(self.inter))
            qf, wf, w_order, zf, z_order, wr = flat_chain_args(self.off)
            qs = arr(qf)
            rs, ro, rn = run_table_args(self.plans)
            _lib.call("ogm_fetch128_online_planned", rows, ctypes.addressof(q2), ctypes.addressof(gd),
                      ctypes.addressof(sr), ctypes.addressof(qs), rs, ro, rn, wr, P(a), P(b), P(c),
                      P(u), P(v), P(wf), w_order, P(zf), z_order, ctypes.addressof(it), P(self.r3),
                      P(self.kc), P(self.kr),
                      P(flags[0]), P(flags[1]), P(flags[2]), P(self.uwf), P(self.vzf), P(self.r1f), P(self.r2f),
                      P(self.f12), P(self.c1f), P(self.r3f), P(self.plain), _lib.stream_ptr())
        mats = (ctypes.c_void_p * 3)(P(self.r1), P(self.r2), P(self.r3))
        outs = (ctypes.c_void_p * 3)(*[P(o) for o in self.outs])
        _lib.call("ogm_keep_rows", rows, P(self.plain), 3, ctypes.addressof(mats), 4, ctypes.addressof(outs), 4,
                  None, P(self.count), P(self.ws), self.ws.numel(), _lib.stream_ptr())

    def opened_host(self) -> tuple:
        """(the opened flag column as uint32 words, the kept count) on the
        host, both copied in one synchronisation of the current stream."""
        nw = words_for(self.rows)
        self.plain_host[:nw].copy_(self.plain[:nw], non_blocking=True)
        self.count_host.copy_(self.count, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        return self.plain_host[:nw].numpy().view(np.uint32), int(self.count_host[0])

    def components(self) -> list:
        """The shuffled table's new components (R1, R2, R3): payload tables
        and flag columns, [(payload, flag bits)] * 3."""
        return [(self.r1, self.r1f), (self.r2, self.r2f), (self.r3, self.r3f)]

    def kept(self) -> int:
        """Host copy of the kept count (one synchronisation)."""
        return int(self.count.item())

    def records(self) -> list:
        """[c1, c2, c3]: the kept rows' payload share components, (k, 4) each."""
        k = self.kept()
        return [o[:k] for o in self.outs]
