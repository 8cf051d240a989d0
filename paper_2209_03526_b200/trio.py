"""Trio fast path: the three co-resident servers stepped together in ONE host thread.

The drop-in API (engine.py + net.run_trio) runs each party on its own thread
exactly like the reference.  When the three logical servers share a GPU
(BASELINE: "the three logical servers' states are simulated on the same
devices"), every protocol step can instead be issued once for all three
parties:

* each share component lives once in HBM and is read once per step
  (party q's view is (x_q, x_{q+1}), src/graphs.py:382-399);
* one launch serves the three parties (``nparty=3`` kernels, zero shares
  for all three from 3 AES streams instead of 6);
* a re-share is a relabelling: party q's new pair is (blinded_{q-1},
  blinded_q), so component j of the result is blinded_{j-1} -- the message
  "sent" to the next party is the very tensor it receives;
* one host synchronisation per public value (opened counts), nothing else.

Randomness is consumed in the same order as the per-party path (zero-share
counter per re-share, table id per shuffle, open label per open; SURVEY
Appendix A.6), so outputs are bit-identical to ``run_trio(sec_match)`` --
tested against the reference's recorded runs.  Each party's computation is
unchanged; only the scheduling is fused.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib, fss
from .bits import BitVector, rows2d, words_for
from .engine import MatchedRecord, MatchResultSet, _assemble
from .net import make_session_configs
from .rss import DBits, SharedBitVector
from .shuffle import LABEL_BLIND, LABEL_RAND, _perm, blind_table, compose, gather

A = _lib.ptr_array


def _nxt(q: int) -> int:
    return (q + 1) % 3


def _pitch(width: int) -> int:
    """16-byte row pitch of the trio path's match tables (zero padding)."""
    return (words_for(width) + 3) // 4 * 4


def _as_pitched(m: torch.Tensor, width: int) -> torch.Tensor:
    """A (rows, pitch) buffer holding m's logical (rows, words) content."""
    p = _pitch(width)
    if m.dim() == 2 and m.shape[1] == p and m.is_contiguous():
        return m
    out = torch.zeros((m.shape[0], p), dtype=m.dtype, device=m.device)
    out[:, :words_for(width)] = m[:, :words_for(width)]
    return out


@dataclass
class PackedRows:
    """The three share components of a match table (src/engine.py:227-233:
    flag bit, then each field at its logical width), described by their
    fields instead of materialised.  The shuffle packs them inside its first
    gathers (ogm_pack_gather), so the packed rows never round-trip HBM."""

    rows: int
    width: int
    flags: list | None            # [f1, f2, f3] bit vectors, or None (no flag bit)
    fields: list                  # [([x1, x2, x3], width), ...]


@dataclass
class TrioGroup:
    """Candidate group with its three share components per field."""

    parent_slot: int | None
    parent_record: int | None
    count: int
    id_width: int
    ids: list                     # [x1, x2, x3] (count, words)
    attrs: dict                   # name -> [x1, x2, x3]
    attr_widths: dict


@dataclass
class TrioRecords:
    """A batch of matched records (rows of the component matrices)."""

    parent_slot: int | None
    parent_record: int | None
    count: int
    id_width: int
    ids: list
    attrs: dict
    attr_widths: dict


def one_hot_rows(x: np.ndarray, shapes: list) -> list:
    """Decode reconstructed one-hot rows (src/bits.py hot_index, as
    src/engine.py:458-500 applies it per record) for many fields at once:
    ``x`` holds the fields' (rows, words) uint32 matrices back to back, row
    major, ``shapes`` their shapes.  Per field, a list with the set bit's
    index per row (None for an all-zero row); a row with more than one bit set
    raises, naming the first such row's weight (fields in order)."""
    counts = [int(r) for r, _ in shapes]
    widths = np.repeat(np.array([int(w) for _, w in shapes], np.int64), counts)
    nrows = widths.size
    hot = np.full(nrows, -1, np.int64)
    pos = np.flatnonzero(widths > 0)              # rows that own words
    if pos.size and x.size:
        starts = np.zeros(nrows, np.int64)
        np.cumsum(widths[:-1], out=starts[1:])
        st = starts[pos]                          # strictly increasing; the last row ends at x's end
        weight = np.add.reduceat(np.bitwise_count(x), st, dtype=np.int64)
        bad = weight > 1
        if bad.any():
            raise ValueError(f"expected Hamming weight <= 1, got {int(weight[bad][0])}")
        nz = np.flatnonzero(x)                    # at most one set word per row
        r = np.searchsorted(st, nz, side="right") - 1
        v = x[nz]
        hot[pos[r]] = (nz - st[r]) * 32 + np.bitwise_count(v - np.uint32(1))
    flat = hot.tolist()
    out, o = [], 0
    for c in counts:
        out.append([None if h < 0 else h for h in flat[o:o + c]])
        o += c
    return out


@dataclass
class TrioResult:
    structure: dict
    records: list                 # per slot: list of (TrioRecords, row)
    subgraphs: list
    opened_flags: list = field(default_factory=list)

    def open(self, schema):
        """engine.open_results(self.party_results()[:2], schema) -- the same
        (matches, details) -- straight from the record batches: ONE
        device-to-host copy of every batch matrix of the three components, then
        one XOR and one one-hot decoding for every batch at once (one_hot_rows;
        src/engine.py:458-500)."""
        slots = self.structure["slots"]
        order, mats = [], [[], [], []]
        for s, slot in enumerate(slots):
            names = sorted({p["attr"] for p in slot["preds"]})
            seen = {}
            for batch, _ in self.records[s]:
                if id(batch) in seen:
                    continue
                seen[id(batch)] = batch
                fields = [("id", batch.ids, batch.id_width)] + [(a, batch.attrs[a], batch.attr_widths[a])
                                                                 for a in names]
                for name, comps, width in fields:
                    order.append((s, id(batch), name, comps[0].shape))
                    for q in range(3):
                        mats[q].append(comps[q].reshape(-1))
        # component-major: every field of component 0, then 1, then 2 -- one XOR for all fields
        host = (torch.cat(mats[0] + mats[1] + mats[2]).cpu().numpy().view(np.uint32) if mats[0]
                else np.zeros(0, np.uint32))
        h = host.reshape(3, -1)
        hots = one_hot_rows(h[0] ^ h[1] ^ h[2], [sh for *_, sh in order])
        plain = {(s, bid, name): hot for (s, bid, name, _), hot in zip(order, hots)}
        decoded = []
        for s, slot in enumerate(slots):
            ts = schema.types[slot["type"]]
            names = sorted({p["attr"] for p in slot["preds"]})
            out = []
            for batch, i in self.records[s]:
                hot = plain[(s, id(batch), "id")][i]
                attrs = {}
                for a in names:
                    idx = plain[(s, id(batch), a)][i]
                    attrs[a] = None if idx is None else ts.attrs[a].values[idx]
                out.append((None if hot is None else ts.ext_ids[hot], attrs))
            decoded.append(out)
        matches, details = [], []
        for combo in self.subgraphs:
            ids = tuple(decoded[s][ri][0] for s, ri in enumerate(combo))
            if any(v is None for v in ids):
                continue
            matches.append(ids)
            details.append([decoded[s][ri] for s, ri in enumerate(combo)])
        return matches, details

    def party_results(self) -> list:
        """Per-party MatchResultSet views (same layout as engine.sec_match)."""
        views: dict = {}

        def rows_of(mats):   # every component's row views, one unbind per matrix
            r = views.get(id(mats))
            if r is None:
                r = views[id(mats)] = [m.unbind(0) for m in mats]
            return r

        out = []
        for q in range(3):
            recs = []
            for slot in self.records:
                lst = []
                for batch, i in slot:
                    def sv(c, width):
                        r = rows_of(c)
                        return SharedBitVector(q + 1, DBits(r[q][i], width), DBits(r[_nxt(q)][i], width))
                    lst.append(MatchedRecord(batch.parent_slot, batch.parent_record, sv(batch.ids, batch.id_width),
                                             {a: sv(batch.attrs[a], batch.attr_widths[a]) for a in batch.attrs}))
                recs.append(lst)
            mrs = MatchResultSet(q + 1, self.structure, recs, self.subgraphs, list(self.opened_flags))
            mrs._trio = self   # engine.open_results reconstructs from the batches when all parties share it
            out.append(mrs)
        return out


class Trio:
    """Session state of the three co-resident parties (src/net.py:221-289)."""

    def __init__(self, master: bytes | None = None, configs=None, device=None):
        configs = sorted(configs or make_session_configs(master), key=lambda c: c.party_index)
        self.k = [c.zero_key_own for c in configs]          # k1, k2, k3
        self.s12 = configs[0].seed_with_next
        self.s23 = configs[1].seed_with_next
        self.s31 = configs[2].seed_with_next
        self.counter = 0          # zero-share counter (lockstep across parties)
        self.table_id = 0
        self.label = 0
        self.opened: list = []
        self.dev = torch.device(device or "cuda")

    # -- RSS ----------------------------------------------------------------
    def _empty(self, n: int) -> torch.Tensor:
        return torch.empty((max(n, 1),), dtype=torch.int32, device=self.dev)[:n]

    def reshare(self, adds: list, nbits: int) -> list:
        """src/rss.py:164-176 for all parties: comp j := blinded_{j-1}."""
        outs = [torch.empty_like(a) for a in adds]
        if nbits:
            _lib.call("ogm_zero_share_trio", self.k[0], self.k[1], self.k[2], self.counter, nbits, A(adds), A(outs),
                      _lib.stream_ptr())
        self.counter += 1
        return [outs[2], outs[0], outs[1]]

    def reshare_matrix(self, adds: list, width: int) -> list:
        """src/engine.py:83-92 for all parties (rows*w*32-bit zero share, row tails masked)."""
        rows, w = adds[0].shape
        flat = [a.reshape(-1) for a in adds]
        outs = [torch.empty_like(f) for f in flat]
        if rows * w:
            _lib.call("ogm_zero_share_trio_rows", self.k[0], self.k[1], self.k[2], self.counter, rows, w, width,
                      A(flat), A(outs), _lib.stream_ptr())
        self.counter += 1
        outs = [o.reshape(rows, w) for o in outs]
        return [outs[2], outs[0], outs[1]]

    def xor(self, a: list, b: list) -> list:
        out = []
        for x, y in zip(a, b):
            o = torch.empty_like(x)
            _lib.call("ogm_xor_words", x.numel(), _lib.ptr(x), _lib.ptr(y), None, _lib.ptr(o), _lib.stream_ptr())
            out.append(o)
        return out

    def and_gate(self, a: list, b: list, nbits: int) -> list:
        """src/rss.py:115-126,179-181 for all parties in one launch."""
        outs = [torch.empty_like(x) for x in a]
        _lib.call("ogm_and_terms", a[0].numel(), 3, A(a), A([a[_nxt(q)] for q in range(3)]), A(b),
                  A([b[_nxt(q)] for q in range(3)]), A(outs), _lib.stream_ptr())
        return self.reshare(outs, nbits)

    def open(self, comps: list, n: int) -> torch.Tensor:
        """src/rss.py:184-206: plain = x1 ^ x2 ^ x3; every party notes it."""
        self.label += 1
        plain = torch.empty_like(comps[0])
        _lib.call("ogm_xor_words", plain.numel(), _lib.ptr(comps[0]), _lib.ptr(comps[1]), _lib.ptr(comps[2]),
                  _lib.ptr(plain), _lib.stream_ptr())
        host = BitVector(plain, n)
        self.opened.append((self.label, host))
        return plain, host

    # -- shuffle --------------------------------------------------------------
    def prepare_shuffle(self, rows: int, width: int) -> None:
        """Offline phase for the NEXT shuffle (table id self.table_id): the
        data-independent permutations, their compositions and the permuted,
        combined blinding tables (see shuffle.ShuffleOffline)."""
        tid = self.table_id
        s12, s23, s31 = self.s12, self.s23, self.s31
        pi12, pi23, pi31 = _perm(s12, tid, rows), _perm(s23, tid, rows), _perm(s31, tid, rows)
        m = self._material(tid, rows, width, pi12, pi23, pi31)
        if not hasattr(self, "_prepared"):
            self._prepared = {}
        self._prepared[(tid, rows, width)] = m

    def _material(self, tid: int, rows: int, width: int, pi12, pi23, pi31) -> dict:
        """The data-independent blinds of one shuffle, permuted and combined
        along each party's gather path (shuffle.ShuffleOffline):
        U = T12[k1] ^ T31[pi31], V = T12[pi12], W = T23[pi23] ^ R2,
        Z = T31[k3] ^ T23[pi23] ^ R1, plus R1, R2.  Narrow rows generate the
        T rows inside the gathers (a 16-B row is one AES block); wide rows
        generate each table once at the AES rate (ogm_prf_rows) and combine
        whole rows with streaming gathers."""
        s12, s23, s31 = self.s12, self.s23, self.s31
        P = _pitch(width)

        def tab():
            return torch.empty((rows, P), dtype=torch.int32, device=self.dev)

        m = {"pi12": pi12, "pi23": pi23, "k1": compose(pi31, pi12), "k3": compose(pi23, pi31)}
        if words_for(width) >= 64:
            def table(seed, label):
                return blind_table(seed, label, tid, rows, width, self.dev, pitch=P)

            t12, t31, t23 = table(s12, LABEL_BLIND), table(s31, LABEL_BLIND), table(s23, LABEL_BLIND)
            m["r1"], m["r2"] = table(s31, LABEL_RAND), table(s12, LABEL_RAND)
            m["u"] = gather(rows, width, tab(), outer=pi31, inner=pi12, t1=t12, t2=t31)
            m["v"] = gather(rows, width, tab(), inner=pi12, t1=t12)
            m["w"] = gather(rows, width, tab(), inner=pi23, t1=t23, r=m["r2"])
            m["z"] = gather(rows, width, tab(), outer=pi23, inner=pi31, t1=t31, t2=t23, r=m["r1"])
            return m
        bt = (LABEL_BLIND, tid)
        m["u"] = gather(rows, width, tab(), outer=pi31, inner=pi12, t1=(s12, *bt), t2=(s31, *bt))
        m["v"] = gather(rows, width, tab(), inner=pi12, t1=(s12, *bt))
        m["w"] = gather(rows, width, tab(), inner=pi23, t1=(s23, *bt), r=(s12, LABEL_RAND, tid))
        m["z"] = gather(rows, width, tab(), outer=pi23, inner=pi31, t1=(s31, *bt), t2=(s23, *bt),
                        r=(s31, LABEL_RAND, tid))
        m["r1"] = gather(rows, width, tab(), r=(s31, LABEL_RAND, tid))
        m["r2"] = gather(rows, width, tab(), r=(s12, LABEL_RAND, tid))
        return m

    def shuffle(self, comps: list, width: int, online_blinds: bool | None = None) -> list:
        """src/shuffle.py:80-144 for the three parties: each permutation and
        blinding table generated once; composed gathers as in ShuffleOffline.
        ``online_blinds`` generates the blinding tables inside the gathers
        (AES-CTR on the fly) instead of materialising them -- the memory-lean
        mode for wide rows (default: on for tables above 4 GiB)."""
        if isinstance(comps, PackedRows):
            rows = comps.rows
        else:
            rows = comps[0].shape[0]
            comps = [_as_pitched(c, width) for c in comps]
        tid = self.table_id
        self.table_id += 1
        prep = getattr(self, "_prepared", {}).pop((tid, rows, width), None)
        if prep is not None:
            return self._shuffle_online(comps, width, prep)
        if online_blinds is None:
            online_blinds = rows * words_for(width) * 4 > (4 << 30)
        if not online_blinds:
            return self._shuffle_native(comps, rows, width, tid)
        # memory-lean mode: blinding rows generated inside the gathers
        s12, s23, s31 = self.s12, self.s23, self.s31
        pi12, pi23, pi31 = _perm(s12, tid, rows), _perm(s23, tid, rows), _perm(s31, tid, rows)

        def tab():
            return torch.empty((rows, _pitch(width)), dtype=torch.int32, device=self.dev)

        bt = (LABEL_BLIND, tid)
        ab = self._xor01(comps)
        x1 = gather(rows, width, tab(), outer=pi31, inner=pi12, m1=ab, t1=(s12, *bt), t2=(s31, *bt))
        del ab
        c3 = self.pack_gather(comps, (2,)) if isinstance(comps, PackedRows) else comps[2]
        y1 = gather(rows, width, tab(), inner=pi12, m1=c3, t1=(s12, *bt))
        del c3
        c1 = gather(rows, width, tab(), inner=pi23, m1=x1, t1=(s23, *bt), r=(s12, LABEL_RAND, tid))
        del x1
        r3 = gather(rows, width, tab(), outer=pi23, inner=pi31, m1=y1, t1=(s31, *bt), t2=(s23, *bt), m3=c1,
                    r=(s31, LABEL_RAND, tid))
        del y1, c1
        r1 = blind_table(s31, LABEL_RAND, tid, rows, width, self.dev, pitch=_pitch(width))
        r2 = blind_table(s12, LABEL_RAND, tid, rows, width, self.dev, pitch=_pitch(width))
        return [r1, r2, r3]

    def _shuffle_native(self, comps, rows: int, width: int, tid: int) -> list:
        """The whole shuffle (material + four online steps) in one
        ogm_trio_shuffle call: the same launches as _material +
        _shuffle_online, without ~25 host dispatches."""
        P = _pitch(width)
        if isinstance(comps, PackedRows):
            fields = list(comps.fields)
            flags = comps.flags
        else:
            fields = [(comps, width)]
            flags = None
        nf = len(fields)
        mats = [fields[f][0][c] for c in range(3) for f in range(nf)]
        pitches = [m.stride(0) if m.dim() == 2 else words_for(fields[f][1])
                   for m, f in zip(mats, [f for _ in range(3) for f in range(nf)])]
        out = [torch.empty((rows, P), dtype=torch.int32, device=self.dev) for _ in range(3)]
        lib = _lib.load()
        nb = int(lib.ogm_trio_shuffle_workspace_bytes(rows, P))
        ws = self.__dict__.get("_shuffle_ws")
        if ws is None or ws.numel() < nb:
            ws = self._shuffle_ws = torch.empty((nb,), dtype=torch.uint8, device=self.dev)
        _lib.call("ogm_trio_shuffle", self.s12, self.s23, self.s31, tid, rows, width, P, nf, A(mats),
                  _lib.i64_array(pitches), _lib.i64_array([w for _, w in fields]), A(flags) if flags else None,
                  A(out), _lib.ptr(ws), nb, _lib.stream_ptr())
        return out

    def _xor01(self, comps) -> torch.Tensor:
        if isinstance(comps, PackedRows):
            return self.pack_gather(comps, (0, 1))
        ab = torch.empty_like(comps[0])
        _lib.call("ogm_xor_words", ab.numel(), _lib.ptr(comps[0]), _lib.ptr(comps[1]), None, _lib.ptr(ab),
                  _lib.stream_ptr())
        return ab

    def pack_gather(self, pr: PackedRows, sets: tuple, idx=None, r=None) -> torch.Tensor:
        """XOR over components `sets` of the packed rows, at source rows idx
        (None = identity), XOR r: one ogm_pack_gather launch."""
        out = torch.empty((pr.rows, _pitch(pr.width)), dtype=torch.int32, device=self.dev)
        mats = [pr.fields[f][0][s] for s in sets for f in range(len(pr.fields))]
        pitches = [m.stride(0) if pr.rows else words_for(pr.fields[f][1])
                   for m, f in zip(mats, [f for _ in sets for f in range(len(pr.fields))])]
        flags = A([pr.flags[s] for s in sets]) if pr.flags is not None else None
        _lib.call("ogm_pack_gather", pr.rows, _lib.ptr(idx), len(sets), flags, len(pr.fields), A(mats),
                  _lib.i64_array(pitches), _lib.i64_array([wd for _, wd in pr.fields]), _lib.ptr(r), _lib.ptr(out),
                  out.shape[1], _lib.stream_ptr())
        return out

    def _shuffle_online(self, comps, width: int, m: dict) -> list:
        rows = comps.rows if isinstance(comps, PackedRows) else comps[0].shape[0]

        def tab():
            return torch.empty((rows, _pitch(width)), dtype=torch.int32, device=self.dev)

        if isinstance(comps, PackedRows):
            # P1 packs a^b at its composed permutation, P2 packs c at pi12
            x1 = self.pack_gather(comps, (0, 1), idx=m["k1"], r=m["u"])             # P1
            y1 = self.pack_gather(comps, (2,), idx=m["pi12"], r=m["v"])              # P2
        else:
            ab = self._xor01(comps)
            x1 = gather(rows, width, tab(), inner=m["k1"], m1=ab, r=m["u"])           # P1
            del ab
            y1 = gather(rows, width, tab(), inner=m["pi12"], m1=comps[2], r=m["v"])   # P2
        c1 = gather(rows, width, tab(), inner=m["pi23"], m1=x1, r=m["w"])         # P2
        del x1
        r3 = gather(rows, width, tab(), inner=m["k3"], m1=y1, m3=c1, r=m["z"])    # P3
        return [m["r1"], m["r2"], r3]

    # -- engine steps -----------------------------------------------------------
    def _fde(self, keys: list, domain: int) -> torch.Tensor:
        return fss.full_domain(fss.KeyBatch.from_keys(keys, self.dev), domain)

    def _pass_indicators(self, key_pairs: list, domain: int, cache: dict) -> list:
        """Per pass, the six full-domain indicator rows [P1 a, P1 b, P2 a,
        P2 b, P3 a, P3 b] of one predicate (src/engine.py:150-158), cached
        per key."""
        parts = [list(zip(fss.key_parts_for_engine(f), fss.key_parts_for_engine(s))) for f, s in key_pairs]
        npass = len(parts[0])
        if any((id(key_pairs[0][0]), ps) not in cache for ps in range(npass)):
            # every pass's keys at once, one full-domain launch per key kind (an interval's two
            # passes are both DCF: one launch of 12 keys instead of two of 6)
            keys = [k for ps in range(npass) for q in range(3) for k in parts[q][ps]]
            by_kind: dict = {}
            for i, k in enumerate(keys):
                by_kind.setdefault(fss.is_comparison(k), []).append(i)
            rows = [None] * len(keys)
            for idxs in by_kind.values():
                fd = self._fde([keys[i] for i in idxs], domain)
                for j, i in enumerate(idxs):
                    rows[i] = fd[j]
            for ps in range(npass):
                cache[(id(key_pairs[0][0]), ps)] = rows[6 * ps:6 * ps + 6]
        return [cache[(id(key_pairs[0][0]), ps)] for ps in range(npass)]

    # a two-pass predicate as one parity pass over folded indicators (sec_eval)
    FOLD_PASSES = True

    def _folded_indicators(self, key_pairs: list, domain: int, cache: dict) -> list:
        """The six indicator rows of a two-pass (interval) predicate XORed
        over the passes, cached per key: parity is linear and a re-share is a
        zero share XORed in, so the XOR of the two passes' re-shared parities
        (src/engine.py:150-165) is ONE parity over the folded indicators with
        both zero shares XORed in (reshare2)."""
        ck = (id(key_pairs[0][0]), "fold")
        if ck not in cache:
            p0, p1 = self._pass_indicators(key_pairs, domain, cache)
            pitch = p0[1].data_ptr() - p0[0].data_ptr()
            if pitch > 0 and all(r.data_ptr() == p0[0].data_ptr() + i * pitch for i, r in enumerate(p0 + p1)):
                # both passes' rows are consecutive rows of one full-domain batch: one launch
                n = 6 * pitch // 4
                out = torch.empty((n,), dtype=torch.int32, device=self.dev)
                _lib.call("ogm_xor_words", n, p0[0].data_ptr(), p1[0].data_ptr(), None, _lib.ptr(out),
                          _lib.stream_ptr())
                w = p0[0].numel()
                rows = [out[i * (pitch // 4): i * (pitch // 4) + w] for i in range(6)]
            else:
                rows = []
                for a, b in zip(p0, p1):
                    o = torch.empty_like(a)
                    _lib.call("ogm_xor_words", a.numel(), _lib.ptr(a), _lib.ptr(b), None, _lib.ptr(o),
                              _lib.stream_ptr())
                    rows.append(o)
            cache[ck] = rows
        return cache[ck]

    def reshare2(self, adds: list, nbits: int) -> list:
        """Two consecutive re-shares (counters c, c + 1) of values whose XOR
        is ``adds``, folded: the XOR of reshare(x0) and reshare(x1) for x0 ^
        x1 = adds (src/rss.py:164-176 twice, comp j := blinded_{j-1})."""
        outs = [torch.empty_like(a) for a in adds]
        if nbits:
            _lib.call("ogm_zero_share_trio_fold2", self.k[0], self.k[1], self.k[2], self.counter, self.counter + 1,
                      nbits, 0, words_for(nbits), A(adds), A(outs), _lib.stream_ptr())
        self.counter += 2
        return [outs[2], outs[0], outs[1]]

    def sec_eval(self, group: TrioGroup, key_pairs: list, attr: str, domain: int, cache: dict) -> list:
        """src/engine.py:139-165 for all parties in one read of the shares; a
        two-pass (interval) predicate as ONE parity pass over the folded
        indicators (_folded_indicators, reshare2) -- the same result shares."""
        inds = self._pass_indicators(key_pairs, domain, cache)
        comps = group.attrs[attr]
        rows = group.count
        words = comps[0].shape[1]
        if len(inds) == 2 and self.FOLD_PASSES:
            outs = [self._empty(words_for(rows)) for _ in range(3)]
            _lib.call("ogm_masked_parity", rows, words, comps[0].stride(0), 3, A(comps), 3, _lib.int_array([0, 1, 2]),
                      _lib.int_array([1, 2, 0]), 1, A(self._folded_indicators(key_pairs, domain, cache)), A(outs),
                      _lib.stream_ptr())
            return self.reshare2(outs, rows)
        npass = len(inds)
        outs = [self._empty(words_for(rows)) for _ in range(3 * npass)]
        _lib.call("ogm_masked_parity", rows, words, comps[0].stride(0), 3, A(comps), 3, _lib.int_array([0, 1, 2]),
                  _lib.int_array([1, 2, 0]), npass, A([t for ps in range(npass) for t in inds[ps]]), A(outs),
                  _lib.stream_ptr())
        result = None
        for ps in range(npass):
            sh = self.reshare(outs[3 * ps:3 * ps + 3], rows)
            result = sh if result is None else self.xor(result, sh)
        return result

    def combine(self, bits: list, combiner: str, any_mode: str, n: int) -> list:
        """src/engine.py:168-189."""
        if not bits:
            raise ValueError("no predicate bits to combine")
        acc = bits[0]
        if combiner == "ALL":
            for nxt in bits[1:]:
                acc = self.and_gate(acc, nxt, n)
            return acc
        if combiner != "ANY":
            raise ValueError(f"unknown combiner {combiner!r}")
        if any_mode == "xor":
            for nxt in bits[1:]:
                acc = self.xor(acc, nxt)
            return acc
        if any_mode != "or":
            raise ValueError(f"unknown ANY mode {any_mode!r}")
        for nxt in bits[1:]:
            conj = self.and_gate(acc, nxt, n)
            acc = self.xor(self.xor(acc, nxt), conj)
        return acc

    def _fold(self, flags: list, mats: list, width: int) -> list:
        rows = mats[0].shape[0]
        flat = [rows2d(m) for m in mats]  # padded row pitches stay zero-copy
        words = flat[0].shape[1]
        outs = [self._empty(words) for _ in range(3)]
        _lib.call("ogm_select_fold", rows, words, flat[0].stride(0) if rows else words, 3, A(flat),
                  A([flat[_nxt(q)] for q in range(3)]), A(flags), A([flags[_nxt(q)] for q in range(3)]), A(outs),
                  _lib.stream_ptr())
        return outs

    def fetch_unique(self, group: TrioGroup, flags: list) -> TrioRecords:
        """src/engine.py:197-217."""
        ids = self.reshare(self._fold(flags, group.ids, group.id_width), group.id_width)
        attrs = {}
        for name in sorted(group.attrs):
            attrs[name] = self.reshare(self._fold(flags, group.attrs[name], group.attr_widths[name]),
                                       group.attr_widths[name])
        return TrioRecords(group.parent_slot, group.parent_record, 1, group.id_width, [c[None] for c in ids],
                           {a: [c[None] for c in v] for a, v in attrs.items()}, dict(group.attr_widths))

    def _open_keep(self, shuffled: list, rows: int, phase: str, audit: list, fields: list) -> tuple:
        """src/engine.py:243-269 / :321-334 for all parties in one synchronous
        call (ogm_trio_open_keep): open the flag column (the next open label),
        keep the flagged rows in order and slice each (bit offset, width)
        field out of the three components.  Returns (k, [[c1, c2, c3] per field])."""
        self.label += 1
        nw = words_for(rows)
        host = np.empty((max(nw, 1),), np.uint32)
        outs = [[torch.empty((max(rows, 1), words_for(w)), dtype=torch.int32, device=self.dev) for _ in range(3)]
                for _, w in fields]
        lib = _lib.load()
        nb = int(lib.ogm_trio_open_keep_workspace_bytes(rows))
        ws = self.__dict__.get("_open_ws")
        if ws is None or ws.numel() < nb:
            ws = self._open_ws = torch.empty((nb,), dtype=torch.uint8, device=self.dev)
        kept = ctypes.c_int64(0)
        nf = len(fields)
        _lib.call("ogm_trio_open_keep", A(shuffled), rows, shuffled[0].stride(0), host.ctypes.data, nf,
                  _lib.i64_array([o for o, _ in fields]), _lib.i64_array([w for _, w in fields]),
                  A([outs[f][c] for c in range(3) for f in range(nf)]),
                  _lib.i64_array([words_for(w) for _, w in fields]), ctypes.byref(kept), _lib.ptr(ws), nb,
                  _lib.stream_ptr())
        opened = BitVector(host[:nw], rows)
        self.opened.append((self.label, opened))
        audit.append((phase, opened.to_bits()))
        k = int(kept.value)
        return k, [[o[:k] for o in per] for per in outs]

    def prepare_fetch(self, rows: int) -> None:
        """Offline phase of the NEXT fetch of ``rows`` flagged 128-bit rows
        (table id self.table_id): the FlaggedFetch material, parked until
        fetch_multi consumes it."""
        from .fetch import FlaggedFetch
        tid = self.table_id
        if not hasattr(self, "_prepared_fetch"):
            self._prepared_fetch = {}
        self._prepared_fetch[(tid, rows)] = FlaggedFetch((self.s12, self.s23, self.s31), tid, rows, self.dev)

    def _fetch_flagged128(self, group: TrioGroup, flags: list, audit: list) -> TrioRecords:
        """src/engine.py:220-270 for a group whose rows are a 128-bit id and
        no attributes (the C5 fetch shape), in the flag-split layout
        (fetch.FlaggedFetch): same table id, open label and records as the
        packed-row path, bit for bit."""
        from .fetch import FlaggedFetch
        rows = group.count
        tid = self.table_id
        self.table_id += 1
        ff = getattr(self, "_prepared_fetch", {}).pop((tid, rows), None)
        if ff is None:
            ff = FlaggedFetch((self.s12, self.s23, self.s31), tid, rows, self.dev)
        payload = [c if c.dim() == 2 and c.shape[1] == 4 and c.is_contiguous() else
                   rows2d(c).reshape(rows, -1)[:, :4].contiguous() for c in group.ids]
        ff.online(list(flags), payload)
        self.label += 1
        words, k = ff.opened_host()   # the opened column and the kept count, one synchronisation
        opened = BitVector(words, rows)   # copies the words
        # the records are views of the fetch's row-sized outputs unless those would pin more than
        # 256 MB for few rows (then copied); the host bookkeeping below overlaps the copies
        ids = [o[:k] if 2 * k >= rows or 3 * rows * 16 <= (256 << 20) else o[:k].clone() for o in ff.outs]
        self.opened.append((self.label, opened))
        audit.append(("fetch", opened.to_bits()))   # a fresh array (unpacked from the words)
        return TrioRecords(group.parent_slot, group.parent_record, k, group.id_width, ids, {}, {})

    def fetch_multi(self, group: TrioGroup, flags: list, audit: list, online_blinds=None) -> TrioRecords:
        """src/engine.py:220-270."""
        if group.id_width == 128 and not group.attrs and group.count > 0:
            return self._fetch_flagged128(group, flags, audit)
        names = sorted(group.attrs)
        widths = [group.attr_widths[a] for a in names]
        row_width = 1 + group.id_width + sum(widths)
        rows = PackedRows(group.count, row_width, list(flags),
                          [(group.ids, group.id_width)] + [(group.attrs[a], w) for a, w in zip(names, widths)])
        sh = self.shuffle(rows, row_width, online_blinds)
        del rows
        fields, off = [(1, group.id_width)], 1 + group.id_width
        for w in widths:
            fields.append((off, w))
            off += w
        k, got = self._open_keep(sh, group.count, "fetch", audit, fields)
        ids = got[0]
        attrs = dict(zip(names, got[1:]))
        return TrioRecords(group.parent_slot, group.parent_record, k, group.id_width, ids, attrs,
                           dict(zip(names, widths)))

    def _consts(self, w: int):
        """Cached all-ones / all-zeros indicator rows of w words."""
        cache = self.__dict__.setdefault("_const_cache", {})
        if w not in cache:
            cache[w] = (torch.full((w,), -1, dtype=torch.int32, device=self.dev),
                        torch.zeros((w,), dtype=torch.int32, device=self.dev))
        return cache[w]

    def _parity_rows(self, mats: list, w) -> list:
        """Row parities of the three components in one trio launch: party q's
        parity(A_q & 1...1 ^ B_q & 0) is the parity of component q's row."""
        rows = mats[0].shape[0]
        outs = [self._empty(words_for(rows)) for _ in range(3)]
        ones, zeros = self._consts(w)
        _lib.call("ogm_masked_parity", rows, w, mats[0].stride(0), 3, A(mats), 3, _lib.int_array([0, 1, 2]),
                  _lib.int_array([1, 2, 0]), 1, A([ones, zeros] * 3), A(outs), _lib.stream_ptr())
        return outs

    def access(self, rec: TrioRecords, i: int, parent_type: str, child_type: str, needed: list, gshares: list,
               provenance: tuple, audit: list) -> TrioGroup:
        """src/engine.py:278-344."""
        schema = gshares[0].schema
        parent_slot, parent_rec = provenance
        x_ne = schema.types[child_type].population
        w_ne = words_for(x_ne)
        widths = {a: schema.types[child_type].attrs[a].domain_size for a in needed}
        lists = [gs.types[parent_type].posting[child_type][0] for gs in gshares]
        l_max = lists[0].shape[1]

        def empty():
            z = lambda w: torch.zeros((0, w), dtype=torch.int32, device=self.dev)  # noqa: E731
            return TrioGroup(parent_slot, parent_rec, 0, x_ne, [z(w_ne)] * 3,
                             {a: [z(words_for(widths[a]))] * 3 for a in needed}, widths)

        if l_max == 0:
            return empty()
        sel = [c[i] for c in rec.ids]
        adds = [a.reshape(l_max, w_ne) for a in self._fold(sel, lists, x_ne)]
        fetched = self.reshare_matrix(adds, x_ne)
        rows = PackedRows(l_max, 1 + x_ne, self._parity_rows(fetched, w_ne), [(fetched, x_ne)])
        sh = self.shuffle(rows, 1 + x_ne)
        k, got = self._open_keep(sh, l_max, "access", audit, [(1, x_ne)])
        if k == 0:
            return empty()
        ids = got[0]
        attrs = {}
        for a in needed:
            va = [gs.types[child_type].attrs[a][0] for gs in gshares]
            n = widths[a]
            adds = []
            for q in range(3):
                x, w = va[q].shape
                out = torch.empty((k, w), dtype=torch.int32, device=self.dev)
                ws = torch.empty((2 * max(x, 1),), dtype=torch.int32, device=self.dev)
                _lib.call("ogm_select_many", k, x, w, va[q].stride(0), _lib.ptr(ids[q]), _lib.ptr(ids[_nxt(q)]),
                          ids[q].stride(0), _lib.ptr(va[q]), _lib.ptr(va[_nxt(q)]), _lib.ptr(out), w, _lib.ptr(ws),
                          _lib.stream_ptr())
                adds.append(out)
            attrs[a] = self.reshare_matrix(adds, n)
        return TrioGroup(parent_slot, parent_rec, k, x_ne, ids, attrs, widths)

    # -- full query ----------------------------------------------------------
    def _root_group(self, gshares: list, vtype: str, ts, needed: list) -> TrioGroup:
        """Every vertex of the root type is a candidate (src/engine.py:372-379)."""
        tps = [gs.types[vtype] for gs in gshares]
        return TrioGroup(None, None, ts.population, ts.population, [t.id_a for t in tps],
                         {a: [t.attrs[a][0] for t in tps] for a in needed},
                         {a: ts.attrs[a].domain_size for a in needed})

    def match(self, tokens: list, gshares: list, any_mode: str = "or", native: bool = True) -> TrioResult:
        """src/engine.py:352-417 for the three parties at once.  gshares are the
        three per-party device shares from graphs.device_trio (component j is
        party j's share_a).  ``native`` runs the schedule in the C++ executor
        (ogm_trio_match: one C-ABI call); ``native=False`` issues the same
        steps from Python (kept as the readable restatement, tested equal).
        The native executor takes at most OGM_TRIO_MAX_ATTRS needed
        attributes per slot; wider slots run the Python schedule (the
        reference has no such limit)."""
        if native:
            from .trio_native import MAX_ATTRS, match_native
            slots = tokens[0].structure["slots"] if tokens else []
            if all(len({p["attr"] for p in sl["preds"]}) <= MAX_ATTRS for sl in slots):
                return match_native(self, tokens, gshares, any_mode)
        schema = gshares[0].schema
        for t in tokens:
            if t.schema_digest != schema.digest():
                raise ValueError("token and graph share were built for different schemas")
        slots = tokens[0].structure["slots"]
        audit: list = []
        groups: list = [[] for _ in slots]
        records: list = [[] for _ in slots]
        cache: dict = {}
        for s, slot in enumerate(slots):
            vtype = slot["type"]
            ts = schema.types[vtype]
            needed = sorted({p["attr"] for p in slot["preds"]})
            if s == 0:
                groups[0] = [self._root_group(gshares, vtype, ts, needed)]
            unique_route = (len(slot["preds"]) == 1 and slot["preds"][0]["kind"] == fss.KIND_EQ
                            and ts.attrs[slot["preds"][0]["attr"]].unique)
            for group in groups[s]:
                if group.count == 0:
                    continue
                bits = [self.sec_eval(group, [tok.slot_keys[s][pi] for tok in tokens], pred["attr"],
                                      ts.attrs[pred["attr"]].domain_size, cache)
                        for pi, pred in enumerate(slot["preds"])]
                flags = self.combine(bits, slot["combiner"], any_mode, group.count)
                batch = self.fetch_unique(group, flags) if unique_route else self.fetch_multi(group, flags, audit)
                records[s].extend((batch, i) for i in range(batch.count))
            for child in slot["children"]:
                ctype = slots[child]["type"]
                cattrs = sorted({p["attr"] for p in slots[child]["preds"]})
                groups[child] = [self.access(b, i, vtype, ctype, cattrs, gshares, (s, ri), audit)
                                 for ri, (b, i) in enumerate(records[s])]
        views = [[_RecView(b.parent_slot, b.parent_record) for b, _ in recs] for recs in records]
        subgraphs = _assemble(slots, views)
        return TrioResult(tokens[0].structure, records, subgraphs, audit)


@dataclass
class _RecView:
    parent_slot: int | None
    parent_record: int | None
