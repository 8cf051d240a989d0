"""ctypes side of the native trio executor (ogm_trio_match, csrc/ogm_trio.cuh).

``match_native`` runs the trio fast path's whole sec_match (src/engine.py:
352-417 for the three co-resident parties) in one C-ABI call: Python only
lays out the plan (type tables, slots, the full-domain indicators of the
query's keys) and wraps the returned record batches as tensor views into the
executor's arena.  Same launches, same randomness order and bit-identical
outputs as the Python ``Trio.match`` (tested side by side).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, fss
from .bits import BitVector, rows2d, words_for

MAX_ATTRS = 8
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u8p = ctypes.c_char_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32


class Mat(ctypes.Structure):
    _fields_ = [("c", ctypes.c_void_p * 3), ("pitch", _i64), ("width", _i64), ("unique", _i32)]


class Posting(ctypes.Structure):
    _fields_ = [("child_type", _i32), ("l_max", _i64), ("lists", Mat)]


class TType(ctypes.Structure):
    _fields_ = [("population", _i64), ("ids", Mat), ("nattrs", _i32), ("attrs", ctypes.POINTER(Mat)),
                ("npostings", _i32), ("postings", ctypes.POINTER(Posting))]


class Pred(ctypes.Structure):
    _fields_ = [("attr", _i32), ("npass", _i32), ("ind", ctypes.c_void_p * 12)]


class Slot(ctypes.Structure):
    _fields_ = [("type", _i32), ("combiner_all", _i32), ("unique_route", _i32), ("npreds", _i32),
                ("preds", ctypes.POINTER(Pred)), ("nneeded", _i32), ("needed", _i32p), ("nchildren", _i32),
                ("children", _i32p)]


class Plan(ctypes.Structure):
    _fields_ = [("zero_key", ctypes.c_void_p * 3), ("s12", ctypes.c_void_p), ("s23", ctypes.c_void_p),
                ("s31", ctypes.c_void_p), ("counter", ctypes.c_uint64), ("table_id", ctypes.c_uint64),
                ("label", ctypes.c_uint32), ("any_xor", _i32), ("ntypes", _i32), ("types", ctypes.POINTER(TType)),
                ("nslots", _i32), ("slots", ctypes.POINTER(Slot))]


class Batch(ctypes.Structure):
    _fields_ = [("slot", _i32), ("parent_slot", _i32), ("parent_record", _i32), ("count", _i64),
                ("id_width", _i64), ("ids", ctypes.c_void_p * 3), ("ids_pitch", _i64), ("nattrs", _i32),
                ("attr_id", _i32 * MAX_ATTRS), ("attr_width", _i64 * MAX_ATTRS),
                ("attrs", (ctypes.c_void_p * 3) * MAX_ATTRS), ("attr_pitch", _i64 * MAX_ATTRS)]


class Open(ctypes.Structure):
    _fields_ = [("phase", _i32), ("label", ctypes.c_uint32), ("nbits", _i64), ("bits_off", _i64)]


class Out(ctypes.Structure):
    _fields_ = [("max_batches", _i32), ("nbatches", _i32), ("batches", ctypes.POINTER(Batch)),
                ("max_opens", _i32), ("nopens", _i32), ("opens", ctypes.POINTER(Open)), ("open_bits", _u32p),
                ("open_bits_cap", _i64), ("open_bits_used", _i64), ("arena_used", _i64)]




def _mat(comps, width: int, unique: bool = False) -> Mat:
    m = Mat()
    for q in range(3):
        m.c[q] = comps[q].data_ptr()
    m.pitch = comps[0].stride(0)
    m.width = width
    m.unique = int(unique)
    return m


def _type_tables(gshares: list):
    """The schema-wide part of the plan (type tables: ids, attributes,
    flattened posting lists of the three components), built once per set of
    device shares and cached on the first share object."""
    key = tuple(id(g) for g in gshares)
    cached = getattr(gshares[0], "_native_plan", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    schema = gshares[0].schema
    keep = []
    tnames = sorted(schema.types)
    tindex = {t: i for i, t in enumerate(tnames)}
    anames = {t: sorted(schema.types[t].attrs) for t in tnames}
    types = (TType * len(tnames))()
    for i, t in enumerate(tnames):
        ts = schema.types[t]
        tp = [gs.types[t] for gs in gshares]
        types[i].population = ts.population
        ids = [x.id_a for x in tp]
        keep.append(ids)
        types[i].ids = _mat(ids, ts.population)
        attrs = (Mat * max(1, len(anames[t])))()
        for j, a in enumerate(anames[t]):
            comps = [x.attrs[a][0] for x in tp]
            keep.append(comps)
            attrs[j] = _mat(comps, ts.attrs[a].domain_size, ts.attrs[a].unique)
        types[i].nattrs = len(anames[t])
        types[i].attrs = attrs
        posts = sorted(tp[0].posting)
        parr = (Posting * max(1, len(posts)))()
        for j, c in enumerate(posts):
            lists = [rows2d(x.posting[c][0]) for x in tp]
            keep.append(lists)
            parr[j].child_type = tindex[c]
            parr[j].l_max = tp[0].posting[c][0].shape[1]
            parr[j].lists = _mat(lists, 32 * lists[0].shape[1])
        types[i].npostings = len(posts)
        types[i].postings = parr
        keep += [attrs, parr]

    out = (tnames, tindex, anames, types)
    gshares[0]._native_plan = (key, out, keep, list(gshares))
    return out


def match_native(trio, tokens: list, gshares: list, any_mode: str = "or"):
    from .trio import TrioRecords, TrioResult, _RecView
    from .engine import _assemble

    schema = gshares[0].schema
    for t in tokens:
        if t.schema_digest != schema.digest():
            raise ValueError("token and graph share were built for different schemas")
    if any_mode not in ("or", "xor"):
        raise ValueError(f"unknown ANY mode {any_mode!r}")
    slots = tokens[0].structure["slots"]
    keep = []  # every tensor / ctypes buffer the call reads stays alive here

    tnames, tindex, anames, types = _type_tables(gshares)
    sarr = (Slot * len(slots))()
    fde_jobs: list = []   # (preds, pred, pass, key positions, keys, domain): expanded after the loop
    for s, slot in enumerate(slots):
        vtype = slot["type"]
        ts = schema.types[vtype]
        needed = sorted({p["attr"] for p in slot["preds"]})
        preds = (Pred * len(slot["preds"]))()
        for pi, pred in enumerate(slot["preds"]):
            key_pairs = [tok.slot_keys[s][pi] for tok in tokens]
            parts = [list(zip(fss.key_parts_for_engine(f), fss.key_parts_for_engine(g))) for f, g in key_pairs]
            npass = len(parts[0])
            domain = ts.attrs[pred["attr"]].domain_size
            preds[pi].attr = anames[vtype].index(pred["attr"])
            preds[pi].npass = npass
            for ps in range(npass):
                keys = [k for q in range(3) for k in parts[q][ps]]
                by_kind: dict = {}
                for i, k in enumerate(keys):
                    by_kind.setdefault(fss.is_comparison(k), []).append(i)
                for idxs in by_kind.values():
                    fde_jobs.append((preds, pi, ps, idxs, [keys[i] for i in idxs], domain))
        unique_route = (len(slot["preds"]) == 1 and slot["preds"][0]["kind"] == fss.KIND_EQ
                        and ts.attrs[slot["preds"][0]["attr"]].unique)
        nd = (_i32 * max(1, len(needed)))(*[anames[vtype].index(a) for a in needed])
        ch = (_i32 * max(1, len(slot["children"])))(*slot["children"])
        keep += [preds, nd, ch]
        sarr[s].type = tindex[vtype]
        sarr[s].combiner_all = int(slot["combiner"] == "ALL")
        if slot["combiner"] not in ("ALL", "ANY"):
            raise ValueError(f"unknown combiner {slot['combiner']!r}")
        sarr[s].unique_route = int(unique_route)
        sarr[s].npreds = len(slot["preds"])
        sarr[s].preds = preds
        sarr[s].nneeded = len(needed)
        sarr[s].needed = nd
        sarr[s].nchildren = len(slot["children"])
        sarr[s].children = ch

    # every predicate pass's key batches: ONE host image, ONE host-to-device copy, then the
    # full-domain expansions (src/fss.py:302-337) straight from device slices
    images, offs, total = [], [], 0
    for *_, ks, _ in fde_jobs:
        img = fss.pack_keys(ks, ks[0].domain_bits)
        offs.append(total)
        images.append(img)
        total += (img.size + 15) // 16 * 16
    if fde_jobs:
        host = np.zeros(total, np.uint8)
        for img, o in zip(images, offs):
            host[o: o + img.size] = img
        dev = torch.from_numpy(host).pin_memory().to(trio.dev, non_blocking=True)
        keep.append(dev)
        # every expansion writes into one allocation (16-byte row pitch), device pointers by offset
        pitches = [(words_for(job[5]) + 3) // 4 * 4 for job in fde_jobs]
        outs = torch.empty((sum(len(job[4]) * p for job, p in zip(fde_jobs, pitches)),), dtype=torch.int32,
                           device=trio.dev)
        keep.append(outs)
        base, obase, oo = dev.data_ptr(), outs.data_ptr(), 0
        stream = _lib.stream_ptr()
        for (preds, pi, ps, idxs, ks, domain), o, pitch in zip(fde_jobs, offs, pitches):
            n, bits = len(ks), ks[0].domain_bits
            if not 1 <= bits <= fss.MAX_DEVICE_BITS:
                raise fss.DomainError(f"domain_bits {bits} outside 1..{fss.MAX_DEVICE_BITS}")
            a, b = 16 * n, 16 * n * (1 + bits)
            kind = _lib.KIND_DCF if fss.is_comparison(ks[0]) else _lib.KIND_DPF
            _lib.call("ogm_fss_full_domain", kind, bits, n, base + o, base + o + a, base + o + b,
                      base + o + b + 12 * n, domain, obase + 4 * oo, pitch, stream)
            for j, i in enumerate(idxs):   # key i of the pass: party i // 2, share i % 2 (a, b)
                preds[pi].ind[ps * 6 + i] = obase + 4 * (oo + j * pitch)
            oo += n * pitch

    seeds = [ctypes.create_string_buffer(bytes(x), 16) for x in (*trio.k, trio.s12, trio.s23, trio.s31)]
    keep.append(seeds)
    fn = _lib.load().ogm_trio_match  # releases the GIL: the call synchronises on every open
    arena_bytes = max(getattr(trio, "_arena_bytes", 0), 64 << 20)
    max_batches, max_opens, bits_cap = 256, 256, 1 << 15
    while True:
        plan = Plan()
        for q in range(3):
            plan.zero_key[q] = ctypes.addressof(seeds[q])
        plan.s12, plan.s23, plan.s31 = (ctypes.addressof(seeds[3]), ctypes.addressof(seeds[4]),
                                        ctypes.addressof(seeds[5]))
        plan.counter, plan.table_id, plan.label = trio.counter, trio.table_id, trio.label
        plan.any_xor = int(any_mode == "xor")
        plan.ntypes, plan.types = len(tnames), types
        plan.nslots, plan.slots = len(slots), sarr
        # a fresh arena per query: the returned records are views into it
        arena = torch.empty((arena_bytes,), dtype=torch.uint8, device=trio.dev)
        batches = (Batch * max_batches)()
        opens = (Open * max_opens)()
        bits = np.empty(bits_cap, np.uint32)
        out = Out(max_batches, 0, batches, max_opens, 0, opens, bits.ctypes.data_as(_u32p), bits_cap, 0, 0)
        rc = fn(ctypes.addressof(plan), ctypes.addressof(out), arena.data_ptr(), arena.numel(), _lib.stream_ptr())
        if rc == _lib.OGM_ERR_NOMEM:
            arena_bytes = max(2 * arena_bytes, int(out.arena_used) * 2)
            max_batches *= 2
            max_opens *= 2
            bits_cap *= 2
            trio._arena_bytes = arena_bytes
            continue
        _lib.check(rc)
        break
    trio.counter, trio.table_id, trio.label = int(plan.counter), int(plan.table_id), int(plan.label)

    base = arena.data_ptr()
    a32 = arena.view(torch.int32)
    n32 = a32.numel()

    def view(ptr, rows, pitch, width):
        w = words_for(width)
        if rows == 0:
            return torch.zeros((0, w), dtype=torch.int32, device=trio.dev)
        off = (ptr - base) // 4
        if off < 0 or off + rows * pitch > n32:
            raise RuntimeError("ogm_trio_match returned a record matrix outside its arena")
        return torch.as_strided(a32, (rows, w), (pitch, 1), off)   # one op: rows of the pitched matrix

    records: list = [[] for _ in slots]
    for bi in range(out.nbatches):
        b = batches[bi]
        n = int(b.count)
        ids = [view(b.ids[q], n, b.ids_pitch, b.id_width) for q in range(3)]
        vtype = slots[b.slot]["type"]
        attrs, widths = {}, {}
        for j in range(b.nattrs):
            name = anames[vtype][b.attr_id[j]]
            attrs[name] = [view(b.attrs[j][q], n, b.attr_pitch[j], b.attr_width[j]) for q in range(3)]
            widths[name] = int(b.attr_width[j])
        batch = TrioRecords(None if b.parent_slot < 0 else int(b.parent_slot),
                            None if b.parent_record < 0 else int(b.parent_record), n, int(b.id_width), ids, attrs,
                            widths)
        records[b.slot].extend((batch, i) for i in range(n))
    audit = []
    for oi in range(out.nopens):
        o = opens[oi]
        bv = BitVector(bits[o.bits_off: o.bits_off + words_for(o.nbits)].copy(), int(o.nbits))
        trio.opened.append((int(o.label), bv))
        audit.append(("fetch" if o.phase == 0 else "access", bv.to_bits()))
    views = [[_RecView(b.parent_slot, b.parent_record) for b, _ in recs] for recs in records]
    result = TrioResult(tokens[0].structure, records, _assemble(slots, views), audit)
    result._keep = (arena, keep)  # the record tensors are views into the arena
    return result
