"""Share, graph-share and result files (src/storage.py), loaded straight into HBM.

Same byte formats as the reference, so files written by either side load on
the other:

* share record  ``"OGMS" | version u16 | party u8 | logical_len u64 | LE words``
* graph share   ``"OGMG" | version u16 | party u8 | schema digest (32)`` then
  one record pair per vector in canonical order (per type sorted, per
  vertex: id, attrs sorted, posting entries by posting type / slot)
* results       ``"OGMR" | ... | JSON manifest | record pairs``

:func:`load_graph_share` is the device loader: every
record offset follows from the public schema, so the record table is built
with numpy, all headers are validated in bulk, the file image is uploaded
once and one kernel (``ogm_unpack_records``) moves every payload -- at
arbitrary byte alignment -- into the device matrices.
"""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .bits import BitVector, words_for
from .engine import MatchedRecord, MatchResultSet
from .graphs import GraphSchema, GraphShare, TypePartyShare
from .rss import DBits, SharedBitVector

SHARE_MAGIC = b"OGMS"
GRAPH_MAGIC = b"OGMG"
RESULT_MAGIC = b"OGMR"
VERSION = 1

_SHARE_HEADER = struct.Struct("<4sHBQ")
_CONTAINER_HEADER = struct.Struct("<4sHB32s")
_HDR = _SHARE_HEADER.size  # 15


class StorageError(ValueError):
    """Corrupt or mismatched share/result files (src/storage.py:39-40)."""


def _host_words(v) -> np.ndarray:
    if isinstance(v, torch.Tensor):
        return v.detach().cpu().contiguous().numpy().view(np.uint32).reshape(-1)
    if isinstance(v, (BitVector, DBits)):
        return _host_words(v.words)
    return np.ascontiguousarray(v, np.uint32).reshape(-1)


def encode_share_vector(party: int, vec) -> bytes:
    """src/storage.py:43-45."""
    return _SHARE_HEADER.pack(SHARE_MAGIC, VERSION, party, vec.logical_len) + _host_words(vec).tobytes()


def decode_share_vector(buf, offset: int = 0):
    """src/storage.py:48-64 -> (party, BitVector, next_offset)."""
    if len(buf) < offset + _HDR:
        raise StorageError("truncated share record")
    magic, version, party, nbits = _SHARE_HEADER.unpack_from(buf, offset)
    if magic != SHARE_MAGIC:
        raise StorageError("bad share record magic")
    if version != VERSION:
        raise StorageError(f"unsupported share record version {version}")
    pos = offset + _HDR
    nwords = words_for(nbits)
    end = pos + 4 * nwords
    if len(buf) < end:
        raise StorageError("truncated share record payload")
    return party, BitVector(np.frombuffer(buf, dtype=np.uint32, count=nwords, offset=pos), nbits), end


def save_schema(path, schema: GraphSchema) -> None:
    Path(path).write_text(schema.to_json() + "\n")


def load_schema(path) -> GraphSchema:
    return GraphSchema.from_json(Path(path).read_text())


# ---------------------------------------------------------------------------
# graph share containers
# ---------------------------------------------------------------------------


def _vectors(gshare: GraphShare):
    """Canonical vector order (src/storage.py:82-99)."""
    schema = gshare.schema
    for vtype in sorted(schema.types):
        ts = schema.types[vtype]
        tps = gshare.types[vtype]
        x = ts.population
        id_a, id_b = _host_rows(tps.id_a), _host_rows(tps.id_b)
        attrs = {a: (_host_rows(tps.attrs[a][0]), _host_rows(tps.attrs[a][1])) for a in sorted(ts.attrs)}
        post = {t: (_host_rows(tps.posting[t][0]), _host_rows(tps.posting[t][1])) for t in ts.posting_types}
        for v in range(x):
            yield id_a[v], id_b[v], x
            for a in sorted(ts.attrs):
                yield attrs[a][0][v], attrs[a][1][v], ts.attrs[a].domain_size
            for t_ne in ts.posting_types:
                width = schema.types[t_ne].population
                for slot in range(ts.padded_len[t_ne][v]):
                    yield post[t_ne][0][v, slot], post[t_ne][1][v, slot], width


def _host_rows(m):
    if isinstance(m, torch.Tensor):
        return m.detach().cpu().numpy().view(np.uint32)
    return np.asarray(m, np.uint32)


def save_graph_share(path, gshare: GraphShare) -> None:
    """src/storage.py:102-107 (host or device shares)."""
    p = gshare.party_index
    parts = [_CONTAINER_HEADER.pack(GRAPH_MAGIC, VERSION, p, gshare.schema.digest())]
    for wa, wb, width in _vectors(gshare):
        for w in (wa, wb):  # BitVector(words, width) in the reference: tails masked
            w = np.array(w, np.uint32)
            if width % 32 and w.size:
                w[-1] &= np.uint32((1 << (width % 32)) - 1)
            parts.append(_SHARE_HEADER.pack(SHARE_MAGIC, VERSION, p, width) + w.tobytes())
    Path(path).write_bytes(b"".join(parts))


def _record_table(schema: GraphSchema):
    """Every record of a graph-share file, in file order, as numpy arrays:
    header byte offset, width, destination (matrix key, word offset)."""
    hdr, width, mat, dst = [], [], [], []
    layout = {}      # matrix key -> (shape, words)
    pos = _CONTAINER_HEADER.size
    for vtype in sorted(schema.types):
        ts = schema.types[vtype]
        x = ts.population
        wid = words_for(x)
        fields = [("id", wid, x)] + [(f"attr:{a}", words_for(ts.attrs[a].domain_size), ts.attrs[a].domain_size)
                                     for a in sorted(ts.attrs)]
        for key, w, _ in fields:
            layout[(vtype, key, "a")] = ((x, w), x * w)
            layout[(vtype, key, "b")] = ((x, w), x * w)
        ptypes = list(ts.posting_types)
        plen = {t: np.asarray(ts.padded_len[t], np.int64) for t in ptypes}
        for t in ptypes:
            wn = words_for(schema.types[t].population)
            lmax = ts.max_padded(t)
            layout[(vtype, f"post:{t}", "a")] = ((x, lmax, wn), x * lmax * wn)
            layout[(vtype, f"post:{t}", "b")] = ((x, lmax, wn), x * lmax * wn)
        fixed = sum(2 * (_HDR + 4 * w) for _, w, _ in fields)
        block = np.full(x, fixed, np.int64)
        for t in ptypes:
            block += 2 * plen[t] * (_HDR + 4 * words_for(schema.types[t].population))
        voff = pos + np.concatenate([[0], np.cumsum(block)[:-1]]) if x else np.zeros(0, np.int64)
        pos += int(block.sum())
        v = np.arange(x, dtype=np.int64)
        # fixed records
        off = 0
        per_vertex = []  # (offset-in-block array or scalar, key, side, width, dst)
        for key, w, bits in fields:
            for side in ("a", "b"):
                per_vertex.append((voff + off, (vtype, key, side), bits, v * w))
                off += _HDR + 4 * w
        # posting records
        cur = np.full(x, fixed, np.int64)
        for t in ptypes:
            wn = words_for(schema.types[t].population)
            lmax = ts.max_padded(t)
            rec = _HDR + 4 * wn
            n = plen[t]
            vv = np.repeat(v, n)
            slot = np.arange(int(n.sum()), dtype=np.int64) - np.repeat(np.concatenate([[0], np.cumsum(n)[:-1]]), n) \
                if n.sum() else np.zeros(0, np.int64)
            start = voff[vv] + cur[vv] + slot * 2 * rec
            for si, side in enumerate(("a", "b")):
                per_vertex.append((start + si * rec, (vtype, f"post:{t}", side), schema.types[t].population,
                                   (vv * lmax + slot) * wn))
            cur += 2 * n * rec
        for h, key, bits, d in per_vertex:
            hdr.append(np.asarray(h, np.int64))
            width.append(np.full(len(d), bits, np.int64))
            mat.append([key] * len(d))
            dst.append(np.asarray(d, np.int64))
    return hdr, width, mat, dst, layout, pos


def _container_party(buf: bytes, magic: bytes, schema: GraphSchema, kind: str) -> int:
    """Check a container header (src/storage.py:108-127, 255-268): length,
    magic, version and schema digest; returns the party index.  ``kind`` is
    "graph" or "result" (the error texts differ as in the reference)."""
    noun = {"graph": ("graph share", "graph share file", "graph share"),
            "result": ("result share", "result file", "result file")}[kind]
    if len(buf) < _CONTAINER_HEADER.size:
        raise StorageError(f"truncated {noun[1]}")
    got_magic, version, party, digest = _CONTAINER_HEADER.unpack_from(buf, 0)
    for ok, msg in ((got_magic == magic, f"not a {noun[0]} file"),
                    (version == VERSION, f"unsupported {noun[2]} version {version}"),
                    (digest == schema.digest(), f"{noun[2]} does not match the schema sidecar")):
        if not ok:
            raise StorageError(msg)
    return party


def load_graph_share(path, schema: GraphSchema, device="cuda") -> GraphShare:
    """src/storage.py:110-169; returns a GraphShare whose matrices live in HBM
    (``device=None``: host numpy, parsed the same way)."""
    buf = Path(path).read_bytes()
    party = _container_party(buf, GRAPH_MAGIC, schema, "graph")
    hdr, width, mats, dsts, layout, end = _record_table(schema)
    if end != len(buf):
        raise StorageError("trailing bytes in graph share file" if end < len(buf) else "truncated graph share file")
    b = np.frombuffer(buf, np.uint8)
    # arena: all matrices back to back
    keys = list(layout)
    base, total = {}, 0
    for k in keys:
        base[k] = total
        total += layout[k][1]
    H = np.concatenate(hdr) if hdr else np.zeros(0, np.int64)
    W = np.concatenate(width) if width else np.zeros(0, np.int64)
    D = np.concatenate([dsts[i] + base[mats[i][0]] if len(dsts[i]) else dsts[i] for i in range(len(dsts))]) \
        if dsts else np.zeros(0, np.int64)
    if H.size:
        if not (b[H[:, None] + np.arange(4)] == np.frombuffer(SHARE_MAGIC, np.uint8)).all():
            raise StorageError("bad share record magic")
        ver = b[H + 4].astype(np.int64) | (b[H + 5].astype(np.int64) << 8)
        if (ver != VERSION).any():
            raise StorageError("unsupported share record version")
        if (b[H + 6] != party).any():
            raise StorageError("record party index mismatch")
        nbits = (b[H[:, None] + 7 + np.arange(8)].astype(np.uint64) << (8 * np.arange(8, dtype=np.uint64))).sum(1)
        if (nbits != W.astype(np.uint64)).any():
            raise StorageError("record width does not match the schema")
    nw = ((W + 31) // 32).astype(np.int32)
    src = H + _HDR
    if device is None:
        arena = np.zeros(total, np.uint32)
        for s, d, n in zip(src, D, nw):
            arena[d:d + n] = np.frombuffer(buf, np.uint32, count=int(n), offset=int(s))
        view = lambda k: arena[base[k]:base[k] + layout[k][1]].reshape(layout[k][0])  # noqa: E731
    else:
        dev = torch.device(device)
        pad = (-len(buf)) % 4
        blob = torch.from_numpy(np.frombuffer(buf + b"\0" * pad, np.uint8).copy()).to(dev)
        arena = torch.zeros(max(total, 1), dtype=torch.int32, device=dev)
        t_src = torch.from_numpy(src).to(dev)
        t_dst = torch.from_numpy(D).to(dev)
        t_nw = torch.from_numpy(nw).to(dev)
        _lib.call("ogm_unpack_records", _lib.ptr(blob), len(buf), int(src.size), _lib.ptr(t_src), _lib.ptr(t_dst),
                  _lib.ptr(t_nw), _lib.ptr(arena), _lib.stream_ptr())
        view = lambda k: arena[base[k]:base[k] + layout[k][1]].view(layout[k][0])  # noqa: E731
    types = {}
    for vtype in sorted(schema.types):
        ts = schema.types[vtype]
        types[vtype] = TypePartyShare(
            view((vtype, "id", "a")), view((vtype, "id", "b")),
            {a: (view((vtype, f"attr:{a}", "a")), view((vtype, f"attr:{a}", "b"))) for a in sorted(ts.attrs)},
            {t: (view((vtype, f"post:{t}", "a")), view((vtype, f"post:{t}", "b"))) for t in ts.posting_types})
    return GraphShare(party, schema, types)


# ---------------------------------------------------------------------------
# result containers (src/storage.py:175-251)
# ---------------------------------------------------------------------------


def save_results(path, results: MatchResultSet, schema: GraphSchema) -> None:
    manifest = {"structure": results.structure,
                "records": [[{"parent_slot": r.parent_slot, "parent_record": r.parent_record} for r in recs]
                            for recs in results.records],
                "subgraphs": [list(sg) for sg in results.subgraphs]}
    blob = json.dumps(manifest, sort_keys=True, separators=(",", ":")).encode()
    parts = [_CONTAINER_HEADER.pack(RESULT_MAGIC, VERSION, results.party_index, schema.digest()),
             struct.pack("<I", len(blob)), blob]
    for recs in results.records:
        for rec in recs:
            parts.append(encode_share_vector(results.party_index, rec.vertex_id.share_a))
            parts.append(encode_share_vector(results.party_index, rec.vertex_id.share_b))
            for a in sorted(rec.attrs):
                parts.append(encode_share_vector(results.party_index, rec.attrs[a].share_a))
                parts.append(encode_share_vector(results.party_index, rec.attrs[a].share_b))
    Path(path).write_bytes(b"".join(parts))


def load_results(path, schema: GraphSchema, device="cuda") -> MatchResultSet:
    buf = Path(path).read_bytes()
    party = _container_party(buf, RESULT_MAGIC, schema, "result")
    (json_len,) = struct.unpack_from("<I", buf, _CONTAINER_HEADER.size)
    pos = _CONTAINER_HEADER.size + 4 + json_len
    try:
        manifest = json.loads(buf[pos - json_len:pos].decode())
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise StorageError(f"corrupt result manifest: {exc}") from None

    def next_shared(w: int):
        nonlocal pos
        p1, va, pos = decode_share_vector(buf, pos)
        p2, vb, pos = decode_share_vector(buf, pos)
        if p1 != party or p2 != party:
            raise StorageError("record party index mismatch")
        if va.logical_len != w or vb.logical_len != w:
            raise StorageError("record width does not match the schema")
        return SharedBitVector(party, DBits.from_host(va, device), DBits.from_host(vb, device))

    def record(ts, needed: list, meta: dict) -> MatchedRecord:
        vid = next_shared(ts.population)   # the id first, then the attributes in name order
        return MatchedRecord(meta["parent_slot"], meta["parent_record"], vid,
                             {a: next_shared(ts.attrs[a].domain_size) for a in needed})

    slots = manifest["structure"]["slots"]
    records = [[record(schema.types[slot["type"]], sorted({p["attr"] for p in slot["preds"]}), meta)
                for meta in metas] for slot, metas in zip(slots, manifest["records"])]
    if pos != len(buf):
        raise StorageError("trailing bytes in result file")
    return MatchResultSet(party, manifest["structure"], records, [tuple(sg) for sg in manifest["subgraphs"]])
