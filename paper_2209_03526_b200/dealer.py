"""Graph outsourcing straight into HBM (src/graphs.py:327-400).

``encrypt_graph(graph, k, rng, device=...)`` draws every random share
component from the same numpy generator stream the reference's host dealer
draws from -- PCG64 through ``Generator.integers(0, 2**32, dtype=uint32)``
(csrc/ogm_dealer.cuh: jump-ahead per thread, identical values) -- and builds
the three XOR share components of every one-hot matrix on the device, in
the reference's draw order (per type: ids, then attributes in name order,
then each neighbour type's posting rows).  The generator's host state is
advanced exactly as the host dealer would advance it, so tokens drawn from
the same generator afterwards are identical too.  The result is the
``graphs.device_trio`` layout: each component stored once, 16-byte row
pitch, party i holding components (i, i+1).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .bits import words_for
from .graphs import GraphShare, TypePartyShare, build_schema
from .net import next_party

_MULT = 0x2360ED051FC65DA44385DF649FCCF645
_M128 = (1 << 128) - 1
_M64 = (1 << 64) - 1


def _advance(state: int, inc: int, delta: int) -> int:
    """PCG64 state after ``delta`` LCG steps (closed-form jump)."""
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, _MULT, inc
    while delta:
        if delta & 1:
            acc_mult = acc_mult * cur_mult & _M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & _M128
        cur_plus = (cur_mult + 1) * cur_plus & _M128
        cur_mult = cur_mult * cur_mult & _M128
        delta >>= 1
    return (acc_mult * state + acc_plus) & _M128


def _output(state: int) -> int:
    """PCG64's XSL-RR output of a state."""
    rot = state >> 122
    x = ((state >> 64) ^ state) & _M64
    return ((x >> rot) | (x << ((64 - rot) & 63))) & _M64


def _u64_pair(x: int) -> np.ndarray:
    return np.array([x & _M64, x >> 64], dtype=np.uint64)


def draw_u32(rng: np.random.Generator, n: int, device) -> torch.Tensor:
    """The next ``n`` values of ``rng.integers(0, 2**32, dtype=np.uint32)``
    as a device int32 tensor, the generator advanced as if they had been
    drawn on the host."""
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("the device dealer follows numpy's PCG64 (default_rng) stream")
    out = torch.empty((max(n, 1),), dtype=torch.int32, device=device)[:n]
    if n == 0:
        return out
    s, inc = st["state"]["state"], st["state"]["inc"]
    has, buf = int(st["has_uint32"]), int(st["uinteger"])
    sp, ip = _u64_pair(s), _u64_pair(inc)
    _lib.call("ogm_pcg64_u32", sp.ctypes.data, ip.ctypes.data, has, buf, n, _lib.ptr(out), _lib.stream_ptr())
    rest = n - has
    if rest <= 0:                                   # only the buffered high half was used
        st["has_uint32"] = 0
    else:
        m = (rest + 1) // 2                         # 64-bit outputs consumed
        s_new = _advance(s, inc, m)
        st["state"]["state"] = s_new
        st["has_uint32"] = rest % 2                 # an odd count leaves the last high half buffered
        st["uinteger"] = _output(s_new) >> 32
    rng.bit_generator.state = st
    return out


def _dev_i64(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, np.int64))


class _DeviceDealer:
    """Draws a share matrix set from the generator and deals it into three
    pitched device components (ogm_deal_rows + ogm_deal_hot_bits)."""

    def __init__(self, rng: np.random.Generator, device):
        self.rng, self.dev = rng, torch.device(device)

    def deal(self, rows: int, width_words: int, drawn: np.ndarray, s1_off: np.ndarray, s2_off: np.ndarray,
             nwords: int, hot_word: np.ndarray, hot_mask: np.ndarray):
        """Rows of ``width_words`` words (16-byte pitch).  Row i's components
        are the ``drawn[i]`` words at s1_off[i] / s2_off[i] of a fresh
        ``nwords``-word draw; the plaintext bits hot_mask[j] are XORed into
        word hot_word[j] of the third component (flat index over the pitched
        matrix)."""
        pitch = (width_words + 3) // 4 * 4
        S = draw_u32(self.rng, nwords, self.dev)
        comps = [torch.empty((rows, pitch), dtype=torch.int32, device=self.dev) for _ in range(3)]
        if rows and pitch:
            up = lambda a: _dev_i64(a).to(self.dev, non_blocking=False)  # noqa: E731
            d1, d2, dn = up(s1_off), up(s2_off), up(drawn)
            _lib.call("ogm_deal_rows", _lib.ptr(S), _lib.ptr(d1), _lib.ptr(d2), _lib.ptr(dn), rows, pitch,
                      *[_lib.ptr(c) for c in comps], _lib.stream_ptr())
            if hot_word.size:
                hw = up(hot_word)
                hm = torch.from_numpy(np.ascontiguousarray(hot_mask, np.uint32).view(np.int32)).to(self.dev)
                _lib.call("ogm_deal_hot_bits", _lib.ptr(hw), _lib.ptr(hm), hot_word.size, _lib.ptr(comps[2]),
                          _lib.stream_ptr())
        return comps, pitch

    def one_hot_matrix(self, hot: np.ndarray, width_bits: int):
        """src/graphs.py:327-332 over the one-hot rows of ``hot``: s1 is the
        whole (X, w) matrix drawn first, then s2."""
        x, w = hot.size, words_for(width_bits)
        rows = np.arange(x, dtype=np.int64)
        comps, pitch = self.deal(x, w, np.full(x, w, np.int64), rows * w, x * w + rows * w, 2 * x * w,
                                 rows * ((w + 3) // 4 * 4) + hot // 32, (np.uint64(1) << (hot % 32).astype(np.uint64))
                                 .astype(np.uint32))
        return [c[:, :w] for c in comps]


def _posting_comps(dealer: _DeviceDealer, graph, ts, members: list, t_ne: str):
    """The (X, L_max, w(X_ne)) posting tensors of one neighbour type: per
    vertex row with a non-zero padded length, s1 then s2 of its (plen, w)
    rows are drawn (src/graphs.py:365-381); the slots past the vertex's
    padded length are public zeros."""
    local = {gi: li for li, gi in enumerate(graph.type_members[t_ne])}
    w = words_for(len(local))
    l_max = ts.max_padded(t_ne)
    x = len(members)
    inner = l_max * w
    pitch = (inner + 3) // 4 * 4
    plen = np.asarray(ts.padded_len[t_ne], np.int64) if x else np.zeros(0, np.int64)
    drawn = plen * w
    start = np.concatenate([[0], np.cumsum(2 * drawn)[:-1]]) if x else np.zeros(0, np.int64)
    hw, hm = [], []
    for r, gi in enumerate(members):
        for slot, ngi in enumerate(graph.posting_list(gi, t_ne)):
            li = local[ngi]
            hw.append(r * pitch + slot * w + li // 32)
            hm.append(1 << (li % 32))
    comps, _ = dealer.deal(x, inner, drawn, start, start + drawn, int(2 * drawn.sum()),
                           np.asarray(hw, np.int64), np.asarray(hm, np.uint64).astype(np.uint32))
    # rows keep their 16-byte pitch; expose (X, L_max, w) like graphs.device_trio
    return [c.as_strided((x, l_max, w), (pitch if x > 1 else max(inner, 1), w, 1)) for c in comps]


def encrypt_graph_device(graph, k: int, rng: np.random.Generator, schema=None, device="cuda"):
    """src/graphs.py:335-400 with every share drawn and dealt on the device:
    the same schema and the same share bytes as the host dealer
    (graphs.encrypt_graph) for the same generator state, in the device_trio
    layout (component j stored once; party i holds (i, i+1))."""
    if schema is None:
        schema = build_schema(graph, k)
    dealer = _DeviceDealer(rng, device)
    comps = {}
    for vtype, ts in schema.types.items():
        members = graph.type_members[vtype]
        comps[(vtype, "id", None)] = dealer.one_hot_matrix(np.arange(ts.population, dtype=np.int64), ts.population)
        for name, attr in ts.attrs.items():
            hot = np.array([attr.index_of[graph.vertices[i].attrs[name]] for i in members], dtype=np.int64)
            comps[(vtype, "attr", name)] = dealer.one_hot_matrix(hot, attr.domain_size)
        for t_ne in ts.posting_types:
            comps[(vtype, "post", t_ne)] = _posting_comps(dealer, graph, ts, members, t_ne)

    def party_share(party: int) -> GraphShare:
        a, b = party - 1, next_party(party) - 1
        types = {}
        for vtype, ts in schema.types.items():
            pair = lambda key: (comps[key][a], comps[key][b])  # noqa: E731
            ida, idb = pair((vtype, "id", None))
            types[vtype] = TypePartyShare(ida, idb, {n: pair((vtype, "attr", n)) for n in ts.attrs},
                                          {t: pair((vtype, "post", t)) for t in ts.posting_types})
        return GraphShare(party, schema, types)

    return schema, tuple(party_share(p) for p in (1, 2, 3))
