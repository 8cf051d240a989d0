"""CPU oracle for the OblivGM hot path -- TEST INFRASTRUCTURE, never the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  It
restates the reference algorithm (``/root/reference/pkg/src/oblivgm``,
abbreviated ``src/``) in plain C (``ogm_oracle.c``, loaded through ctypes)
plus small numpy helpers, each citing the reference line it follows.

Parity of the restatement is pinned against the live reference by
``tests/golden/make_golden.py`` (fixtures committed under ``tests/golden/``)
and checked by ``tests/test_oracle_golden.py``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libogm_oracle.so"

_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)

_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with its own Makefile (gcc; seconds)."""
    src = HERE / "ogm_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "-B", "libogm_oracle.so"], check=True,
                       stdout=subprocess.DEVNULL)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        L.ogm_or_prg_expand.argtypes = [_u8p, ctypes.c_int64, _u8p, _u8p, _u8p, _u8p, _u8p]
        L.ogm_or_prf_stream.argtypes = [_u8p, _u8p, ctypes.c_uint64, ctypes.c_uint64, _u8p,
                                        ctypes.c_int64]
        L.ogm_or_seeded_permutation.argtypes = [_u8p, _u8p, ctypes.c_uint64, ctypes.c_int64, _i64p]
        L.ogm_or_tree_gen.argtypes = [ctypes.c_uint64, ctypes.c_int, _u8p, _u8p, ctypes.c_int,
                                      _u8p, _u8p, _u8p]
        L.ogm_or_tree_gen_batch.argtypes = [ctypes.c_int64, ctypes.c_int, _u64p, _u8p, _u8p,
                                            ctypes.c_int, _u8p, _u8p, _u8p, ctypes.c_int]
        L.ogm_or_eval_points.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, _u8p, _u8p,
                                         _u8p, _u8p, _u8p, _u8p, _u64p, _u8p, ctypes.c_int]
        L.ogm_or_eval_points.restype = ctypes.c_int
        L.ogm_or_full_domain.argtypes = [ctypes.c_int, ctypes.c_int, _u8p, ctypes.c_int, _u8p,
                                         _u8p, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _u32p]
        L.ogm_or_full_domain.restype = ctypes.c_int
        L.ogm_or_masked_parity.argtypes = [_u32p, _u32p, ctypes.c_int64, ctypes.c_int64, _u32p,
                                           _u32p, _u8p]
        L.ogm_or_aes128_expand.argtypes = [_u8p, _u32p]
        L.ogm_or_aes128_encrypt.argtypes = [_u32p, _u8p, _u8p]
        _lib = L
    return _lib


def _p(arr, typ):
    return arr.ctypes.data_as(typ)


def _buf(b: bytes) -> np.ndarray:
    return np.frombuffer(bytes(b), dtype=np.uint8).copy()


# ---------------------------------------------------------------------------
# AES / PRG / PRF / permutation  (src/prf.py)
# ---------------------------------------------------------------------------


def aes128_encrypt_blocks(key: bytes, data: bytes) -> bytes:
    rk = np.zeros(44, np.uint32)
    lib().ogm_or_aes128_expand(_p(_buf(key), _u8p), _p(rk, _u32p))
    src = _buf(data)
    out = np.zeros_like(src)
    for i in range(0, len(src), 16):
        lib().ogm_or_aes128_encrypt(_p(rk, _u32p), _p(src[i:], _u8p), _p(out[i:], _u8p))
    return out.tobytes()


def prg_expand(seeds: np.ndarray):
    """src/prf.py:41-57 -- same signature and return layout as the reference."""
    seeds = np.ascontiguousarray(seeds, dtype=np.uint64).reshape(-1, 2)
    n = seeds.shape[0]
    left = np.zeros((n, 2), np.uint64)
    right = np.zeros((n, 2), np.uint64)
    tl = np.zeros(n, np.uint8)
    tr = np.zeros(n, np.uint8)
    v = np.zeros(n, np.uint8)
    lib().ogm_or_prg_expand(_p(seeds.view(np.uint8), _u8p), n, _p(left.view(np.uint8), _u8p),
                            _p(right.view(np.uint8), _u8p), _p(tl, _u8p), _p(tr, _u8p),
                            _p(v, _u8p))
    return left, right, tl, tr, v


def prf_stream(key: bytes, label: bytes, index: int, nbytes: int, block_offset: int = 0) -> bytes:
    """src/prf.py:70-84 (block_offset 0 is the reference call)."""
    if nbytes == 0:
        return b""
    out = np.zeros(nbytes, np.uint8)
    lib().ogm_or_prf_stream(_p(_buf(key), _u8p), _p(_buf(label), _u8p), index, block_offset,
                            _p(out, _u8p), nbytes)
    return out.tobytes()


def words_for(nbits: int) -> int:
    return (nbits + 31) // 32


def mask_tail(words: np.ndarray, nbits: int) -> np.ndarray:
    """src/bits.py:24-29."""
    rem = nbits % 32
    if rem and words.size:
        words[..., -1] &= np.uint32((1 << rem) - 1)
    return words


def prf_words(key: bytes, label: bytes, index: int, nbits: int) -> np.ndarray:
    """src/prf.py:87-92."""
    nw = words_for(nbits)
    w = np.frombuffer(prf_stream(key, label, index, 4 * nw), dtype=np.uint32).copy()
    return mask_tail(w, nbits)


def seeded_permutation(key: bytes, label: bytes, index: int, n: int) -> np.ndarray:
    """src/prf.py:95-105."""
    perm = np.zeros(n, np.int64)
    if n == 0:
        return perm
    lib().ogm_or_seeded_permutation(_p(_buf(key), _u8p), _p(_buf(label), _u8p), index, n,
                                    _p(perm, _i64p))
    return perm


def zero_share(key_own: bytes, key_prev: bytes, counter: int, nbits: int) -> np.ndarray:
    """src/rss.py:143-148 ZeroShareContext.next_share at counter ``counter``."""
    w = prf_words(key_own, b"ZSHR", counter, nbits) ^ prf_words(key_prev, b"ZSHR", counter, nbits)
    return mask_tail(w, nbits)


# ---------------------------------------------------------------------------
# FSS (src/fss.py)
# ---------------------------------------------------------------------------


class TreeKey:
    """Key-major restatement of DpfKey/DcfKey (src/fss.py:55-70) for a batch."""

    def __init__(self, bits, comparison, root, root_t, seed_cw, ctrl_cw, final_cw, add_const):
        self.bits = int(bits)
        self.comparison = bool(comparison)
        self.root = np.ascontiguousarray(root, np.uint8).reshape(-1, 16)
        k = self.root.shape[0]
        self.root_t = np.ascontiguousarray(root_t, np.uint8).reshape(k)
        self.seed_cw = np.ascontiguousarray(seed_cw, np.uint8).reshape(k, self.bits, 16)
        self.ctrl_cw = np.ascontiguousarray(ctrl_cw, np.uint8).reshape(k, self.bits)
        self.final_cw = np.ascontiguousarray(final_cw, np.uint8).reshape(k)
        self.add_const = np.ascontiguousarray(add_const, np.uint8).reshape(k)

    @property
    def count(self) -> int:
        return self.root.shape[0]


def tree_gen_batch(alphas, bits: int, roots0, roots1, comparison: bool, nthreads: int = 0):
    """Batched src/fss.py:116-157 with injected roots.  Returns (k0, k1) TreeKeys."""
    alphas = np.ascontiguousarray(alphas, np.uint64)
    k = alphas.size
    r0 = np.ascontiguousarray(roots0, np.uint8).reshape(k, 16)
    r1 = np.ascontiguousarray(roots1, np.uint8).reshape(k, 16)
    scw = np.zeros((k, bits, 16), np.uint8)
    ccw = np.zeros((k, bits), np.uint8)
    fin = np.zeros(k, np.uint8)
    nt = nthreads or (os.cpu_count() or 1)
    lib().ogm_or_tree_gen_batch(k, bits, _p(alphas, _u64p), _p(r0, _u8p), _p(r1, _u8p),
                                int(comparison), _p(scw, _u8p), _p(ccw, _u8p), _p(fin, _u8p), nt)
    zero = np.zeros(k, np.uint8)
    k0 = TreeKey(bits, comparison, r0, zero, scw, ccw, fin, zero)
    k1 = TreeKey(bits, comparison, r1, np.ones(k, np.uint8), scw, ccw, fin, zero)
    return k0, k1


def eval_points(key: TreeKey, points, nthreads: int = 0) -> np.ndarray:
    """src/fss.py:257-281 for every (key, point) pair; returns uint8 0/1."""
    pts = np.ascontiguousarray(points, np.uint64).reshape(key.count)
    out = np.zeros(key.count, np.uint8)
    nt = nthreads or (os.cpu_count() or 1)
    rc = lib().ogm_or_eval_points(key.bits, int(key.comparison), key.count, _p(key.root, _u8p),
                                  _p(key.root_t, _u8p), _p(key.seed_cw, _u8p),
                                  _p(key.ctrl_cw, _u8p), _p(key.final_cw, _u8p),
                                  _p(key.add_const, _u8p), _p(pts, _u64p), _p(out, _u8p), nt)
    if rc != 0:
        raise ValueError("point outside the key domain")
    return out


def full_domain(key: TreeKey, index: int, n: int) -> np.ndarray:
    """src/fss.py:302-337 for key ``index`` of the batch; packed words."""
    out = np.zeros(words_for(n), np.uint32)
    rc = lib().ogm_or_full_domain(key.bits, int(key.comparison), _p(key.root[index], _u8p),
                                  int(key.root_t[index]), _p(key.seed_cw[index], _u8p),
                                  _p(key.ctrl_cw[index], _u8p), int(key.final_cw[index]),
                                  int(key.add_const[index]), n, _p(out, _u32p))
    if rc != 0:
        raise ValueError("domain too small")
    return out


def key_from_reference(ref_key) -> TreeKey:
    """Lift a reference DpfKey/DcfKey object (src/fss.py:55-70) into a 1-key batch."""
    comparison = type(ref_key).__name__ == "DcfKey"
    return TreeKey(ref_key.domain_bits, comparison,
                   np.frombuffer(ref_key.root_seed, np.uint8), [ref_key.root_t],
                   np.ascontiguousarray(ref_key.seed_cw, np.uint64).view(np.uint8),
                   ref_key.ctrl_cw, [ref_key.final_cw], [ref_key.add_const])


# ---------------------------------------------------------------------------
# Engine / shuffle restatements (numpy over the C primitives)
# ---------------------------------------------------------------------------


def masked_parity(da, db, ia, ib) -> np.ndarray:
    """src/engine.py:76-80 + :162 additive bit per candidate."""
    da = np.ascontiguousarray(da, np.uint32)
    db = np.ascontiguousarray(db, np.uint32)
    rows, w = da.shape
    out = np.zeros(rows, np.uint8)
    lib().ogm_or_masked_parity(_p(da, _u32p), _p(db, _u32p), rows, w,
                               _p(np.ascontiguousarray(ia, np.uint32), _u32p),
                               _p(np.ascontiguousarray(ib, np.uint32), _u32p), _p(out, _u8p))
    return out


def pack_bits(bits: np.ndarray) -> np.ndarray:
    """src/bits.py:32-41."""
    bits = np.ascontiguousarray(bits, np.uint8)
    n = bits.shape[-1]
    pad = (-n) % 32
    if pad:
        bits = np.concatenate([bits, np.zeros(bits.shape[:-1] + (pad,), np.uint8)], axis=-1)
    packed = np.packbits(bits, axis=-1, bitorder="little")
    return packed.view(np.uint32).reshape(bits.shape[:-1] + (words_for(n),))


def unpack_bits(words: np.ndarray, nbits: int) -> np.ndarray:
    """src/bits.py:44-49."""
    words = np.ascontiguousarray(words, np.uint32)
    return np.unpackbits(words.view(np.uint8), axis=-1, bitorder="little")[..., :nbits]


def blind_table(seed: bytes, label: bytes, table_id: int, rows: int, width: int) -> np.ndarray:
    """src/shuffle.py:69-73."""
    nw = rows * words_for(width)
    mat = np.frombuffer(prf_stream(seed, label, table_id, nw * 4), np.uint32)
    return mask_tail(mat.reshape(rows, words_for(width)).copy(), width)


def shuffle_trio(s12: bytes, s23: bytes, s31: bytes, tid: int, comps, width: int):
    """src/shuffle.py:80-144 for all three parties at once.

    ``comps`` = (x1, x2, x3) share components; party i holds (x_i, x_{i+1}).
    Returns the new components (R1, R2, R3) and the three wire messages
    (x1 from P1, y1 and c1 from P2, R3 from P3)."""
    x1c, x2c, x3c = (np.ascontiguousarray(c, np.uint32) for c in comps)
    rows = x1c.shape[0]
    pi12 = seeded_permutation(s12, b"SHPI", tid, rows)
    pi23 = seeded_permutation(s23, b"SHPI", tid, rows)
    pi31 = seeded_permutation(s31, b"SHPI", tid, rows)
    t12 = blind_table(s12, b"SHTB", tid, rows, width)
    t23 = blind_table(s23, b"SHTB", tid, rows, width)
    t31 = blind_table(s31, b"SHTB", tid, rows, width)
    r1 = blind_table(s31, b"SHRD", tid, rows, width)
    r2 = blind_table(s12, b"SHRD", tid, rows, width)
    # P1 (src/shuffle.py:106-116)
    msg_x1 = ((x1c ^ x2c ^ t12)[pi12] ^ t31)[pi31]
    # P2 (src/shuffle.py:117-130)
    msg_y1 = (x3c ^ t12)[pi12]
    msg_c1 = (msg_x1 ^ t23)[pi23] ^ r2
    # P3 (src/shuffle.py:131-143)
    c2 = ((msg_y1 ^ t31)[pi31] ^ t23)[pi23] ^ r1
    r3 = msg_c1 ^ c2
    return (r1, r2, r3), (msg_x1, msg_y1, msg_c1, r3)


def fetch_multi_trio(s12: bytes, s23: bytes, s31: bytes, tid: int, flag_comps, id_comps, id_width: int):
    """src/engine.py:220-270 (sec_fetch_multi with ``attrs={}``) for all three
    parties at once: rows = flag bit ‖ id bits (src/engine.py:227-237, bit 0 =
    flag), one shuffle of table id ``tid`` (src/shuffle.py:80-144), open the
    flag column (src/rss.py:184-206: plain = R1 ^ R2 ^ R3), keep the flagged
    rows in order and slice the id back out (src/engine.py:249-269).

    ``flag_comps`` = three packed bit vectors, ``id_comps`` = three (rows,
    words_for(id_width)) matrices.  Returns (kept row indices, opened flag
    bits (rows,), [id share component c of every kept row for c = 0, 1, 2])."""
    rows = int(np.asarray(id_comps[0]).shape[0])
    width = 1 + id_width
    comps = []
    for f, ids in zip(flag_comps, id_comps):
        fbits = unpack_bits(np.asarray(f, np.uint32), rows)
        ibits = unpack_bits(np.asarray(ids, np.uint32).reshape(rows, -1), id_width)
        comps.append(pack_bits(np.concatenate([fbits[:, None], ibits], axis=1)))
    (r1, r2, r3), _ = shuffle_trio(s12, s23, s31, tid, comps, width)
    plain = ((r1 ^ r2 ^ r3)[:, 0] & 1).astype(np.uint8)
    keep = np.nonzero(plain)[0]
    recs = [pack_bits(unpack_bits(m[keep], width)[:, 1:]) for m in (r1, r2, r3)]
    return keep, plain, recs
