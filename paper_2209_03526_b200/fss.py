"""Function secret sharing with output group Z2 (src/fss.py), on the B200.

Same key types, key-generation signatures and evaluation functions as the
reference; key generation and every evaluation run in the sm_100a kernels of
``libogm_b200.so`` (``ogm_fss_gen``, ``ogm_fss_eval_points``,
``ogm_fss_full_domain``).  Key generation draws its two root seeds with
``rng.bytes(16)`` exactly as src/fss.py:117-118 does, so a generator in the
same state yields byte-identical keys.

Bulk work goes through :class:`KeyBatch`: a structure-of-arrays,
level-major device layout (include/oblivgm_b200.h) in which thread k of a
warp reads key k with coalesced 128-bit loads.
"""

from __future__ import annotations

import functools
import itertools
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .bits import BitVector, words_for
from .errors import DomainError

KIND_EQ = "eq"
KIND_LT = "lt"
KIND_LE = "le"
KIND_GT = "gt"
KIND_GE = "ge"
KIND_INTERVAL = "iv"
COMPARISON_KINDS = (KIND_LT, KIND_LE, KIND_GT, KIND_GE)
PREDICATE_KINDS = (KIND_EQ,) + COMPARISON_KINDS + (KIND_INTERVAL,)

SEED_BYTES = 16
MAX_DEVICE_BITS = 32

_TAG_DPF = 1
_TAG_DCF = 2
_TAG_INTERVAL = 3


def domain_bits_for(domain_size: int) -> int:
    """src/fss.py:48-52."""
    if domain_size < 1:
        raise DomainError("domain size must be positive")
    return max(1, (domain_size - 1).bit_length())


@dataclass(frozen=True, eq=False)
class DpfKey:
    """One party's point-function key (src/fss.py:55-65)."""

    domain_bits: int
    root_seed: bytes
    root_t: int
    seed_cw: np.ndarray  # (levels, 2) uint64
    ctrl_cw: np.ndarray  # (levels,) uint8: bit0 tau_left, bit1 tau_right, bit2 value
    final_cw: int
    add_const: int = 0


@dataclass(frozen=True, eq=False)
class DcfKey(DpfKey):
    """One party's comparison key (x < threshold) (src/fss.py:68-70)."""


@dataclass(frozen=True, eq=False)
class IntervalKey:
    """Containment key (src/fss.py:73-84)."""

    lower: DcfKey
    upper: DcfKey
    closed_low: bool = True
    closed_high: bool = True

    @property
    def domain_bits(self) -> int:
        return self.lower.domain_bits


@dataclass(frozen=True)
class FssKeyBundle:
    """Three independent key pairs for one private predicate (src/fss.py:90-108)."""

    predicate_kind: str
    pairs: tuple

    def __post_init__(self):
        if self.predicate_kind not in PREDICATE_KINDS:
            raise ValueError(f"unknown predicate kind {self.predicate_kind!r}")
        if len(self.pairs) != 3:
            raise ValueError("a bundle holds exactly three key pairs")
        if len(set(k.domain_bits for k in itertools.chain.from_iterable(self.pairs))) > 1:
            raise ValueError("all six keys must share domain_bits")

    @property
    def domain_bits(self) -> int:
        first, _ = self.pairs[0]
        return first.domain_bits


def is_comparison(key) -> bool:
    # duck-typed so reference key objects (src/fss.py:68) are accepted too
    return type(key).__name__ == "DcfKey"


# ---------------------------------------------------------------------------
# device key batches
# ---------------------------------------------------------------------------


def pack_keys(keys: list, bits: int) -> np.ndarray:
    """Host image of a KeyBatch, one buffer for one H2D copy:
    root (n,16) | seed_cw (bits,n,16) | ctrl (3,n) u32 bit-planes over levels
    | flags (n,) u8 (bit0 root_t, bit1 final_cw, bit2 add_const).  Every
    offset is a multiple of 16 bytes except the trailing flags."""
    n = len(keys)
    a, b = 16 * n, 16 * n * (1 + bits)
    buf = np.empty(b + 12 * n + n, np.uint8)
    buf[:a] = np.frombuffer(b"".join([k.root_seed for k in keys]), np.uint8)
    scw = np.frombuffer(b"".join([np.ascontiguousarray(k.seed_cw, np.uint64).tobytes() for k in keys]),
                        np.uint8).reshape(n, bits, 16)
    buf[a:b].reshape(bits, n, 16)[...] = scw.transpose(1, 0, 2)
    cc = np.frombuffer(b"".join([np.asarray(k.ctrl_cw, np.uint8).tobytes() for k in keys]),
                       np.uint8).reshape(n, bits)
    planes = (cc[None, :, :] >> np.arange(3, dtype=np.uint8)[:, None, None]) & 1   # (3, n, bits)
    packed = np.zeros((3, n, 4), np.uint8)
    packed[:, :, :(bits + 7) // 8] = np.packbits(planes, axis=2, bitorder="little")
    buf[b:b + 12 * n] = packed.reshape(-1)
    buf[b + 12 * n:] = [(k.root_t & 1) | ((k.final_cw & 1) << 1) | ((k.add_const & 1) << 2) for k in keys]
    return buf


class KeyBatch:
    """K tree keys of one kind and depth in the device SoA layout.

    root (K,16) u8 | seed_cw (bits,K,16) u8 | ctrl (3,K) i32 | flags (K,) u8
    (flags: bit0 root_t, bit1 final_cw, bit2 add_const).
    """

    def __init__(self, kind: int, bits: int, root, seed_cw, ctrl, flags):
        if not 1 <= bits <= MAX_DEVICE_BITS:
            raise DomainError(f"domain_bits {bits} outside 1..{MAX_DEVICE_BITS}")
        self.kind = kind
        self.bits = bits
        self.root = root
        self.seed_cw = seed_cw
        self.ctrl = ctrl
        self.flags = flags

    @property
    def count(self) -> int:
        return self.root.shape[0]

    @property
    def comparison(self) -> bool:
        return self.kind == _lib.KIND_DCF

    @classmethod
    def from_keys(cls, keys, device="cuda") -> "KeyBatch":
        """Pack DpfKey/DcfKey objects (all of one kind and depth)."""
        keys = list(keys)
        if not keys:
            raise ValueError("empty key batch")
        bits = keys[0].domain_bits
        comp = is_comparison(keys[0])
        for k in keys:
            if k.domain_bits != bits or is_comparison(k) != comp:
                raise ValueError("a key batch needs one kind and one domain size")
        if not 1 <= bits <= MAX_DEVICE_BITS:
            raise DomainError(f"domain_bits {bits} outside 1..{MAX_DEVICE_BITS}")
        n = len(keys)
        buf = pack_keys(keys, bits)
        a, b = 16 * n, 16 * n * (1 + bits)
        dev = torch.device(device)
        host = torch.from_numpy(buf)
        if dev.type == "cuda":
            # pinned + non-blocking: a pageable copy would synchronise the stream on every batch
            d = host.pin_memory().to(dev, non_blocking=True)
        else:
            d = host.to(dev)
        return cls(_lib.KIND_DCF if comp else _lib.KIND_DPF, bits, d[:a].view(n, 16), d[a:b].view(bits, n, 16),
                   d[b:b + 12 * n].view(torch.int32).view(3, n), d[b + 12 * n:])

    def to_keys(self) -> list:
        """Unpack into DpfKey/DcfKey objects (host)."""
        root = self.root.cpu().numpy()
        scw = self.seed_cw.cpu().numpy()
        ctrl = self.ctrl.cpu().numpy().view(np.uint32)
        flags = self.flags.cpu().numpy()
        lv = np.arange(self.bits, dtype=np.uint32)
        cls = DcfKey if self.comparison else DpfKey
        out = []
        for k in range(self.count):
            cc = (((ctrl[0, k] >> lv) & 1) | (((ctrl[1, k] >> lv) & 1) << 1)
                  | (((ctrl[2, k] >> lv) & 1) << 2)).astype(np.uint8)
            out.append(cls(domain_bits=self.bits, root_seed=root[k].tobytes(),
                           root_t=int(flags[k] & 1),
                           seed_cw=np.ascontiguousarray(scw[:, k, :]).view(np.uint64).reshape(self.bits, 2).copy(),
                           ctrl_cw=cc, final_cw=int((flags[k] >> 1) & 1),
                           add_const=int((flags[k] >> 2) & 1)))
        return out


def gen_batch(comparison: bool, bits: int, alphas: torch.Tensor, roots0: torch.Tensor,
              roots1: torch.Tensor) -> tuple[KeyBatch, KeyBatch]:
    """Batched src/fss.py:116-157 on the device (injected roots).

    alphas: (K,) int32/uint32 device tensor; roots0/roots1: (K,16) uint8.
    Returns the two parties' batches (root_t 0 and 1, shared corrections).
    """
    if not 1 <= bits <= MAX_DEVICE_BITS:
        raise DomainError(f"domain_bits {bits} outside 1..{MAX_DEVICE_BITS}")
    k = alphas.numel()
    dev = alphas.device
    scw = torch.empty((bits, k, 16), dtype=torch.uint8, device=dev)
    ctrl = torch.empty((3, k), dtype=torch.int32, device=dev)
    f0 = torch.empty((k,), dtype=torch.uint8, device=dev)
    f1 = torch.empty((k,), dtype=torch.uint8, device=dev)
    kind = _lib.KIND_DCF if comparison else _lib.KIND_DPF
    _lib.call("ogm_fss_gen_pair", kind, bits, k, _lib.ptr(alphas), _lib.ptr(roots0), _lib.ptr(roots1),
              _lib.ptr(scw), _lib.ptr(ctrl), _lib.ptr(f0), _lib.ptr(f1), _lib.stream_ptr())
    return (KeyBatch(kind, bits, roots0, scw, ctrl, f0), KeyBatch(kind, bits, roots1, scw, ctrl, f1))


def eval_points(batch: KeyBatch, points: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """src/fss.py:257-299 for every (key k, points[k]); packed output bits."""
    k = batch.count
    if points.numel() != k:
        raise ValueError("one point per key is required")
    if out is None:
        out = torch.empty((words_for(k),), dtype=torch.int32, device=points.device)
    if batch.bits < 32:
        # the reference raises DomainError for x outside 2^bits (src/fss.py:259-260)
        if bool(((points.to(torch.int64) & 0xFFFFFFFF) >> batch.bits).any()):
            raise DomainError(f"point outside 2^{batch.bits} domain")
    _lib.call("ogm_fss_eval_points", batch.kind, batch.bits, k, _lib.ptr(batch.root),
              _lib.ptr(batch.seed_cw), _lib.ptr(batch.ctrl), _lib.ptr(batch.flags), _lib.ptr(points),
              _lib.ptr(out), _lib.stream_ptr())
    return out


def full_domain(batch: KeyBatch, n: int, out: torch.Tensor | None = None) -> torch.Tensor:
    """src/fss.py:302-337 for every key of the batch: (K, words(n)) packed."""
    if n > (1 << batch.bits):
        raise DomainError(f"requested {n} points from a 2^{batch.bits} domain")
    w = words_for(n)
    if out is None:
        # 16-byte row pitch so every key's indicator row feeds 128-bit loads
        pitch = (w + 3) // 4 * 4
        out = torch.empty((batch.count, pitch), dtype=torch.int32, device=batch.root.device)[:, :w]
    _lib.call("ogm_fss_full_domain", batch.kind, batch.bits, batch.count, _lib.ptr(batch.root),
              _lib.ptr(batch.seed_cw), _lib.ptr(batch.ctrl), _lib.ptr(batch.flags), n, _lib.ptr(out),
              out.stride(0), _lib.stream_ptr())
    return out


# ---------------------------------------------------------------------------
# reference-shaped key generation (src/fss.py:160-249)
# ---------------------------------------------------------------------------


def _tree_gen(alpha: int, bits: int, rng: np.random.Generator, comparison: bool):
    """src/fss.py:116-157: same rng draws, evaluated on the device."""
    root0 = rng.bytes(SEED_BYTES)
    root1 = rng.bytes(SEED_BYTES)
    if not 1 <= bits <= MAX_DEVICE_BITS:
        raise DomainError(f"domain_bits {bits} outside 1..{MAX_DEVICE_BITS}")
    dev = torch.device("cuda")
    a = torch.tensor([alpha], dtype=torch.int64).to(torch.int32).to(dev)
    r0 = torch.frombuffer(bytearray(root0), dtype=torch.uint8).reshape(1, 16).to(dev)
    r1 = torch.frombuffer(bytearray(root1), dtype=torch.uint8).reshape(1, 16).to(dev)
    b0, b1 = gen_batch(comparison, bits, a, r0, r1)
    k0 = b0.to_keys()[0]
    k1 = b1.to_keys()[0]
    return k0, k1


def dpf_gen(alpha: int, domain_size: int, rng: np.random.Generator):
    """src/fss.py:160-164."""
    if not 0 <= alpha < domain_size:
        raise DomainError(f"alpha {alpha} outside domain of size {domain_size}")
    return _tree_gen(alpha, domain_bits_for(domain_size), rng, comparison=False)


def dcf_gen(alpha: int, domain_size: int, rng: np.random.Generator):
    """src/fss.py:167-171."""
    if not 0 <= alpha < domain_size:
        raise DomainError(f"alpha {alpha} outside domain of size {domain_size}")
    return _tree_gen(alpha, domain_bits_for(domain_size), rng, comparison=True)


def _with_const(key: DcfKey, const: int):
    """src/fss.py:174-185."""
    if const == 0:
        return key
    return type(key)(domain_bits=key.domain_bits, root_seed=key.root_seed, root_t=key.root_t,
                     seed_cw=key.seed_cw, ctrl_cw=key.ctrl_cw, final_cw=key.final_cw,
                     add_const=key.add_const ^ const)


def cmp_gen(kind: str, alpha: int, domain_size: int, rng: np.random.Generator):
    """src/fss.py:188-210: <, <=, >, >= via a strict tree plus a public constant."""
    if kind not in COMPARISON_KINDS:
        raise ValueError(f"not a comparison kind: {kind!r}")
    if not 0 <= alpha < domain_size:
        raise DomainError(f"alpha {alpha} outside domain of size {domain_size}")
    bits = domain_bits_for(domain_size)
    # every kind is the strict tree "x < t" plus a public constant on key 1;
    # at the top of the domain "x < 2^bits" is always true, so t wraps to 0
    # and the constant flips (src/fss.py:199-210)
    wraps = alpha + 1 == 1 << bits
    threshold, const = {KIND_LT: (alpha, 0), KIND_GE: (alpha, 1),
                        KIND_LE: (0, 1) if wraps else (alpha + 1, 0),
                        KIND_GT: (0, 0) if wraps else (alpha + 1, 1)}[kind]
    k1, k2 = _tree_gen(threshold, bits, rng, comparison=True)
    return _with_const(k1, const), k2


def ic_gen(low: int, high: int, domain_size: int, rng: np.random.Generator,
           closed_low: bool = True, closed_high: bool = True):
    """src/fss.py:213-234."""
    if low > high:
        raise DomainError(f"empty interval bounds: {low} > {high}")
    if not (0 <= low < domain_size and 0 <= high < domain_size):
        raise DomainError("interval bounds outside domain")
    bits = domain_bits_for(domain_size)
    full = 1 << bits
    lo_t = low + (0 if closed_low else 1)
    hi_t = high + (1 if closed_high else 0)
    const = 0
    if lo_t >= hi_t:
        lo_t = hi_t = 0
    if hi_t == full:
        hi_t = 0
        const = 1
    low1, low2 = _tree_gen(lo_t, bits, rng, comparison=True)
    up1, up2 = _tree_gen(hi_t, bits, rng, comparison=True)
    up1 = _with_const(up1, const)
    return (IntervalKey(low1, up1, closed_low, closed_high),
            IntervalKey(low2, up2, closed_low, closed_high))


def bundle_gen(kind: str, operands: tuple, domain_size: int, rng: np.random.Generator) -> FssKeyBundle:
    """src/fss.py:237-249: three independent pairs, generated one after the other."""
    if kind == KIND_EQ:
        make = functools.partial(dpf_gen, operands[0], domain_size, rng)
    elif kind in COMPARISON_KINDS:
        make = functools.partial(cmp_gen, kind, operands[0], domain_size, rng)
    elif kind == KIND_INTERVAL:
        make = functools.partial(ic_gen, operands[0], operands[1], domain_size, rng)
    else:
        raise ValueError(f"unknown predicate kind {kind!r}")
    return FssKeyBundle(kind, tuple(make() for _ in range(3)))


# ---------------------------------------------------------------------------
# reference-shaped evaluation (src/fss.py:257-344, 472-480)
# ---------------------------------------------------------------------------


def _walk_eval(key, x: int) -> int:
    bits = key.domain_bits
    if not 0 <= x < (1 << bits):
        raise DomainError(f"point {x} outside 2^{bits} domain")
    batch = KeyBatch.from_keys([key])
    pts = torch.tensor([x], dtype=torch.int64).to(torch.int32).cuda()
    return int(eval_points(batch, pts).cpu()[0].item()) & 1


def dpf_eval(key, x: int) -> int:
    return _walk_eval(key, x)


def dcf_eval(key, x: int) -> int:
    return _walk_eval(key, x)


def ic_eval(key: IntervalKey, x: int) -> int:
    return _walk_eval(key.lower, x) ^ _walk_eval(key.upper, x)


def eval_key(key, x: int) -> int:
    if isinstance(key, IntervalKey) or type(key).__name__ == "IntervalKey":
        return ic_eval(key, x)
    return _walk_eval(key, x)


def key_parts_for_engine(key) -> list:
    """src/fss.py:472-480."""
    if type(key).__name__ == "IntervalKey":
        return [key.lower, key.upper]
    return [key]


def full_domain_eval(key, n: int) -> BitVector:
    """src/fss.py:340-344 (host BitVector result)."""
    parts = key_parts_for_engine(key)
    for p in parts:
        if n > (1 << p.domain_bits):
            raise DomainError(f"requested {n} points from a 2^{p.domain_bits} domain")
    words = None
    for p in parts:
        w = full_domain(KeyBatch.from_keys([p]), n)[0].cpu().numpy().view(np.uint32)
        words = w if words is None else words ^ w
    return BitVector(words, n)


# ---------------------------------------------------------------------------
# serialization (src/fss.py:351-469), byte-identical wire form
# ---------------------------------------------------------------------------

# Tree key: <tag, domain_bits, add_const, root_t> + 16-byte root seed, then
# per level the 16-byte seed correction and the control byte, then final_cw.
# Interval key: <tag, domain_bits, closed flags, 0> + two length-prefixed
# tree keys (lower, upper).
_HEAD = struct.Struct("<BBBB")
_U32 = struct.Struct("<I")
_LEVEL = np.dtype([("cw", "<u8", (2,)), ("ctrl", "u1")])   # 17 bytes, packed


def _serialize_tree_key(key) -> bytes:
    levels = np.empty(key.domain_bits, dtype=_LEVEL)
    levels["cw"] = np.asarray(key.seed_cw, np.uint64).reshape(key.domain_bits, 2)
    levels["ctrl"] = np.asarray(key.ctrl_cw, np.uint8)
    tag = _TAG_DCF if is_comparison(key) else _TAG_DPF
    return b"".join((_HEAD.pack(tag, key.domain_bits, key.add_const, key.root_t), bytes(key.root_seed),
                     levels.tobytes(), bytes([key.final_cw])))


def serialize_key(key) -> bytes:
    if type(key).__name__ != "IntervalKey":
        return _serialize_tree_key(key)
    flags = int(bool(key.closed_low)) | (int(bool(key.closed_high)) << 1)
    parts = [_HEAD.pack(_TAG_INTERVAL, key.domain_bits, flags, 0)]
    for sub in (key.lower, key.upper):
        blob = _serialize_tree_key(sub)
        parts += [_U32.pack(len(blob)), blob]
    return b"".join(parts)


def _parse_tree_key(buf: bytes, offset: int = 0):
    """(key, end offset) of the tree key at ``offset``."""
    tag, bits, add_const, root_t = _HEAD.unpack_from(buf, offset)
    if tag not in (_TAG_DPF, _TAG_DCF):
        raise ValueError(f"bad key tag {tag}")
    seed_at = offset + _HEAD.size
    levels_at = seed_at + SEED_BYTES
    final_at = levels_at + bits * _LEVEL.itemsize
    if final_at + 1 > len(buf):
        raise ValueError("truncated key")
    levels = np.frombuffer(buf, dtype=_LEVEL, count=bits, offset=levels_at)
    cls = DcfKey if tag == _TAG_DCF else DpfKey
    key = cls(domain_bits=bits, root_seed=bytes(buf[seed_at:levels_at]), root_t=root_t,
              seed_cw=levels["cw"].copy(), ctrl_cw=levels["ctrl"].copy(), final_cw=buf[final_at],
              add_const=add_const)
    return key, final_at + 1


def parse_key(buf: bytes):
    if not buf:
        raise ValueError("empty key buffer")
    if buf[0] != _TAG_INTERVAL:
        key, end = _parse_tree_key(buf, 0)
        if end != len(buf):
            raise ValueError("trailing bytes after key")
        return key
    _, bits, flags, _ = _HEAD.unpack_from(buf, 0)
    subs, pos = [], _HEAD.size
    for last in (False, True):
        (declared,) = _U32.unpack_from(buf, pos)
        sub, end = _parse_tree_key(buf, pos + _U32.size)
        if end - (pos + _U32.size) != declared or (last and end != len(buf)):
            raise ValueError("interval sub-key length mismatch")
        subs.append(sub)
        pos = end
    lower, upper = subs
    if not (is_comparison(lower) and is_comparison(upper)):
        raise ValueError("interval sub-keys must be comparison keys")
    if {lower.domain_bits, upper.domain_bits} != {bits}:
        raise ValueError("interval sub-key domain mismatch")
    return IntervalKey(lower, upper, bool(flags & 1), bool(flags & 2))
