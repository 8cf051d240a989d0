"""Three-party replicated secret sharing over device bit vectors (src/rss.py).

A secret x = x1 ^ x2 ^ x3; party i holds (x_i, x_{i+1}).  Shares live in HBM
as uint32 words (:class:`DBits`); the local algebra runs in libogm_b200.so
kernels, the communicating operations (reshare, AND, open) exchange device
tensors through the runtime in :mod:`paper_2209_03526_b200.net`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .bits import BitVector, words_for
from .errors import ProtocolError
from .net import OP_OPEN, OP_RESHARE, Message, next_party, u32le

PARTIES = (1, 2, 3)


class DBits:
    """A device-resident packed bit vector: int32 words + logical length.

    Bits past ``logical_len`` are zero (the kernels keep tails clean)."""

    __slots__ = ("words", "logical_len")

    def __init__(self, words: torch.Tensor, logical_len: int):
        if words.numel() != words_for(logical_len):
            raise ValueError(f"expected {words_for(logical_len)} words for {logical_len} bits, "
                             f"got {words.numel()}")
        # a torch call here is a GIL hand-off point for the three party threads: skip it when the
        # words are already a flat vector
        self.words = words if words.dim() == 1 else words.reshape(-1)
        self.logical_len = logical_len

    @classmethod
    def from_host(cls, bv: BitVector, device=None) -> "DBits":
        t = torch.from_numpy(np.ascontiguousarray(bv.words, np.uint32).view(np.int32).copy())
        return cls(t.to(device or "cuda"), bv.logical_len)

    @classmethod
    def zeros(cls, nbits: int, device=None) -> "DBits":
        return cls(torch.zeros(words_for(nbits), dtype=torch.int32, device=device or "cuda"), nbits)

    def to_host(self) -> BitVector:
        return BitVector(self.words.detach().cpu().numpy().view(np.uint32), self.logical_len)

    def to_bits(self) -> np.ndarray:
        return self.to_host().to_bits()

    def popcount(self) -> int:
        return self.to_host().popcount()

    def hot_index(self):
        return self.to_host().hot_index()

    def _check_len(self, other: "DBits") -> None:
        if self.logical_len != other.logical_len:
            raise ValueError(f"length mismatch: {self.logical_len} vs {other.logical_len}")

    def __xor__(self, other: "DBits") -> "DBits":
        self._check_len(other)
        out = torch.empty_like(self.words)
        xor_words(self.words, other.words, None, out)
        return DBits(out, self.logical_len)

    def __len__(self) -> int:
        return self.logical_len

    def __eq__(self, other) -> bool:
        if isinstance(other, DBits):
            other = other.to_host()
        return self.to_host() == other

    def __repr__(self) -> str:
        return f"DBits({self.to_host()!r})"


def xor_words(a: torch.Tensor, b: torch.Tensor, c: torch.Tensor | None, out: torch.Tensor) -> torch.Tensor:
    _lib.call("ogm_xor_words", a.numel(), _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), _lib.ptr(out),
              _lib.stream_ptr())
    return out


def prev_party(i: int) -> int:
    return (i + 1) % 3 + 1


@dataclass(frozen=True)
class SharedBitVector:
    """One party's view (x_i, x_{i+1}) of a replicated sharing (src/rss.py:35-70)."""

    party_index: int
    share_a: DBits
    share_b: DBits

    def __post_init__(self):
        if self.party_index not in PARTIES:
            raise ValueError(f"party_index must be in {PARTIES}")
        if self.share_a.logical_len != self.share_b.logical_len:
            raise ValueError("share pair length mismatch")

    @property
    def logical_len(self) -> int:
        return self.share_a.logical_len

    def xor(self, other: "SharedBitVector") -> "SharedBitVector":
        if self.party_index != other.party_index:
            raise ValueError("cannot combine shares of different parties")
        return SharedBitVector(self.party_index, self.share_a ^ other.share_a, self.share_b ^ other.share_b)

    def xor_public(self, const) -> "SharedBitVector":
        if isinstance(const, BitVector):
            const = DBits.from_host(const, self.share_a.words.device)
        if const.logical_len != self.logical_len:
            raise ValueError("length mismatch")
        a, b = self.share_a, self.share_b
        if self.party_index == 1:
            a = a ^ const
        elif self.party_index == 3:
            b = b ^ const
        return SharedBitVector(self.party_index, a, b)

    def to_host(self):
        """Host (reference-typed) copy: (party, BitVector a, BitVector b)."""
        return self.party_index, self.share_a.to_host(), self.share_b.to_host()


def xor_local(a: SharedBitVector, b: SharedBitVector) -> SharedBitVector:
    return a.xor(b)


def share(plaintext: BitVector, rng: np.random.Generator, device=None):
    """src/rss.py:77-88 (same rng draws: s1, s2 random, s3 = x ^ s1 ^ s2)."""
    n = plaintext.logical_len
    if n == 0:
        raise ValueError("cannot share a zero-length vector")
    s1 = BitVector.random(n, rng)
    s2 = BitVector.random(n, rng)
    s3 = plaintext ^ s1 ^ s2
    parts = {i: DBits.from_host(v, device) for i, v in ((1, s1), (2, s2), (3, s3))}
    return tuple(SharedBitVector(i, parts[i], parts[next_party(i)]) for i in PARTIES)


def reconstruct(shares) -> BitVector:
    """src/rss.py:91-112 (host result)."""
    shares = list(shares)
    if not shares:
        raise ValueError("no shares given")
    n = shares[0].logical_len
    comps: dict[int, BitVector] = {}
    for sv in shares:
        if sv.logical_len != n:
            raise ValueError("length mismatch between share pairs")
        for idx, vec in ((sv.party_index, sv.share_a), (next_party(sv.party_index), sv.share_b)):
            hv = vec.to_host() if isinstance(vec, DBits) else vec
            if idx in comps:
                if comps[idx] != hv:
                    raise ValueError(f"inconsistent copies of share {idx}")
            else:
                comps[idx] = hv
    if set(comps) != set(PARTIES):
        raise ValueError(f"share indices {sorted(comps)} do not cover all of {PARTIES}")
    return comps[1] ^ comps[2] ^ comps[3]


def and_terms(a: SharedBitVector, b: SharedBitVector) -> DBits:
    """src/rss.py:115-126 local additive share of a AND b."""
    if a.party_index != b.party_index:
        raise ValueError("cannot combine shares of different parties")
    if a.logical_len != b.logical_len:
        raise ValueError("length mismatch")
    out = torch.empty_like(a.share_a.words)
    A = _lib.ptr_array
    _lib.call("ogm_and_terms", out.numel(), 1, A([a.share_a.words]), A([a.share_b.words]),
              A([b.share_a.words]), A([b.share_b.words]), A([out]), _lib.stream_ptr())
    return DBits(out, a.logical_len)


class ZeroShareContext:
    """src/rss.py:129-154: PRF-based fresh sharings of zero, counter-driven."""

    LABEL = b"ZSHR"

    def __init__(self, prf_key_own: bytes, prf_key_prev: bytes, counter: int = 0):
        self.prf_key_own = prf_key_own
        self.prf_key_prev = prf_key_prev
        self.counter = counter

    def _share(self, nbits: int, j: int, xor_into: torch.Tensor | None = None) -> DBits:
        out = torch.empty(words_for(nbits), dtype=torch.int32, device="cuda")
        if nbits:
            _lib.call("ogm_zero_share", self.prf_key_own, self.prf_key_prev, j, nbits, _lib.ptr(xor_into),
                      _lib.ptr(out), _lib.stream_ptr())
        return DBits(out, nbits)

    def next_share(self, nbits: int, xor_into: torch.Tensor | None = None) -> DBits:
        j = self.counter
        self.counter += 1
        return self._share(nbits, j, xor_into)

    def peek(self, nbits: int, j: int) -> DBits:
        return self._share(nbits, j)


def reshare(rt, additive: DBits) -> SharedBitVector:
    """src/rss.py:164-176: blind with a fresh zero share, send to next,
    receive from previous; result (received, blinded)."""
    n = additive.logical_len
    blinded = rt.zs.next_share(n, xor_into=additive.words)
    rt.send_next(OP_RESHARE, Message(b"", blinded.words), logical_bits=n)
    msg = rt.recv_prev(OP_RESHARE)
    if msg.tensor is None or msg.tensor.numel() != words_for(n):
        raise ValueError("re-share message has wrong length")
    return SharedBitVector(rt.index, DBits(msg.tensor, n), blinded)


def and_gate(rt, a: SharedBitVector, b: SharedBitVector) -> SharedBitVector:
    """src/rss.py:179-181."""
    return reshare(rt, and_terms(a, b))


def open_shared(rt, x: SharedBitVector, label: int = 0) -> DBits:
    """src/rss.py:184-206: forward share_a (with a 4-byte label) to next;
    plain = a ^ b ^ received.  Returns the public vector on the device and
    records a host copy in rt.opened."""
    n = x.logical_len
    rt.send_next(OP_OPEN, Message(u32le(label), x.share_a.words), logical_bits=n)
    msg = rt.recv_prev(OP_OPEN)
    peer_label = int.from_bytes(msg.head[:4], "little")
    if peer_label != label:
        raise ProtocolError(f"open label mismatch: local {label}, peer {peer_label}")
    if msg.tensor is None or msg.tensor.numel() != words_for(n):
        raise ValueError("open message has wrong length")
    out = torch.empty_like(x.share_a.words)
    xor_words(x.share_a.words, x.share_b.words, msg.tensor, out)
    plain = DBits(out, n)
    rt.note_opened(label, plain.to_host())
    return plain
