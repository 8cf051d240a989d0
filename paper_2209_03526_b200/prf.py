"""Deterministic randomness on the B200 (src/prf.py).

* :func:`prg_expand` -- fixed-key AES MMO node expansion (src/prf.py:41-57)
* :func:`prf_words` / :func:`prf_stream` -- AES-128-CTR keyed streams,
  random access by block (src/prf.py:70-92)
* :func:`seeded_permutation` -- bit-exact Fisher-Yates (src/prf.py:95-105)
  computed on the device by deterministic reservations
* :func:`derive_key` -- SHA-256 key derivation (src/prf.py:108-110; host)
"""

from __future__ import annotations

import hashlib

import threading

import numpy as np
import torch

from . import _lib
from .bits import words_for

SEED_BYTES = 16


def _dev(device=None):
    return torch.device(device) if device is not None else torch.device("cuda")


def prg_expand(seeds):
    """Same signature/returns as src/prf.py:41-57 (numpy in, numpy out), or
    a (N,16) uint8 CUDA tensor in -> tensors out."""
    host = not isinstance(seeds, torch.Tensor)
    if host:
        arr = np.ascontiguousarray(seeds, dtype=np.uint64).reshape(-1, 2)
        s = torch.from_numpy(arr.view(np.uint8).reshape(-1, 16).copy()).cuda()
    else:
        s = seeds.contiguous()
    n = s.shape[0]
    left = torch.empty_like(s)
    right = torch.empty_like(s)
    tl = torch.empty((n,), dtype=torch.uint8, device=s.device)
    tr = torch.empty_like(tl)
    v = torch.empty_like(tl)
    _lib.call("ogm_prg_expand", _lib.ptr(s), n, _lib.ptr(left), _lib.ptr(right), _lib.ptr(tl),
              _lib.ptr(tr), _lib.ptr(v), _lib.stream_ptr())
    if not host:
        return left, right, tl, tr, v
    to64 = lambda t: t.cpu().numpy().view(np.uint64).reshape(n, 2)  # noqa: E731
    return to64(left), to64(right), tl.cpu().numpy(), tr.cpu().numpy(), v.cpu().numpy()


def prf_words_device(key: bytes, label: bytes, index: int, nwords: int, first_word: int = 0,
                     out: torch.Tensor | None = None, device=None) -> torch.Tensor:
    """AES-CTR keystream words [first_word, first_word + nwords) on the device."""
    if len(key) != SEED_BYTES:
        raise ValueError("PRF key must be 16 bytes")
    if len(label) != 4:
        raise ValueError("label must be 4 bytes")
    if out is None:
        out = torch.empty((nwords,), dtype=torch.int32, device=_dev(device))
    _lib.call("ogm_prf_words", key, label, index, first_word, nwords, _lib.ptr(out), _lib.stream_ptr())
    return out


def prf_stream(key: bytes, label: bytes, index: int, nbytes: int) -> bytes:
    """src/prf.py:70-84 (bytes out)."""
    if len(key) != SEED_BYTES:
        raise ValueError("PRF key must be 16 bytes")
    if len(label) != 4:
        raise ValueError("label must be 4 bytes")
    if nbytes == 0:
        return b""
    w = prf_words_device(key, label, index, (nbytes + 3) // 4)
    return w.cpu().numpy().tobytes()[:nbytes]


def prf_words(key: bytes, label: bytes, index: int, nbits: int) -> np.ndarray:
    """src/prf.py:87-92 (host words with a clean tail)."""
    nw = words_for(nbits)
    w = prf_words_device(key, label, index, nw).cpu().numpy().view(np.uint32).copy()
    rem = nbits % 32
    if rem and w.size:
        w[-1] &= np.uint32((1 << rem) - 1)
    return w


def zero_share_device(key_own: bytes, key_prev: bytes, counter: int, nbits: int,
                      xor_into: torch.Tensor | None = None, out: torch.Tensor | None = None,
                      device=None) -> torch.Tensor:
    """src/rss.py:143-148 at an explicit counter; optionally XORed into a buffer."""
    if out is None:
        out = torch.empty((words_for(nbits),), dtype=torch.int32,
                          device=xor_into.device if xor_into is not None else _dev(device))
    _lib.call("ogm_zero_share", key_own, key_prev, counter, nbits, _lib.ptr(xor_into), _lib.ptr(out),
              _lib.stream_ptr())
    return out


_TLS = threading.local()


def _thread_workspace(nbytes: int, dev) -> torch.Tensor:
    """Scratch for the permutation rounds, kept per host thread (each party
    thread launches on its own stream, so reuse is stream-ordered) and grown
    on demand: one allocation instead of one per permutation.  Only
    scratch up to WORKSPACE_CACHE_MAX is kept (large permutations, e.g. 4 GB
    at 2^28 rows, allocate per call and free with the caching allocator);
    the key is the stream of ``dev`` itself, not the current device's."""
    dev = torch.device(dev)
    if nbytes > WORKSPACE_CACHE_MAX:
        return torch.empty((nbytes,), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream if dev.type == "cuda" else 0
    key = (str(dev), stream)   # reuse is ordered only on the same stream
    cache = getattr(_TLS, "ws", None)
    if cache is None:
        cache = _TLS.ws = {}
    buf = cache.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = cache[key] = torch.empty((max(nbytes, 1 << 16),), dtype=torch.uint8, device=dev)
    return buf


WORKSPACE_CACHE_MAX = 256 << 20


def release_workspaces() -> None:
    """Drop this thread's cached permutation scratch."""
    _TLS.ws = {}


def seeded_permutation_device(key: bytes, label: bytes, index: int, n: int,
                              out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                              device=None) -> torch.Tensor:
    """src/prf.py:95-105 on the device; int32 gather permutation."""
    dev = _dev(device)
    if out is None:
        out = torch.empty((n,), dtype=torch.int32, device=dev)
    nbytes = int(_lib.load().ogm_perm_workspace_bytes(n))
    if workspace is None or workspace.numel() < nbytes:
        workspace = _thread_workspace(nbytes, dev)
    _lib.call("ogm_seeded_permutation", key, label, index, n, _lib.ptr(out), _lib.ptr(workspace),
              _lib.stream_ptr())
    return out


def seeded_permutation(key: bytes, label: bytes, index: int, n: int) -> np.ndarray:
    """src/prf.py:95-105 (int64 numpy result, like the reference)."""
    if n == 0:
        return np.zeros(0, np.int64)
    return seeded_permutation_device(key, label, index, n).cpu().numpy().astype(np.int64)


def derive_key(master: bytes, label: str) -> bytes:
    """src/prf.py:108-110 (host-side session setup, not on the data path)."""
    return hashlib.sha256(master + b"/" + label.encode()).digest()[:SEED_BYTES]
