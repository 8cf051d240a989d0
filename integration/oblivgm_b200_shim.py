"""Reference-side binding of libogm_b200.so.

What a maintainer of the reference package would add as oblivgm/_b200.py: a
ctypes shim that replaces the reference's hot loops while keeping its numpy
data model.  Library path resolution: OGM_B200_LIB or the in-tree build.
"""
import os
from pathlib import Path

import ctypes, numpy as np
import torch  # only for device buffers / streams

_lib = ctypes.CDLL(os.environ.get("OGM_B200_LIB", str(Path(__file__).resolve().parent.parent / "paper_2209_03526_b200" / "libogm_b200.so")))
_lib.ogm_last_error.restype = ctypes.c_char_p
_vp, _i64 = ctypes.c_void_p, ctypes.c_int64


def _check(rc):
    if rc:
        try:
            from .fss import DomainError  # inside the reference package
        except ImportError:
            from paper_2209_03526_b200.errors import DomainError
        msg = _lib.ogm_last_error().decode()
        raise (DomainError if rc == -2 else ValueError if rc == -1 else RuntimeError)(msg)


def _soa(keys):
    """DcfKey/DpfKey list -> level-major SoA expected by the ABI."""
    bits = keys[0].domain_bits
    root = np.frombuffer(b"".join(k.root_seed for k in keys), np.uint8).reshape(-1, 16)
    cw = np.stack([np.ascontiguousarray(k.seed_cw).view(np.uint8).reshape(bits, 16) for k in keys], 1)
    cc = np.stack([k.ctrl_cw for k in keys]).astype(np.uint32)
    sh = np.uint32(1) << np.arange(bits, dtype=np.uint32)
    ctrl = np.stack([(((cc >> j) & 1) * sh).sum(1, dtype=np.uint64) for j in range(3)]).astype(np.uint32)
    flags = np.array([k.root_t | (k.final_cw << 1) | (k.add_const << 2) for k in keys], np.uint8)
    return bits, root, np.ascontiguousarray(cw), ctrl, flags


def eval_points(keys, points):
    """Batched fss._walk_eval (src/fss.py:257-281) from host buffers."""
    bits, root, cw, ctrl, flags = _soa(keys)
    pts = np.ascontiguousarray(points, np.uint32)
    out = np.zeros((len(keys) + 31) // 32, np.uint32)
    kind = 1 if type(keys[0]).__name__ == "DcfKey" else 0
    P = lambda a: a.ctypes.data_as(_vp)
    _check(_lib.ogm_fss_eval_points_host(kind, bits, _i64(len(keys)), P(root), P(cw), P(ctrl), P(flags),
                                         P(pts), P(out)))
    return np.unpackbits(out.view(np.uint8), bitorder="little")[: len(keys)]


def parity_rows_device(da, db, ia, ib):
    """engine._parity_rows(da & ia) ^ _parity_rows(db & ib) (src/engine.py:162) on the GPU."""
    rows, w = da.shape
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint32).view(np.int32)).cuda()
    A, B, IA, IB = t(da), t(db), t(ia), t(ib)
    out = torch.empty((rows + 31) // 32, dtype=torch.int32, device="cuda")
    arr = lambda *xs: (ctypes.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
    i32 = lambda *v: (ctypes.c_int32 * len(v))(*v)
    _check(_lib.ogm_masked_parity(_i64(rows), _i64(w), _i64(w), 2, arr(A, B), 1, i32(0), i32(1), 1,
                                  arr(IA, IB), arr(out), _vp(torch.cuda.current_stream().cuda_stream)))
    return np.unpackbits(out.cpu().numpy().view(np.uint8), bitorder="little")[:rows]
