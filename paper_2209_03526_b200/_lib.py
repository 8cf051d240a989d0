"""ctypes binding of libogm_b200.so (the C ABI in include/oblivgm_b200.h).

The product path has no CPU fallback: if the shared library is missing, or no
CUDA device is visible, every call raises.  Return codes map to the
reference's exception types (src/fss.py:44-45 DomainError, src/net.py:38-39
ProtocolError, ValueError for shape/length errors).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import torch

from .errors import DomainError, ProtocolError

LIB_PATH = Path(__file__).resolve().parent / "libogm_b200.so"

OGM_ERR_ARG = -1
OGM_ERR_DOMAIN = -2
OGM_ERR_CUDA = -3
OGM_ERR_PROTOCOL = -4
OGM_ERR_NOMEM = -5

KIND_DPF = 0
KIND_DCF = 1

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_int = ctypes.c_int
_cp = ctypes.c_char_p

# name -> argtypes (every symbol declared in include/oblivgm_b200.h)
SIGNATURES = {
    "ogm_last_error": ([], ctypes.c_char_p),
    "ogm_abi_version": ([], _int),
    "ogm_init": ([], _int),
    "ogm_prg_expand": ([_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_prf_rows": ([_cp, _cp, _u64, _i64, _i64, _i64, _vp, _vp], _int),
    "ogm_prf_words": ([_cp, _cp, _u64, _u64, _i64, _vp, _vp], _int),
    "ogm_zero_share": ([_cp, _cp, _u64, _i64, _vp, _vp, _vp], _int),
    "ogm_zero_share_slice": ([_cp, _cp, _u64, _i64, _u64, _i64, _vp, _vp, _vp], _int),
    "ogm_perm_workspace_bytes": ([_i64], _i64),
    "ogm_seeded_permutation": ([_cp, _cp, _u64, _i64, _vp, _vp, _vp], _int),
    "ogm_fss_gen": ([_int, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_fss_gen_pair": ([_int, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_fss_eval_points": ([_int, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_fss_eval_points_host": ([_int, _int, _i64, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_fss_full_domain": ([_int, _int, _int, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp], _int),
    "ogm_zero_share_trio": ([_cp, _cp, _cp, _u64, _i64, _vp, _vp, _vp], _int),
    "ogm_zero_share_trio_rows": ([_cp, _cp, _cp, _u64, _i64, _i64, _i64, _vp, _vp, _vp], _int),
    "ogm_zero_share_trio_slice2": ([_cp, _cp, _cp, _u64, _u64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_zero_share_trio_fold2": ([_cp, _cp, _cp, _u64, _u64, _i64, _i64, _i64, _vp, _vp, _vp], _int),
    "ogm_zero_share_trio_slice": ([_cp, _cp, _cp, _u64, _i64, _i64, _i64, _vp, _vp, _vp], _int),
    "ogm_and_terms": ([_i64, _int, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_xor_words": ([_i64, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_masked_parity": ([_i64, _i64, _i64, _int, _vp, _int, _vp, _vp, _int, _vp, _vp, _vp], _int),
    "ogm_masked_parity_acc": ([_i64, _i64, _i64, _int, _vp, _int, _vp, _vp, _int, _vp, _vp, _vp], _int),
    "ogm_select_fold": ([_i64, _i64, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_select_many": ([_i64, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp, _i64, _vp, _vp], _int),
    "ogm_pack_fields": ([_i64, _vp, _int, _vp, _vp, _vp, _vp, _i64, _vp], _int),
    "ogm_pack_gather": ([_i64, _vp, _int, _vp, _int, _vp, _vp, _vp, _vp, _vp, _i64, _vp], _int),
    "ogm_extract_field": ([_vp, _i64, _vp, _i64, _i64, _i64, _vp, _i64, _vp], _int),
    "ogm_mask_row_tails": ([_vp, _i64, _i64, _i64, _vp], _int),
    "ogm_unpack_records": ([_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp], _int),
    "ogm_column_bits": ([_vp, _i64, _i64, _vp, _vp], _int),
    "ogm_compact_workspace_bytes": ([_i64], _i64),
    "ogm_compact_bits": ([_i64, _vp, _vp, _vp, _vp, _i64, _vp], _int),
    "ogm_keep_rows_workspace_bytes": ([_i64], _i64),
    "ogm_pcg64_u32": ([_vp, _vp, _int, ctypes.c_uint32, _i64, _vp, _vp], _int),
    "ogm_deal_rows": ([_vp, _vp, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp], _int),
    "ogm_deal_hot_bits": ([_vp, _vp, _i64, _vp, _vp], _int),
    "ogm_keep_rows": ([_i64, _vp, _int, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _i64, _vp], _int),
    "ogm_split_flag_rows": ([_i64, _vp, _i64, _vp, _vp, _vp], _int),
    "ogm_flag_shuffle_trio": ([_i64] + [_vp] * 19, _int),
    "ogm_fetch128_online_planned": ([_i64] + [_vp] * 14 + [_int, _vp, _int] + [_vp] * 16, _int),
    "ogm_flag_open_composed": ([_i64] + [_vp] * 14, _int),
    "ogm_fetch128_online_fused": ([_i64] + [_vp] * 27, _int),
    "ogm_shuffle_online_planned_slots": ([_i64] + [_vp] * 14 + [_int, _vp, _int] + [_vp] * 3, _int),
    "ogm_shuffle_gather": ([_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _cp, _cp, _u64, _vp, _cp, _cp, _u64,
                            _vp, _cp, _cp, _u64, _vp, _i64, _i64, _vp, _vp], _int),
    "ogm_perm_compose": ([_i64, _vp, _vp, _vp, _vp], _int),
    "ogm_perm_invert": ([_i64, _vp, _vp, _vp], _int),
    "ogm_gather_window_rows": ([_i64], _i64),
    "ogm_gather_tile_rows": ([_i64], _i64),
    "ogm_gather_plan_workspace_bytes": ([_i64, _i64, _i64], _i64),
    "ogm_gather_plan": ([_i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp], _int),
    "ogm_gather_plan_runs": ([_i64, _i64, _i64, _vp, _vp, _vp, _vp], _int),
    "ogm_gather_planned": ([_i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _int, _vp], _int),
    "ogm_trio_shuffle_workspace_bytes": ([_i64, _i64], _i64),
    "ogm_trio_shuffle": ([_cp, _cp, _cp, _u64, _i64, _i64, _i64, _int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp], _int),
    "ogm_trio_open_keep_workspace_bytes": ([_i64], _i64),
    "ogm_trio_open_keep": ([_vp, _i64, _i64, _vp, _int, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp], _int),
    "ogm_shuffle_online_fused": ([_i64] + [_vp] * 15 + [_vp], _int),
    "ogm_shuffle_online_planned": ([_i64] + [_vp] * 16, _int),
    "ogm_shuffle_online_planned_ex": ([_i64] + [_vp] * 8 + [_int, _vp, _int, _vp, _int] + [_vp] * 6, _int),
    "ogm_shuffle_online_planned_w_output_order": ([_i64], _int),
    "ogm_trio_match": ([_vp, _vp, _vp, _i64, _vp], _int),
    "ogm_measure_int_peak": ([ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)], _int),
}

# Entry points that may block on the device (host syncs); every other entry
# point only enqueues work on the caller's stream and returns in microseconds.
BLOCKING = {"ogm_init", "ogm_seeded_permutation", "ogm_fss_eval_points_host", "ogm_measure_int_peak",
            "ogm_trio_open_keep", "ogm_trio_shuffle", "ogm_trio_match"}

_lib = None
_fast = None
_device_ok = False


def load(require_device: bool = True):
    """Load the library (and, by default, insist on a CUDA device)."""
    global _lib, _fast, _device_ok
    if _lib is not None and (_device_ok or not require_device):
        return _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2209_03526_b200.build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(str(LIB_PATH))
        # the same library through PyDLL: calls keep the GIL.  For the
        # non-blocking launchers that beats releasing it -- with three party
        # threads, every released GIL has to be won back (measured on the
        # per-party C1 path)
        fast = ctypes.PyDLL(str(LIB_PATH))
        for name, (args, res) in SIGNATURES.items():
            for h in (lib, fast):
                fn = getattr(h, name)
                fn.argtypes = args
                fn.restype = res
        _lib, _fast = lib, fast
    if require_device:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2209_03526_b200 needs a CUDA device (no CPU fallback)")
        _device_ok = True
    return _lib


def check(rc: int) -> None:
    if rc == 0:
        return
    msg = (_lib.ogm_last_error() or b"").decode(errors="replace")
    if rc == OGM_ERR_DOMAIN:
        raise DomainError(msg)
    if rc == OGM_ERR_PROTOCOL:
        raise ProtocolError(msg)
    if rc == OGM_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"libogm_b200 error {rc}: {msg}")


_fns: dict = {}


def call(name: str, *args) -> None:
    fn = _fns.get(name)
    if fn is None:
        load()
        fn = _fns[name] = getattr(_lib if name in BLOCKING else _fast, name)
    rc = fn(*args)
    if rc:
        check(rc)


def ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def ptr_array(tensors) -> ctypes.Array:
    """Host array of device pointers (NULL for None) for the const T* const* args."""
    arr = (ctypes.c_void_p * max(1, len(tensors)))()
    for i, t in enumerate(tensors):
        arr[i] = None if t is None else t.data_ptr()
    return arr


def int_array(vals) -> ctypes.Array:
    arr = (ctypes.c_int32 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr


def i64_array(vals) -> ctypes.Array:
    arr = (ctypes.c_int64 * max(1, len(vals)))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr


def stream_ptr(stream: torch.cuda.Stream | None = None):
    """cudaStream_t of `stream` or of the calling thread's current stream
    (raw accessor: torch.cuda.current_stream() costs ~10 us per call)."""
    if stream is not None:
        return stream.cuda_stream
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())
