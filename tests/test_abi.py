"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/oblivgm_b200.h declares, and rejects bad arguments with the
reference's error classes before touching the device."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2209_03526_b200 import _lib
from paper_2209_03526_b200.build import build
from paper_2209_03526_b200.errors import DomainError

HEADER = Path(__file__).resolve().parent.parent / "include" / "oblivgm_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ogm_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    build()
    return _lib.load(require_device=False)


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s


def test_binding_table_covers_header(lib):
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_abi_version(lib):
    assert lib.ogm_abi_version() == 3


def test_argument_errors_map_to_reference_exceptions(lib):
    # rejected before any device work, so this runs on a CPU-only host
    rc = lib.ogm_fss_gen(1, 0, 4, None, None, None, None, None, None, None)
    assert rc == _lib.OGM_ERR_DOMAIN
    assert b"domain_bits" in lib.ogm_last_error()
    with pytest.raises(DomainError):
        _lib.check(rc)
    rc = lib.ogm_fss_eval_points(7, 8, 4, None, None, None, None, None, None, None)
    assert rc == _lib.OGM_ERR_ARG
    with pytest.raises(ValueError, match="kind"):
        _lib.check(rc)
    rc = lib.ogm_fss_full_domain(0, 3, 1, None, None, None, None, 9, None, 1, None)
    assert rc == _lib.OGM_ERR_DOMAIN  # 9 points from a 2^3 domain (src/fss.py:304-305)


def test_zero_sized_calls_are_noops(lib):
    assert lib.ogm_prg_expand(None, 0, None, None, None, None, None, None) == 0
    assert lib.ogm_fss_eval_points(1, 32, 0, None, None, None, None, None, None, None) == 0


def test_product_refuses_without_device(monkeypatch):
    import torch
    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    monkeypatch.setattr(_lib, "_device_ok", False)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()
