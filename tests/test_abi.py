"""C-ABI tests that need no GPU: the library loads, exports every symbol
include/mpsp.h declares, and rejects invalid inputs with the documented error
codes (validation runs on the host before any CUDA call)."""
import ctypes
import os
import re

import numpy as np
import pytest

import __graft_entry__  # noqa: F401  (builds nothing; import check)
from paper_1411_2377_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    __graft_entry__.build()
    return _lib.lib()


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mpsp.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mpsp_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(L):
    syms = header_symbols()
    assert len(syms) >= 12
    assert set(syms) == set(_lib.SYMBOLS)
    for s in syms:
        assert hasattr(L, s), s


def test_error_codes_match_header(L):
    txt = open(os.path.join(ROOT, "include", "mpsp.h")).read()
    codes = {m.group(1): int(m.group(2)) for m in re.finditer(r"#define (MPSP_E_\w+)\s+(-?\d+)", txt)}
    assert codes == _lib.ERROR_CODES
    for c in codes.values():
        assert _lib.strerror(c) != "unknown error code"
    assert _lib.strerror(0) == "ok"


def test_supported_precisions(L):
    for p in (32, 64, 128, 256, 512, 1024, 2048, 4096, 8192):
        assert _lib.supported_precision(p)
    for p in (0, 16, 33, 96, 3072, 16384):
        assert not _lib.supported_precision(p)


def create(p, rowptr, colidx, limbs, exps, signs, rb=0, re=None, flags=0):
    n = len(rowptr) - 1
    re = n if re is None else re
    h = ctypes.c_void_p()
    arrs = [np.ascontiguousarray(a) for a in (rowptr, colidx, limbs, exps, signs)]
    rc = _lib.lib().mpsp_csr_create(ctypes.byref(h), p, n, *[a.ctypes.data for a in arrs],
                                    rb, re, flags)
    return rc, h


def good(p=64, n=3):
    L = p // 32
    rowptr = np.array([0, 2, 3, 3], np.int64)
    colidx = np.array([0, 2, 1], np.int32)
    limbs = np.zeros((3, L), np.uint32)
    limbs[:, -1] = 0x80000000
    return [p, rowptr, colidx, limbs, np.zeros(3, np.int32), np.zeros(3, np.uint8)]


def test_create_validation_errors(L):
    E = _lib.ERROR_CODES
    p, rp, ci, li, ex, sg = good()
    # precision
    assert create(96, rp, ci, np.zeros((3, 3), np.uint32), ex, sg)[0] == E["MPSP_E_PREC"]
    assert create(48, rp, ci, li, ex, sg)[0] == E["MPSP_E_PREC"]
    # csr structure
    assert create(p, np.array([1, 2, 3, 3], np.int64), ci, li, ex, sg)[0] == E["MPSP_E_CSR"]
    assert create(p, np.array([0, 2, 1, 3], np.int64), ci, li, ex, sg)[0] == E["MPSP_E_CSR"]
    assert create(p, rp, np.array([0, 3, 1], np.int32), li, ex, sg)[0] == E["MPSP_E_CSR"]
    assert create(p, rp, np.array([0, -1, 1], np.int32), li, ex, sg)[0] == E["MPSP_E_CSR"]
    # unsorted / duplicate
    assert create(p, rp, np.array([2, 0, 1], np.int32), li, ex, sg)[0] == E["MPSP_E_UNSORTED"]
    assert create(p, rp, np.array([1, 1, 1], np.int32), li, ex, sg)[0] == E["MPSP_E_UNSORTED"]
    # values: unnormalised, exponent out of range (zeros may carry junk exps)
    bad = li.copy()
    bad[1, -1] = 0x40000000
    assert create(p, rp, ci, bad, ex, sg)[0] == E["MPSP_E_VALUE"]
    assert create(p, rp, ci, li, np.array([0, 2 ** 29 + 1, 0], np.int32), sg)[0] == E["MPSP_E_VALUE"]
    assert create(p, rp, ci, li, np.array([0, -(2 ** 29) - 1, 0], np.int32), sg)[0] == E["MPSP_E_VALUE"]
    # bad ranges / flags
    assert create(p, rp, ci, li, ex, sg, rb=2, re=1)[0] == E["MPSP_E_ARG"]
    assert create(p, rp, ci, li, ex, sg, rb=0, re=4)[0] == E["MPSP_E_ARG"]
    assert create(p, rp, ci, li, ex, sg, flags=0x10)[0] == E["MPSP_E_ARG"]
    # null out-pointer
    assert _lib.lib().mpsp_csr_create(None, 64, 0, None, None, None, None, None, 0, 0, 0) == E["MPSP_E_ARG"]


def test_null_handle_calls(L):
    E = _lib.ERROR_CODES
    L.mpsp_destroy(None)                     # NULL-safe
    assert L.mpsp_spmv(None, None, None, None, None, None, None, None) == E["MPSP_E_ARG"]
    assert L.mpsp_spmv_t(None, None, None, None, None, None, None, None) == E["MPSP_E_ARG"]
    assert L.mpsp_spmv_host(None, None, None, None, None, None, None) == E["MPSP_E_ARG"]
    info = (ctypes.c_int64 * 10)()
    assert L.mpsp_csr_info(None, info) == E["MPSP_E_ARG"]
    assert L.mpsp_launch_count() >= 0


def test_product_path_has_no_oracle_or_fallback():
    """The product package never imports/executes the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_1411_2377_b200")
    pat = re.compile(r"^\s*(from|import)\s+oracle|oracle[/.]|run_parallel|mpref", re.M)
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dp, f)).read()
                assert not pat.search(txt), f
