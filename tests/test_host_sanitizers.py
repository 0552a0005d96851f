"""The host half of mpsp_csr_create (validation, transpose, row binning, row
chunks, chunk-major repack: SURVEY.md 8(a) rows a1-a3) built with
AddressSanitizer and UndefinedBehaviorSanitizer and driven by a random-CSR
fuzz driver (tests/native/host_builder_fuzz.cpp, through
mpsp_debug_host_build - no GPU needed): every valid input accepted and built
deterministically, every invalid one rejected with its documented code, and
no sanitizer report (the CSR invariants of SPEC S:122-126).
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_host_builder_under_asan_ubsan(tmp_path):
    env = dict(os.environ, ASAN_OUT=str(tmp_path))
    r = subprocess.run(["bash", os.path.join(ROOT, "tools", "asan_host.sh"), "150", "11"],
                       capture_output=True, text=True, timeout=900, env=env)
    out = r.stdout + r.stderr
    assert "AddressSanitizer" not in out and "runtime error" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    assert "host builder fuzz ok" in out


def test_debug_host_build_matches_device_sizes():
    """mpsp_debug_host_build reports the same part sizes the handle info
    does (CPU: compared with the builder's own invariants)."""
    import ctypes
    import numpy as np
    import gen
    from paper_1411_2377_b200 import _lib
    import __graft_entry__
    __graft_entry__.build()
    d = gen.make("C4", n=4000, seed=1)
    arrs = [np.ascontiguousarray(a) for a in (d["rowptr"], d["colidx"], d["limbs"], d["exps"],
                                              d["signs"])]
    out = (ctypes.c_int64 * 12)()
    rc = _lib.lib().mpsp_debug_host_build(d["p"], d["n"], *[a.ctypes.data for a in arrs], 0, d["n"],
                                          _lib.MPSP_WITH_TRANSPOSE, out)
    assert rc == 0
    assert out[0] == d["meta"]["nnz"] and out[6] == d["meta"]["nnz"]
    assert out[1] >= out[0] and out[7] >= out[6]
    assert out[2] == int((np.diff(d["rowptr"]) > 32).sum())     # rows over 32 take a warp (< 32768 rows)
