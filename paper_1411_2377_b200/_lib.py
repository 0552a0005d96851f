"""ctypes binding of libmpsp.so (include/mpsp.h).  Argument marshalling only.

Fails loudly when the library is missing: there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
# MPSP_LIB selects an in-tree tuning variant (tools/variants.sh); default libmpsp.so
LIB_PATH = os.path.join(_PKG, os.environ.get("MPSP_LIB", "libmpsp.so"))

MPSP_OK = 0
MPSP_WITH_TRANSPOSE = 0x1
ERRORS = {
    -1: "MPSP_E_ARG", -2: "MPSP_E_PREC", -3: "MPSP_E_CSR", -4: "MPSP_E_UNSORTED",
    -5: "MPSP_E_VALUE", -6: "MPSP_E_NOMEM", -7: "MPSP_E_CUDA", -8: "MPSP_E_ALIAS",
    -9: "MPSP_E_DEVICE", -10: "MPSP_E_NOTRANS",
}
ERROR_CODES = {v: k for k, v in ERRORS.items()}

# every symbol include/mpsp.h declares
SYMBOLS = ("mpsp_csr_create", "mpsp_dense_create", "mpsp_spmv", "mpsp_spmv_t", "mpsp_spmv_host", "mpsp_spmv_t_host",
           "mpsp_destroy", "mpsp_strerror", "mpsp_last_cuda_error", "mpsp_csr_info",
           "mpsp_launch_count", "mpsp_imad_bench", "mpsp_supported_precision",
           "mpsp_dot", "mpsp_axpy", "mpsp_bicg", "mpsp_gpbicg", "mpsp_debug_dot_stats",
           "mpsp_vec_pack", "mpsp_vec_unpack", "mpsp_debug_host_build")
BICG_STATUS = {0: "converged", 1: "breakdown", 2: "max_iter"}


class MpspError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        self.name = ERRORS.get(code, str(code))
        msg = f"{self.name} ({code}): {strerror(code)}"
        if code == -7:
            msg += f" [{last_cuda_error()}]"
        if what:
            msg = f"{what}: {msg}"
        super().__init__(msg)


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmpsp.so not built at {LIB_PATH}; run __graft_entry__.build() "
                          "(python -m paper_1411_2377_b200._build)")
    L = ctypes.CDLL(LIB_PATH)
    P, I, I64, U32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint32
    L.mpsp_csr_create.argtypes = [ctypes.POINTER(P), I, I64, P, P, P, P, P, I64, I64, U32]
    L.mpsp_csr_create.restype = I
    L.mpsp_dense_create.argtypes = [ctypes.POINTER(P), I, I64, P, P, P, I64, I64, U32]
    L.mpsp_dense_create.restype = I
    for name in ("mpsp_spmv", "mpsp_spmv_t"):
        f = getattr(L, name)
        f.argtypes = [P, P, P, P, P, P, P, P]
        f.restype = I
    for name in ("mpsp_spmv_host", "mpsp_spmv_t_host"):
        f = getattr(L, name)
        f.argtypes = [P, P, P, P, P, P, P]
        f.restype = I
    L.mpsp_destroy.argtypes = [P]
    L.mpsp_destroy.restype = None
    L.mpsp_strerror.argtypes = [I]
    L.mpsp_strerror.restype = ctypes.c_char_p
    L.mpsp_last_cuda_error.argtypes = []
    L.mpsp_last_cuda_error.restype = ctypes.c_char_p
    L.mpsp_csr_info.argtypes = [P, ctypes.POINTER(I64)]
    L.mpsp_csr_info.restype = I
    L.mpsp_launch_count.argtypes = []
    L.mpsp_launch_count.restype = I64
    L.mpsp_imad_bench.argtypes = [ctypes.POINTER(ctypes.c_double)]
    L.mpsp_imad_bench.restype = I
    L.mpsp_supported_precision.argtypes = [I]
    L.mpsp_supported_precision.restype = I
    L.mpsp_dot.argtypes = [I, I64] + [P] * 9 + [P]
    L.mpsp_dot.restype = I
    L.mpsp_axpy.argtypes = [I, I64, P, P, P, I] + [P] * 9 + [P]
    L.mpsp_axpy.restype = I
    L.mpsp_bicg.argtypes = [P, P, P, P, P, P, P, I, ctypes.POINTER(I), ctypes.POINTER(I), P]
    L.mpsp_bicg.restype = I
    L.mpsp_gpbicg.argtypes = L.mpsp_bicg.argtypes
    L.mpsp_gpbicg.restype = I
    L.mpsp_debug_dot_stats.argtypes = [P]
    L.mpsp_debug_dot_stats.restype = I
    L.mpsp_vec_pack.argtypes = [I, I64, P, P, P, P, P]
    L.mpsp_vec_pack.restype = I
    L.mpsp_vec_unpack.argtypes = [I, I64, P, P, P, P, P]
    L.mpsp_vec_unpack.restype = I
    L.mpsp_debug_host_build.argtypes = [I, I64, P, P, P, P, P, I64, I64, U32, ctypes.POINTER(I64)]
    L.mpsp_debug_host_build.restype = I
    _lib = L
    return L


def strerror(code: int) -> str:
    return lib().mpsp_strerror(code).decode()


def last_cuda_error() -> str:
    return lib().mpsp_last_cuda_error().decode()


def check(rc: int, what: str = "") -> None:
    if rc != MPSP_OK:
        raise MpspError(rc, what)


def launch_count() -> int:
    return int(lib().mpsp_launch_count())


def imad_bench() -> dict:
    out = (ctypes.c_double * 5)()
    check(lib().mpsp_imad_bench(out), "mpsp_imad_bench")
    return {"limb_macs_per_s": out[0], "seconds": out[1], "sms": int(out[2]),
            "comba_limb_macs_per_s": out[3], "operand_scan_limb_macs_per_s": out[4]}


def supported_precision(p: int) -> bool:
    return bool(lib().mpsp_supported_precision(int(p)))


def dot_stats() -> dict:
    """Segments of the segmented dot evaluated step by step / committed from
    their speculative sums since the last call (then reset)."""
    out = (ctypes.c_ulonglong * 2)()
    check(lib().mpsp_debug_dot_stats(out), "mpsp_debug_dot_stats")
    return {"sequential": int(out[0]), "validated": int(out[1])}
