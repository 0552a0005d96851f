"""mpsp - multiple-precision CSR SpMV on NVIDIA B200 (arXiv 1411.2377 hot path).

y = A x and y = A^T x for p-bit binary floating-point CSR matrices with
round-to-nearest-even after every multiply and add, rows summed in ascending
column order (A^T: ascending row index of A), computed bit-exactly by
hand-written sm_100a kernels behind a C ABI (include/mpsp.h).
"""
from ._lib import MpspError, imad_bench, launch_count, supported_precision, LIB_PATH
from .csr import CSR, MPVec

__all__ = ["CSR", "MPVec", "MpspError", "imad_bench", "launch_count", "supported_precision",
           "LIB_PATH"]
