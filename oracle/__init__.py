"""CPU oracle for multiple-precision CSR SpMV (test infrastructure only).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  See oracle/mpref.py for the citations.
"""
from .mpref import (ZERO, rn, mul, add, unpack, unpack_vec, pack_vec, row_chain,
                    spmv, spmv_rows, spmv_t, spmv_t_cols, transpose, transpose_np, dense_mv)

__all__ = ["ZERO", "rn", "mul", "add", "unpack", "unpack_vec", "pack_vec",
           "row_chain", "spmv", "spmv_rows", "spmv_t", "spmv_t_cols", "transpose",
           "transpose_np", "dense_mv"]
from . import krylov  # noqa: E402  (BiCG oracle)
