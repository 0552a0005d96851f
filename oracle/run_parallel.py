"""Row-chunked multiprocessing driver for the oracle (test/bench infrastructure).

Runs ``oracle.mpref.spmv_rows`` unchanged over nnz-balanced row chunks on the
host's cores.  Only tests/ and bench.py's cpu_baseline /
reference legs use it.  ``spmv_t_parallel`` applies the same chains to the
transpose built by ``mpref.transpose_np`` (step 5 of SURVEY 8(c): A^T x is
the row chain over the transposed CSR, ascending row index of A).  Pinned
against the serial oracle in tests/test_oracle_invariants.py.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import mpref

_G = {}


def _work(rows):
    p, rowptr, colidx, limbs, exps, signs, xl, xe, xs = _G['args']
    return rows[0], mpref.spmv_rows(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs, rows)


def _work_packed(rows):
    p, rowptr, colidx, limbs, exps, signs, xl, xe, xs = _G['args']
    vals = mpref.spmv_rows(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs, rows)
    return rows[0], mpref.pack_vec(vals, p)


def n_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _chunks(rowptr, rows, nchunks):
    rows = np.asarray(rows, dtype=np.int64)
    if len(rows) == 0:
        return []
    cost = (rowptr[rows + 1] - rowptr[rows]).astype(np.float64) + 1.0
    cum = np.cumsum(cost)
    bounds = np.searchsorted(cum, np.linspace(0, cum[-1], nchunks + 1)[1:-1])
    parts = np.split(rows, bounds)
    return [list(map(int, c)) for c in parts if len(c)]


def _run(args, rows, workers, fn):
    import multiprocessing as mp
    rowptr = args[1]
    chunks = _chunks(rowptr, rows, workers * 4)
    if workers == 1 or len(chunks) <= 1:
        _G['args'] = args
        return [fn(c) for c in chunks]
    ctx = mp.get_context('fork')
    _G['args'] = args  # inherited by fork
    with ctx.Pool(workers) as pool:
        return pool.map(fn, chunks)


def spmv_rows_parallel(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs, rows, workers=None):
    """Same result as mpref.spmv_rows(..., rows), computed on `workers` processes.

    Returns (list of triples in `rows` order, wall seconds, workers used).
    """
    workers = workers or n_cores()
    rowptr = np.asarray(rowptr, dtype=np.int64)
    args = (p, rowptr, colidx, limbs, exps, signs, xl, xe, xs)
    t0 = time.perf_counter()
    parts = _run(args, rows, workers, _work)
    out = []
    for _, vals in parts:          # chunks are consecutive slices of `rows`, in order
        out.extend(vals)
    return out, time.perf_counter() - t0, workers


def spmv_parallel(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs, rows=None, workers=None):
    """Packed y = A x (all rows, or the listed rows in order) on `workers` processes.

    Returns ((limbs [r, L], exps, signs), wall seconds, workers used).
    """
    workers = workers or n_cores()
    rowptr = np.asarray(rowptr, dtype=np.int64)
    n = len(rowptr) - 1
    rows = np.arange(n, dtype=np.int64) if rows is None else np.asarray(rows, dtype=np.int64)
    args = (p, rowptr, colidx, limbs, exps, signs, xl, xe, xs)
    t0 = time.perf_counter()
    parts = _run(args, rows, workers, _work_packed)
    L = p // 32
    if parts:
        out = tuple(np.concatenate([pk[i] for _, pk in parts]) for i in range(3))
    else:
        out = (np.zeros((0, L), np.uint32), np.zeros(0, np.int32), np.zeros(0, np.uint8))
    return out, time.perf_counter() - t0, workers


def transposed(p, rowptr, colidx, limbs, exps, signs):
    """(rowptr_t, colidx_t, limbs_t, exps_t, signs_t) of A^T (mpref.transpose_np)."""
    L = p // 32
    n = len(rowptr) - 1
    rowptr_t, colidx_t, perm = mpref.transpose_np(n, rowptr, colidx)
    limbs = np.asarray(limbs, dtype=np.uint32).reshape(-1, L)
    return rowptr_t, colidx_t, limbs[perm], np.asarray(exps)[perm], np.asarray(signs)[perm]


def spmv_t_parallel(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs, cols=None, workers=None,
                    T=None):
    """Packed y = A^T x (all columns, or the listed ones) on `workers` processes.

    T: a precomputed ``transposed(...)`` tuple.  Returns (packed y, wall seconds
    of the chains, workers used, wall seconds of the transpose).
    """
    t0 = time.perf_counter()
    if T is None:
        T = transposed(p, rowptr, colidx, limbs, exps, signs)
    t_tr = time.perf_counter() - t0
    out, wall, used = spmv_parallel(p, *T, xl, xe, xs, rows=cols, workers=workers)
    return out, wall, used, t_tr
