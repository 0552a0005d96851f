"""Row-chunked multiprocessing driver for the oracle (test/bench infrastructure).

Runs ``oracle.mpref.spmv_rows`` unchanged over nnz-balanced row chunks on the
host's cores.  Only tests/ and bench.py's cpu_baseline /
reference legs use it.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import mpref

_G = {}


def _init(args):
    _G['args'] = args


def _work(rows):
    p, rowptr, colidx, limbs, exps, signs, xl, xe, xs = _G['args']
    return rows[0], mpref.spmv_rows(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs, rows)


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


def spmv_rows_parallel(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs, rows, workers=None):
    """Same result as mpref.spmv_rows(..., rows), computed on `workers` processes.

    Returns (list of triples in `rows` order, wall seconds, workers used).
    """
    import multiprocessing as mp
    workers = workers or n_cores()
    rowptr = np.asarray(rowptr, dtype=np.int64)
    chunks = _chunks(rowptr, rows, workers * 4)
    args = (p, rowptr, colidx, limbs, exps, signs, xl, xe, xs)
    t0 = time.perf_counter()
    if workers == 1 or len(chunks) <= 1:
        res = [mpref.spmv_rows(*args, rows)] if len(rows) else [[]]
        out = res[0]
    else:
        ctx = mp.get_context('fork')
        _G['args'] = args  # inherited by fork
        with ctx.Pool(workers) as pool:
            parts = pool.map(_work, chunks)
        pos = {first: vals for first, vals in parts}
        out = []
        for c in chunks:
            out.extend(pos[c[0]])
    return out, time.perf_counter() - t0, workers
