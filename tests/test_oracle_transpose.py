"""Pins for the oracle's full-size helpers (CPU only): the numpy transpose,
the sampled-column A^T checker ``spmv_t_cols`` and the multiprocess drivers
of oracle/run_parallel.py - each against the plain serial oracle functions
(``transpose`` sorts (col, row, k) Python tuples; ``spmv``/``spmv_t`` are
themselves pinned by test_oracle_pins.py / test_oracle_invariants.py).

Why it matters: ``spmv_t_cols`` and ``spmv_t_parallel`` are the checkers
behind full-size A^T parity (tests/test_gpu_fullsize.py, bench.py's parity
field) - the second SpMV of each BiCG iteration, z~ = A^T p~
(reading c3: ascending row index of A).
"""
import random

import numpy as np
import pytest

import gen
import oracle
from oracle import mpref, run_parallel


def rand_pattern(R, n, density):
    rowptr, cols = [0], []
    for i in range(n):
        for j in range(n):
            if R.random() < density:
                cols.append(j)
        rowptr.append(len(cols))
    return np.array(rowptr, np.int64), np.array(cols, np.int32)


@pytest.mark.parametrize("n,density", [(0, 0.0), (1, 1.0), (5, 0.0), (9, 0.3), (17, 0.8), (40, 0.1)])
def test_transpose_np_equals_sorted_triples(n, density):
    R = random.Random(n * 1000 + int(density * 100))
    rowptr, cols = rand_pattern(R, n, density)
    want = oracle.transpose(n, rowptr, cols)
    got = oracle.transpose_np(n, rowptr, cols)
    for g, w in zip(got, want):
        assert np.array_equal(np.asarray(g, np.int64), np.asarray(w, np.int64))


def test_transpose_np_is_involution_and_orders_rows():
    d = gen.make("C4", n=3000, seed=5)
    n = d["n"]
    rt, ct, perm = oracle.transpose_np(n, d["rowptr"], d["colidx"])
    # ascending row index of A inside each transposed row (strictly: a pattern
    # holds (i, j) at most once)
    for j in range(n):
        seg = ct[rt[j]:rt[j + 1]]
        assert np.all(np.diff(seg) > 0)
    rtt, ctt, perm2 = oracle.transpose_np(n, rt, ct)
    assert np.array_equal(rtt, d["rowptr"]) and np.array_equal(ctt, d["colidx"])
    assert np.array_equal(perm[perm2], np.arange(len(perm)))


def _args(d):
    return (d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
            d["x_limbs"], d["x_exps"], d["x_signs"])


CASES = [("C1", 300, None), ("C2", 400, 64), ("C3", 300, 512), ("C4", 1500, 256),
         ("C5", 400, 96), ("C1", 200, 2048)]


@pytest.mark.parametrize("cfg,n,p", CASES)
def test_spmv_t_cols_equals_spmv_t(cfg, n, p):
    d = gen.make(cfg, n=n, seed=2, p=p)
    want = oracle.spmv_t(*_args(d))
    rng = np.random.default_rng(7)
    cols = sorted(set(rng.choice(d["n"], size=min(60, d["n"]), replace=False).tolist())
                  | {0, d["n"] - 1})
    got = oracle.pack_vec(oracle.spmv_t_cols(*_args(d), cols), d["p"])
    for g, w in zip(got, want):
        assert np.array_equal(g, w[cols])


def test_spmv_t_cols_on_stress_corpus():
    d = gen.stress(64, seed=4, long_len=300, n_random_rows=40)
    want = oracle.spmv_t(*_args(d))
    cols = list(range(d["n"]))
    got = oracle.pack_vec(oracle.spmv_t_cols(*_args(d), cols), d["p"])
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("cfg,n,p", [("C1", 300, None), ("C4", 1200, 128), ("C5", 400, 64)])
def test_parallel_drivers_equal_serial_oracle(cfg, n, p):
    d = gen.make(cfg, n=n, seed=3, p=p)
    want = oracle.spmv(*_args(d))
    want_t = oracle.spmv_t(*_args(d))
    got, _, used = run_parallel.spmv_parallel(*_args(d), workers=3)
    assert used == 3
    for g, w in zip(got, want):
        assert np.array_equal(g, w)
    got_t, _, _, _ = run_parallel.spmv_t_parallel(*_args(d), workers=2)
    for g, w in zip(got_t, want_t):
        assert np.array_equal(g, w)
    rows = [5, 0, 17, d["n"] - 1]
    vals, _, _ = run_parallel.spmv_rows_parallel(*_args(d), rows, workers=2)
    assert vals == mpref.spmv_rows(*_args(d), rows)
    sub, _, _ = run_parallel.spmv_parallel(*_args(d), rows=rows, workers=2)
    for g, w in zip(sub, want):
        assert np.array_equal(g, w[rows])
