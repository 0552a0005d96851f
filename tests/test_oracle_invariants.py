"""Invariant pins for oracle.spmv / oracle.spmv_t (SURVEY.md 8(c) list 1-9).

CPU only.  Each invariant is a property of the defined operation that holds
bitwise, checked on small random CSR matrices (n <= 24) at several p:
  1 identity . x = x      2 permutation permutes x     3 (A^T)^T = A
  4 spmv_t(A) = spmv(explicit A^T built densely)      5 small integers exact
  6 2^k scaling           7 negation                   8 densification / zeros
  9 determinism.
"""
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import mpref
import pinlib

PS = [32, 64, 128, 256]


def rand_csr(R, n, p, density=0.35, small_int=False, espread=6):
    top = 1 << (p - 1)
    rowptr, cols, vals = [0], [], []
    for i in range(n):
        for j in range(n):
            if R.random() < density:
                cols.append(j)
                if small_int:
                    v = R.randint(-(2 ** 7), 2 ** 7)
                    vals.append(int_to_triple(v, p))
                elif R.random() < 0.08:
                    vals.append((0, 0, 0))
                else:
                    vals.append((R.getrandbits(1), top | R.getrandbits(p - 1), R.randint(-espread, espread)))
        rowptr.append(len(cols))
    return np.array(rowptr, np.int64), np.array(cols, np.int32), vals


def int_to_triple(v, p):
    if v == 0:
        return (0, 0, 0)
    s = 1 if v < 0 else 0
    a = abs(v)
    b = a.bit_length()
    assert b <= p
    return (s, a << (p - b), b)


def rand_x(R, n, p, small_int=False, espread=6):
    top = 1 << (p - 1)
    if small_int:
        return [int_to_triple(R.randint(-(2 ** 7), 2 ** 7), p) for _ in range(n)]
    return [(R.getrandbits(1), top | R.getrandbits(p - 1), R.randint(-espread, espread))
            if R.random() > 0.1 else (0, 0, 0) for _ in range(n)]


def run(p, rowptr, cols, vals, x, t=False):
    al, ae, as_ = mpref.pack_vec(vals, p)
    xl, xe, xs = mpref.pack_vec(x, p)
    f = mpref.spmv_t if t else mpref.spmv
    return mpref.unpack_vec(*f(p, rowptr, cols, al, ae, as_, xl, xe, xs), p)


def dense_of(n, rowptr, cols, vals):
    D = [[None] * n for _ in range(n)]
    for i in range(n):
        for k in range(rowptr[i], rowptr[i + 1]):
            D[i][cols[k]] = vals[k]
    return D


def csr_of_dense(D, keep_none=False):
    n = len(D)
    rowptr, cols, vals = [0], [], []
    for i in range(n):
        for j in range(n):
            if D[i][j] is not None:
                cols.append(j)
                vals.append(D[i][j])
        rowptr.append(len(cols))
    return np.array(rowptr, np.int64), np.array(cols, np.int32), vals


@pytest.mark.parametrize("p", PS)
def test_identity_and_permutation(p):
    R = random.Random(p)
    n = 17
    x = rand_x(R, n, p)
    one = (0, 1 << (p - 1), 1)
    ident = (np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), [one] * n)
    assert run(p, *ident, x) == [v if v[1] else (0, 0, 0) for v in x]
    perm = list(range(n))
    R.shuffle(perm)
    P = (np.arange(n + 1, dtype=np.int64), np.array(perm, np.int32), [one] * n)
    assert run(p, *P, x) == [x[perm[i]] for i in range(n)]


@pytest.mark.parametrize("p", PS)
def test_transpose_invariants(p):
    R = random.Random(100 + p)
    for trial in range(6):
        n = R.randint(1, 14)
        rowptr, cols, vals = rand_csr(R, n, p)
        x = rand_x(R, n, p)
        D = dense_of(n, rowptr, cols, vals)
        DT = [[D[j][i] for j in range(n)] for i in range(n)]
        rpt, ct, vt = csr_of_dense(DT)
        # 4: spmv_t(A, x) == spmv(explicit A^T, x)
        assert run(p, rowptr, cols, vals, x, t=True) == run(p, rpt, ct, vt, x)
        # 3: (A^T)^T == A (CSR arrays identical) via the oracle's own transpose
        r1, c1, perm1 = mpref.transpose(n, rowptr, cols)
        r2, c2, perm2 = mpref.transpose(n, r1, c1)
        assert np.array_equal(r2, rowptr) and np.array_equal(c2, cols)
        assert np.array_equal(np.asarray(perm1)[perm2], np.arange(len(cols)))


@pytest.mark.parametrize("p", [32, 64, 128])
def test_small_integers_exact(p):
    """|entries| < 2^8, n <= 24 -> every partial sum < 2^21 <= 2^p: exact."""
    R = random.Random(200 + p)
    for trial in range(6):
        n = R.randint(1, 24)
        rowptr, cols, vals = rand_csr(R, n, p, density=0.5, small_int=True)
        xi = [R.randint(-(2 ** 7), 2 ** 7) for _ in range(n)]
        x = [int_to_triple(v, p) for v in xi]
        y = run(p, rowptr, cols, vals, x)
        for i in range(n):
            exact = 0
            for k in range(rowptr[i], rowptr[i + 1]):
                exact += int(pinlib.to_frac(vals[k], p)) * xi[cols[k]]
            assert y[i] == int_to_triple(exact, p)


@pytest.mark.parametrize("p", PS)
def test_scaling_and_negation(p):
    R = random.Random(300 + p)
    for trial in range(5):
        n = R.randint(1, 14)
        rowptr, cols, vals = rand_csr(R, n, p)
        x = rand_x(R, n, p)
        y = run(p, rowptr, cols, vals, x)
        for kexp in (-3, 5):
            vs = [(s, M, e + kexp) if M else (s, M, e) for (s, M, e) in vals]
            ys = run(p, rowptr, cols, vs, x)
            assert ys == [(s, M, e + kexp) if M else (0, 0, 0) for (s, M, e) in y]
        vn = [(1 - s, M, e) if M else (s, M, e) for (s, M, e) in vals]
        yn = run(p, rowptr, cols, vn, x)
        assert yn == [(1 - s, M, e) if M else (0, 0, 0) for (s, M, e) in y]


@pytest.mark.parametrize("p", PS)
def test_densification_changes_nothing(p):
    """Adding explicit zeros (any sign/exp) anywhere, i.e. dense MV, is bitwise equal."""
    R = random.Random(400 + p)
    for trial in range(5):
        n = R.randint(1, 12)
        rowptr, cols, vals = rand_csr(R, n, p)
        x = rand_x(R, n, p)
        D = dense_of(n, rowptr, cols, vals)
        Dd = [[D[i][j] if D[i][j] is not None else (R.getrandbits(1), 0, R.randint(-9, 9))
               for j in range(n)] for i in range(n)]
        rpd, cd, vd = csr_of_dense(Dd)
        al, ae, as_ = mpref.pack_vec(vd, p)
        for k, v in enumerate(vd):   # junk sign/exp on zeros
            if v[1] == 0:
                ae[k], as_[k] = v[2], v[0]
        xl, xe, xs = mpref.pack_vec(x, p)
        yd = mpref.unpack_vec(*mpref.spmv(p, rpd, cd, al, ae, as_, xl, xe, xs), p)
        assert yd == run(p, rowptr, cols, vals, x)


def test_chain_is_not_exact_sum():
    """Sanity: the chain is NOT a single rounding of the exact row sum (A.2)."""
    p = 32
    one = (0, 1 << 31, 1)
    tiny = (0, 1 << 31, -31)
    s = mpref.row_chain(p, [(one, one), (one, tiny), (one, tiny)])
    exact = pinlib.frac_round(Fraction(1) + Fraction(2, 2 ** 32), p)
    assert s == one and exact != one


def test_empty_rows_and_determinism():
    p = 64
    R = random.Random(5)
    rowptr = np.array([0, 0, 2, 2], np.int64)
    cols = np.array([0, 2], np.int32)
    vals = [(0, 1 << 63, 1), (1, 1 << 63, 2)]
    x = rand_x(R, 3, p)
    y1 = run(p, rowptr, cols, vals, x)
    y2 = run(p, rowptr, cols, vals, x)
    assert y1 == y2 and y1[0] == (0, 0, 0) and y1[2] == (0, 0, 0)
