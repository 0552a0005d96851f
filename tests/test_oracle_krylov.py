"""Pins of the BiCG oracle (oracle/krylov.py).

Scalar operations against MPFR (mpfr_div / mpfr_sqrt, RNDN, through ctypes)
and against exact rational arithmetic with one correct rounding; the solver
against properties the mathematics fixes: BiCG on the identity converges in
one iteration to x = b exactly, the first iterates agree with an exact
rational-arithmetic BiCG to within the rounding error of p bits, and on a
well-conditioned diagonally dominant system the residual falls below the
paper's threshold and A x reproduces b to p-bit accuracy."""
import random
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle
from oracle import krylov as K
from pinlib import frac_round, to_frac, try_mpfr

MP = try_mpfr()


def _rand(rng, p, elo=-40, ehi=40, sign=True):
    return ((rng.getrandbits(1) if sign else 0), (1 << (p - 1)) | rng.getrandbits(p - 1),
            rng.randint(elo, ehi))


@pytest.mark.parametrize("p", [32, 64, 128, 256, 512, 1024])
def test_div_sqrt_vs_fraction(p):
    rng = random.Random(p)
    for _ in range(300):
        a, b = _rand(rng, p), _rand(rng, p)
        assert K.div(a, b, p) == frac_round(to_frac(a, p) / to_frac(b, p), p)
        c = (0,) + _rand(rng, p)[1:]
        # sqrt: exact check via the defining inequality of RN
        r = K.sqrt(c, p)
        v = to_frac(c, p)
        rv = to_frac(r, p)
        ulp = Fraction(2) ** (r[2] - p)
        lo, hi = rv - ulp / 2, rv + ulp / 2
        if r[1] == 1 << (p - 1):                  # lower binade below a power of 2
            lo = rv - ulp / 4
        assert lo * lo <= v <= hi * hi


@pytest.mark.skipif(MP is None, reason="libmpfr not available")
@pytest.mark.parametrize("p", [32, 64, 128, 256, 512, 1024])
def test_div_sqrt_vs_mpfr(p):
    import ctypes
    rng = random.Random(7 * p)
    for _ in range(400):
        a, b = _rand(rng, p), _rand(rng, p)
        assert K.div(a, b, p) == MP.op("mpfr_div", a, b, p)
        c = (0,) + _rand(rng, p)[1:]
        xa, xr = MP._new(p), MP._new(p)
        try:
            MP._set(xa, c, p)
            MP.lib.mpfr_sqrt(ctypes.byref(xr), ctypes.byref(xa), 0)
            assert K.sqrt(c, p) == MP._get(xr, p)
        finally:
            MP.lib.mpfr_clear(ctypes.byref(xa))
            MP.lib.mpfr_clear(ctypes.byref(xr))


@pytest.mark.parametrize("p", [64, 128, 256])
def test_scalar_special_cases(p):
    two = K.from_int(2, p)
    three = K.from_int(3, p)
    assert K.div(K.from_int(6, p), three, p) == two                 # exact quotient
    assert K.sqrt(K.from_int(9, p), p) == three                      # perfect square
    assert K.sqrt(K.from_int(2, p), p)[2] == 1                       # 1.414 in [1, 2)
    assert K.div(oracle.ZERO, three, p) == oracle.ZERO
    with pytest.raises(ZeroDivisionError):
        K.div(three, oracle.ZERO, p)
    for k in (1, 20, 50):
        c = K.recip_pow10(k, p)
        assert c == frac_round(Fraction(1, 10 ** k), p)
    # comparisons
    assert K.le(K.from_int(-5, p), K.from_int(3, p)) and not K.le(three, two)
    assert K.cmp(oracle.ZERO, oracle.ZERO) == 0 and K.cmp(K.from_int(-2, p), K.from_int(-3, p)) == 1


def _diag_dominant(n, p, seed):
    """Banded system like C2 with off-diagonal exponents U[-8, 0] (SURVEY 8(f):
    diagonally dominant), diagonal exponent +4."""
    rng = np.random.default_rng(seed)
    rowptr, colidx = gen.configs.pattern_band(n, 2)
    L = p // 32
    limbs, exps, signs = gen.configs.rand_values(rng, len(colidx), L, -8, 0)
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    exps[colidx == rows] = 4
    return rowptr, colidx, limbs, exps, signs


def test_identity_converges_in_one_step():
    p, n = 128, 12
    rowptr = np.arange(n + 1, dtype=np.int64)
    colidx = np.arange(n, dtype=np.int32)
    one = K.from_int(1, p)
    limbs, exps, signs = oracle.pack_vec([one] * n, p)
    b = [K.from_int(i + 1, p) for i in range(n)]
    res = K.bicg(p, (rowptr, colidx, limbs, exps, signs), b, 20)
    assert res["status"] == "converged" and res["iters"] == 1
    assert res["x"] == b


def _frac_bicg(Af, bf, iters):
    n = len(bf)
    x = [Fraction(0)] * n
    r = list(bf)
    rt = list(r)
    out = []
    rho_prev = pv = pt = None
    for i in range(1, iters + 1):
        rho = sum(a * b for a, b in zip(rt, r))
        if i == 1:
            pv, pt = list(r), list(rt)
        else:
            beta = rho / rho_prev
            pv = [a + beta * b for a, b in zip(r, pv)]
            pt = [a + beta * b for a, b in zip(rt, pt)]
        z = [sum(Af[k][j] * pv[j] for j in range(n)) for k in range(n)]
        zt = [sum(Af[j][k] * pt[j] for j in range(n)) for k in range(n)]
        alpha = rho / sum(a * b for a, b in zip(pt, z))
        x = [a + alpha * b for a, b in zip(x, pv)]
        r = [a - alpha * b for a, b in zip(r, z)]
        rt = [a - alpha * b for a, b in zip(rt, zt)]
        out.append(x)
        rho_prev = rho
    return out


def test_first_iterates_match_exact_rational_bicg():
    """p = 256: iterates x_1..x_3 agree with exact rational BiCG to ~2^-240."""
    p, n = 256, 8
    A = _diag_dominant(n, p, 3)
    rowptr, colidx, limbs, exps, signs = A
    vals = oracle.unpack_vec(limbs, exps, signs, p)
    Af = [[Fraction(0)] * n for _ in range(n)]
    for i in range(n):
        for k in range(rowptr[i], rowptr[i + 1]):
            Af[i][colidx[k]] = to_frac(vals[k], p)
    xt = [K.from_int(i + 1, p) for i in range(n)]
    xl, xe, xs = oracle.pack_vec(xt, p)
    b = oracle.unpack_vec(*oracle.spmv(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs), p)
    bf = [to_frac(v, p) for v in b]
    res = K.bicg(p, A, b, 3)
    exact = _frac_bicg(Af, bf, 3)
    for i in range(n):
        got = to_frac(res["x"][i], p)
        want = exact[2][i]
        assert abs(got - want) <= abs(want) * Fraction(1, 2 ** 240) + Fraction(1, 2 ** 250)


@pytest.mark.parametrize("p", [128, 256])
def test_converges_on_diagonally_dominant_band(p):
    n = 40
    A = _diag_dominant(n, p, 5)
    rowptr, colidx, limbs, exps, signs = A
    xt = [K.from_int(i + 1, p) for i in range(n)]
    xl, xe, xs = oracle.pack_vec(xt, p)
    b = oracle.unpack_vec(*oracle.spmv(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs), p)
    res = K.bicg(p, A, b, 200, trace=True)
    assert res["status"] == "converged", res["status"]
    # residual below the paper's threshold, and x close to [1..n]
    assert K.le(res["norms"][-1], res["thr"])
    for i, v in enumerate(res["x"]):
        assert abs(to_frac(v, p) - (i + 1)) < Fraction(1, 10 ** 15)


def test_gpbicg_identity_converges_in_one_step():
    p, n = 128, 10
    rowptr = np.arange(n + 1, dtype=np.int64)
    colidx = np.arange(n, dtype=np.int32)
    limbs, exps, signs = oracle.pack_vec([K.from_int(1, p)] * n, p)
    b = [K.from_int(i + 1, p) for i in range(n)]
    res = K.gpbicg(p, (rowptr, colidx, limbs, exps, signs), b, 10)
    assert res["status"] == "converged" and res["iters"] == 1
    assert res["x"] == b


@pytest.mark.parametrize("p", [128, 256])
def test_gpbicg_converges_on_diagonally_dominant_band(p):
    n = 40
    A = _diag_dominant(n, p, 6)
    rowptr, colidx, limbs, exps, signs = A
    xt = [K.from_int(i + 1, p) for i in range(n)]
    xl, xe, xs = oracle.pack_vec(xt, p)
    b = oracle.unpack_vec(*oracle.spmv(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs), p)
    res = K.gpbicg(p, A, b, 200)
    assert res["status"] == "converged", res["status"]
    assert K.le(res["norms"][-1], res["thr"])
    for i, v in enumerate(res["x"]):
        assert abs(to_frac(v, p) - (i + 1)) < Fraction(1, 10 ** 15)
    # same system, same solution as BiCG to the test's accuracy, and GPBiCG
    # (transpose-free, two A products per iteration) does not need A^T
    res_b = K.bicg(p, A, b, 200)
    assert res_b["status"] == "converged"


def _frac_gpbicg(Af, bf, iters):
    """Zhang's GPBiCG in exact rational arithmetic (same readings)."""
    n = len(bf)
    mv = lambda v: [sum(Af[k][j] * v[j] for j in range(n)) for k in range(n)]
    dp = lambda a, b: sum(x * y for x, y in zip(a, b))
    x = [Fraction(0)] * n
    r = list(bf)
    rt = list(r)
    u = [Fraction(0)] * n
    z = [Fraction(0)] * n
    out = []
    for i in range(1, iters + 1):
        rho = dp(rt, r)
        if i == 1:
            pv = list(r)
            q = mv(pv)
            alpha = rho / dp(rt, q)
            t = [a - alpha * c for a, c in zip(r, q)]
            v = mv(t)
            y = [alpha * c - a for a, c in zip(r, q)]
            zeta, eta = dp(v, t) / dp(v, v), Fraction(0)
            u = [zeta * c for c in q]
        else:
            beta = (rho / rho_prev) * (alpha_prev / zeta)
            w = [a + beta * c for a, c in zip(v, q)]
            pv = [a + beta * (c - d) for a, c, d in zip(r, pv, u)]
            q = mv(pv)
            alpha = rho / dp(rt, q)
            s = [a - c for a, c in zip(t, r)]
            t = [a - alpha * c for a, c in zip(r, q)]
            v = mv(t)
            y = [a - alpha * (c - d) for a, c, d in zip(s, w, q)]
            m1, m2, m3, m4, m5 = dp(y, y), dp(v, t), dp(y, t), dp(v, y), dp(v, v)
            tau = m5 * m1 - m4 * m4
            zeta = (m1 * m2 - m3 * m4) / tau
            eta = (m5 * m3 - m4 * m2) / tau
            u = [zeta * c + eta * (a + beta * d) for c, a, d in zip(q, s, u)]
        z = [zeta * a + eta * c - alpha * d for a, c, d in zip(r, z, u)]
        x = [a + alpha * c + d for a, c, d in zip(x, pv, z)]
        r = [a - eta * c - zeta * d for a, c, d in zip(t, y, v)]
        out.append(x)
        rho_prev, alpha_prev = rho, alpha
    return out


def test_gpbicg_first_iterates_match_exact_rational():
    p, n = 256, 8
    A = _diag_dominant(n, p, 4)
    rowptr, colidx, limbs, exps, signs = A
    vals = oracle.unpack_vec(limbs, exps, signs, p)
    Af = [[Fraction(0)] * n for _ in range(n)]
    for i in range(n):
        for k in range(rowptr[i], rowptr[i + 1]):
            Af[i][colidx[k]] = to_frac(vals[k], p)
    xl, xe, xs = oracle.pack_vec([K.from_int(i + 1, p) for i in range(n)], p)
    b = oracle.unpack_vec(*oracle.spmv(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs), p)
    res = K.gpbicg(p, A, b, 3)
    exact = _frac_gpbicg(Af, [to_frac(v, p) for v in b], res["iters"])
    for i in range(n):
        got, want = to_frac(res["x"][i], p), exact[-1][i]
        assert abs(got - want) <= abs(want) * Fraction(1, 2 ** 230) + Fraction(1, 2 ** 240)
