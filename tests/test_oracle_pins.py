"""Pins for the CPU oracle (oracle/mpref.py) against things other than itself.

CPU only (no gpu marker).  Each pin is chosen so a plausible mistake in the
oracle (a dropped sticky term, a wrong tie rule, a swapped sign, an off-by-one
exponent, a transposed operand) fails one of them:

  * MPFR mpfr_mul/mpfr_add RNDN (library routine).
  * mpmath.libmp mpf_mul/mpf_add rnd='n' (a second library routine).
  * exact Fraction value + one correct rounding (tests/pinlib.frac_round).
  * hand-worked examples (tests/golden/hand_examples.json).
  * the far-path lemma of SURVEY.md 8(c) at its tight boundary.
  * brute force over exponent gaps x sign pairs x mantissa corpus at p=32/64.
"""
import json
import os
import random

import numpy as np
import pytest

import oracle
from oracle import mpref
import pinlib

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")


def T(v, p):
    """golden [s, [limbs], e] -> oracle triple."""
    s, limbs, e = v
    M = 0
    for i, l in enumerate(limbs):
        M |= int(l) << (32 * i)
    return (0, 0, 0) if M == 0 else (s, M, e)


# --------------------------------------------------------------- corpora
def corpus_mantissas(p, rng):
    top = 1 << (p - 1)
    full = (1 << p) - 1
    ms = [top, full, top | 1, top | (1 << (p // 2)), full ^ 1, full ^ (1 << (p - 2)),
          top | ((1 << (p - 2)) - 1)]
    # limb-boundary patterns: low limbs all ones / single bits at limb edges
    for k in range(1, p // 32):
        ms.append(top | ((1 << (32 * k)) - 1))
        ms.append(top | (1 << (32 * k)))
        ms.append(top | (1 << (32 * k - 1)))
    for _ in range(6):
        ms.append(top | rng.getrandbits(p - 1))
    return ms


def rand_val(p, rng, espread=8, tieprone=False):
    if tieprone:
        # few significant bits -> products/sums land on ties often
        nb = rng.randint(1, min(p, 6))
        M = (1 << (nb - 1)) | rng.getrandbits(nb - 1) if nb > 1 else 1
        M <<= (p - nb)
    else:
        M = (1 << (p - 1)) | rng.getrandbits(p - 1)
    return (rng.getrandbits(1), M, rng.randint(-espread, espread))


# --------------------------------------------------------------- golden
def test_golden_ops():
    g = json.load(open(GOLDEN))
    for c in g["mul"]:
        p = c["p"]
        assert mpref.mul(T(c["a"], p), T(c["b"], p), p) == T(c["r"], p), c["name"]
    for c in g["add"]:
        p = c["p"]
        assert mpref.add(T(c["a"], p), T(c["b"], p), p) == T(c["r"], p), c["name"]


def _golden_csr(c):
    p = c["p"]
    L = p // 32
    A = [T(v, p) for v in c["A"]]
    x = [T(v, p) for v in c["x"]]
    al, ae, as_ = mpref.pack_vec(A, p)
    xl, xe, xs = mpref.pack_vec(x, p)
    return p, np.array(c["rowptr"], np.int64), np.array(c["colidx"], np.int32), al, ae, as_, xl, xe, xs


def test_golden_spmv():
    g = json.load(open(GOLDEN))
    for c in g["spmv"]:
        p, rp, ci, al, ae, as_, xl, xe, xs = _golden_csr(c)
        y = mpref.unpack_vec(*mpref.spmv(p, rp, ci, al, ae, as_, xl, xe, xs), p)
        assert y == [T(v, p) for v in c["y"]], c["name"]
        if "yt" in c:
            yt = mpref.unpack_vec(*mpref.spmv_t(p, rp, ci, al, ae, as_, xl, xe, xs), p)
            assert yt == [T(v, p) for v in c["yt"]], c["name"]


def test_golden_values_agree_with_mpfr():
    """The hand-worked expectations themselves are right (checked by MPFR)."""
    mp = pinlib.try_mpfr()
    if mp is None:
        pytest.skip("libmpfr not present")
    g = json.load(open(GOLDEN))
    for c in g["mul"]:
        p = c["p"]
        assert mp.mul(T(c["a"], p), T(c["b"], p), p) == T(c["r"], p), c["name"]
    for c in g["add"]:
        p = c["p"]
        assert mp.add(T(c["a"], p), T(c["b"], p), p) == T(c["r"], p), c["name"]
    for c in g["spmv"]:
        p = c["p"]
        A = [T(v, p) for v in c["A"]]
        x = [T(v, p) for v in c["x"]]
        rp, ci = c["rowptr"], c["colidx"]
        n = c["n"]
        y = []
        for i in range(n):
            s = (0, 0, 0)
            for k in range(rp[i], rp[i + 1]):
                s = mp.add(s, mp.mul(A[k], x[ci[k]], p), p)
            y.append(s)
        assert y == [T(v, p) for v in c["y"]], c["name"]


# --------------------------------------------------------------- libraries
PS = [32, 64, 96, 128, 256, 512, 1024]


@pytest.mark.parametrize("p", PS)
def test_vs_mpfr_random(p):
    mp = pinlib.try_mpfr()
    if mp is None:
        pytest.skip("libmpfr not present")
    rng = random.Random(1000 + p)
    nops = 1500 if p <= 256 else 600
    for it in range(nops):
        kind = it % 4
        if kind == 0:
            a, b = rand_val(p, rng, 3 * p), rand_val(p, rng, 3 * p)
        elif kind == 1:
            a, b = rand_val(p, rng, 4, True), rand_val(p, rng, 4, True)
        elif kind == 2:  # near cancellation
            a = rand_val(p, rng, 4)
            s, M, E = a
            delta = rng.randint(-3, 3)
            M2 = min(max(M + delta, 1 << (p - 1)), (1 << p) - 1)
            b = (1 - s, M2, E + rng.choice([0, 0, 1, -1]))
        else:  # gap near p
            a = rand_val(p, rng, 2)
            b = rand_val(p, rng, 2)
            b = (b[0], b[1], a[2] - rng.choice([p - 1, p, p + 1, p + 2, 31, 32, 33]))
        assert mpref.add(a, b, p) == mp.add(a, b, p), (p, a, b)
        assert mpref.mul(a, b, p) == mp.mul(a, b, p), (p, a, b)


@pytest.mark.parametrize("p", PS)
def test_vs_mpmath_random(p):
    mmul, madd = pinlib.mpmath_ops()
    rng = random.Random(2000 + p)
    for it in range(800):
        tie = (it % 2 == 0)
        a = rand_val(p, rng, 2 * p, tie)
        b = rand_val(p, rng, 2 * p, tie)
        if it % 5 == 0:
            b = (1 - a[0], a[1], a[2])  # exact cancellation
        assert mpref.add(a, b, p) == madd(a, b, p), (p, a, b)
        assert mpref.mul(a, b, p) == mmul(a, b, p), (p, a, b)


# --------------------------------------------------------------- Fraction
@pytest.mark.parametrize("p", [32, 64, 128])
def test_vs_fraction_single_rounding(p):
    rng = random.Random(3000 + p)
    for it in range(600):
        a = rand_val(p, rng, 2 * p, it % 3 == 0)
        b = rand_val(p, rng, 2 * p, it % 3 == 0)
        fa, fb = pinlib.to_frac(a, p), pinlib.to_frac(b, p)
        assert mpref.mul(a, b, p) == pinlib.frac_round(fa * fb, p)
        assert mpref.add(a, b, p) == pinlib.frac_round(fa + fb, p)


def test_rn_vs_fraction():
    rng = random.Random(7)
    for p in (32, 64, 96):
        for _ in range(500):
            N = rng.getrandbits(rng.randint(1, 3 * p)) | 1
            f = rng.randint(-200, 200)
            M, E = mpref.rn(N, f, p)
            ref = pinlib.frac_round(pinlib.Fraction(N) * pinlib.Fraction(2) ** f, p)
            assert (0, M, E) == ref


def test_one_nnz_row_is_single_rounding():
    """A 1-nnz row is exactly RN(a*x): chain start at +0 adds nothing."""
    rng = random.Random(11)
    p = 64
    for _ in range(200):
        a, x = rand_val(p, rng, 8), rand_val(p, rng, 8)
        s = mpref.row_chain(p, [(a, x)])
        assert s == pinlib.frac_round(pinlib.to_frac(a, p) * pinlib.to_frac(x, p), p)


# --------------------------------------------------------------- brute force
@pytest.mark.parametrize("p", [32, 64])
def test_brute_force_gaps(p):
    """Every exponent gap d in [-2p-4, 2p+4] x sign pairs x mantissa corpus."""
    rng = random.Random(4000 + p)
    ms = corpus_mantissas(p, rng)[:9]
    mmul, madd = pinlib.mpmath_ops()
    for d in range(-2 * p - 4, 2 * p + 5):
        for sa in (0, 1):
            for sb in (0, 1):
                for Ma in ms[::2]:
                    for Mb in ms[1::2]:
                        a, b = (sa, Ma, 5), (sb, Mb, 5 - d)
                        r = mpref.add(a, b, p)
                        assert r == pinlib.frac_round(pinlib.to_frac(a, p) + pinlib.to_frac(b, p), p)
                        assert r == madd(a, b, p)


# --------------------------------------------------------------- far path
@pytest.mark.parametrize("p", [32, 64, 128])
def test_far_path_lemma(p, monkeypatch):
    """d >= p+2 -> RN(big + small) = big; tight: d = p+1 can differ."""
    rng = random.Random(5000 + p)
    differs_at_p1 = 0
    for _ in range(400):
        big = rand_val(p, rng, 4)
        if rng.random() < 0.3:
            big = (big[0], 1 << (p - 1), big[2])  # power of two: lower binade
        small = rand_val(p, rng, 0)
        for d in (p + 1, p + 2, p + 3, 2 * p, 8 * p):
            sm = (small[0], small[1], big[2] - d)
            exact = pinlib.frac_round(pinlib.to_frac(big, p) + pinlib.to_frac(sm, p), p)
            assert mpref.add(big, sm, p) == exact
            if d >= p + 2:
                assert exact == big
            elif exact != big:
                differs_at_p1 += 1
    assert differs_at_p1 > 0
    # the shortcut branch itself (threshold lowered) agrees with exact alignment
    monkeypatch.setattr(mpref, "FAR_THRESHOLD", 0)
    for _ in range(200):
        big = rand_val(p, rng, 4)
        small = rand_val(p, rng, 0)
        for d in (p + 2, p + 5, 3 * p):
            sm = (small[0], small[1], big[2] - d)
            assert mpref.add(big, sm, p) == big
            assert mpref.add(sm, big, p) == big


def test_huge_exponent_gap_uses_lemma():
    p = 64
    big = (0, (1 << 63) | 12345, 1 << 29)
    small = (1, (1 << 63) | 999, -(1 << 29))
    assert mpref.add(big, small, p) == big
    assert mpref.add(small, big, p) == big


# --------------------------------------------------------------- conversions
def test_pack_unpack_roundtrip():
    rng = random.Random(6)
    for p in (32, 128, 1024):
        vals = [rand_val(p, rng, 100) for _ in range(20)] + [(0, 0, 0)]
        l, e, s = mpref.pack_vec(vals, p)
        assert l.dtype == np.uint32 and l.shape == (21, p // 32)
        assert mpref.unpack_vec(l, e, s, p) == vals
        # limb 0 least significant: the top limb carries the MSB
        assert all(int(l[i, -1]) >> 31 == 1 for i in range(20))


def test_zero_with_junk_sign_exp_reads_as_zero():
    p = 64
    l = np.zeros((1, 2), np.uint32)
    assert mpref.unpack(l[0], 77, 1, p) == (0, 0, 0)


def test_unnormalised_input_rejected():
    with pytest.raises(ValueError):
        mpref.unpack(np.array([1, 0], np.uint32), 0, 0, 64)
