"""GPU parity of the BiCG path against the CPU oracle
(oracle/krylov.py), bit-exact: the ordered-chain dot product, axpy, and whole
BiCG solves (iterate x, iteration count, status) on diagonally dominant
banded systems and C1-like random systems, b = A [1..n]^T."""
import zlib

import numpy as np
import pytest

import gen
import oracle
from oracle import krylov as K
from gpu_util import assert_same

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    import __graft_entry__
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    __graft_entry__.build()


def _vec(vals, p):
    from paper_1411_2377_b200 import MPVec
    return MPVec.from_host(*oracle.pack_vec(vals, p), device="cuda:0")


def _rand_vals(rng, n, p, elo, ehi, zeros=0.0):
    L = p // 32
    l, e, s = gen.configs.rand_values(rng, n, L, elo, ehi)
    if zeros:
        z = rng.random(n) < zeros
        l[z] = 0
    return oracle.unpack_vec(l, e, s, p)


@pytest.mark.parametrize("p", [32, 64, 128, 256, 512, 1024])
@pytest.mark.parametrize("n", [1, 31, 33, 200, 3000])
def test_dot_parity(p, n):
    import torch
    from paper_1411_2377_b200.csr import dot
    rng = np.random.default_rng(p * 7 + n)
    u = _rand_vals(rng, n, p, -30, 30, zeros=0.05)
    v = _rand_vals(rng, n, p, -30, 30)
    got = dot(p, _vec(u, p), _vec(v, p))
    torch.cuda.synchronize()
    want = oracle.pack_vec([K.dot(u, v, p)], p)
    assert_same(got.to_host(), want, f"dot p={p} n={n}")


def test_dot_cancellation_and_ties():
    """(u, -u) = +0 exactly; tie-prone sums; an empty vector gives +0."""
    import torch
    from paper_1411_2377_b200.csr import dot
    p = 128
    rng = np.random.default_rng(1)
    u = _rand_vals(rng, 100, p, -4, 4)
    ones = [K.from_int(1, p)] * 100
    neg = [K.neg(a) for a in u]
    both = u + neg
    got = dot(p, _vec(both, p), _vec(ones + ones, p))
    torch.cuda.synchronize()
    assert_same(got.to_host(), oracle.pack_vec([K.dot(both, ones + ones, p)], p), "cancel")
    # products 1, 2^-p, 2^-p, ... : every add a grid tie
    tiny = (0, 1 << (p - 1), 1 - p)
    w = [K.from_int(1, p)] + [tiny] * 40
    got = dot(p, _vec(w, p), _vec([K.from_int(1, p)] * 41, p))
    torch.cuda.synchronize()
    assert_same(got.to_host(), oracle.pack_vec([K.dot(w, [K.from_int(1, p)] * 41, p)], p), "ties")


@pytest.mark.parametrize("p", [64, 256, 1024])
@pytest.mark.parametrize("negate", [False, True])
def test_axpy_parity(p, negate):
    import torch
    from paper_1411_2377_b200.csr import axpy
    rng = np.random.default_rng(p + int(negate))
    n = 1000
    x = _rand_vals(rng, n, p, -10, 10, zeros=0.05)
    y = _rand_vals(rng, n, p, -10, 10, zeros=0.05)
    al = _rand_vals(rng, 1, p, -3, 3)
    got = axpy(p, _vec(al, p), _vec(x, p), _vec(y, p), negate=negate)
    torch.cuda.synchronize()
    want = oracle.pack_vec(K.axpy(al[0], x, y, p, negate=negate), p)
    assert_same(got.to_host(), want, f"axpy p={p} neg={negate}")


def _system(kind, n, p, seed):
    rng = np.random.default_rng(seed)
    L = p // 32
    if kind == "band":                         # C2 with off-diag exp U[-8, 0]
        rowptr, colidx = gen.configs.pattern_band(n, 5)
        limbs, exps, signs = gen.configs.rand_values(rng, len(colidx), L, -8, 0)
        rows = np.repeat(np.arange(n), np.diff(rowptr))
        exps[colidx == rows] = 4
    else:                                      # C1-like random pattern, dominant diagonal
        rowptr, colidx = gen.configs.pattern_diag_plus_random(rng, n, np.full(n, 3))
        limbs, exps, signs = gen.configs.rand_values(rng, len(colidx), L, -6, 0)
        rows = np.repeat(np.arange(n), np.diff(rowptr))
        exps[colidx == rows] = 3
    xt = [K.from_int(i + 1, p) for i in range(n)]
    xl, xe, xs = oracle.pack_vec(xt, p)
    b = oracle.unpack_vec(*oracle.spmv(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs), p)
    return (rowptr, colidx, limbs, exps, signs), b


@pytest.mark.parametrize("kind,n,p,max_iter", [("band", 60, 128, 200), ("band", 150, 256, 300),
                                               ("random", 80, 128, 300), ("band", 40, 512, 100),
                                               ("band", 30, 1024, 3), ("random", 50, 256, 5)])
def test_bicg_parity(kind, n, p, max_iter):
    import torch
    from paper_1411_2377_b200 import CSR
    A, b = _system(kind, n, p, seed=n + p)
    want = K.bicg(p, A, b, max_iter)
    H = CSR(p, *A, transpose=True)
    x, it, status = H.bicg(_vec(b, p), max_iter)
    torch.cuda.synchronize()
    assert (it, status) == (want["iters"], want["status"])
    assert_same(x.to_host(), oracle.pack_vec(want["x"], p), f"bicg {kind} n={n} p={p}")
    H.close()


def test_bicg_identity_and_errors():
    import torch
    from paper_1411_2377_b200 import CSR, MpspError
    p, n = 128, 20
    one = K.from_int(1, p)
    limbs, exps, signs = oracle.pack_vec([one] * n, p)
    rowptr = np.arange(n + 1, dtype=np.int64)
    colidx = np.arange(n, dtype=np.int32)
    b = [K.from_int(i + 1, p) for i in range(n)]
    H = CSR(p, rowptr, colidx, limbs, exps, signs, transpose=True)
    x, it, status = H.bicg(_vec(b, p), 10)
    torch.cuda.synchronize()
    assert (it, status) == (1, "converged")
    assert_same(x.to_host(), oracle.pack_vec(b, p), "identity")
    H.close()
    H = CSR(p, rowptr, colidx, limbs, exps, signs, transpose=False)
    with pytest.raises(MpspError):
        H.bicg(_vec(b, p), 10)                    # needs the transpose
    H.close()
    l64, e64, s64 = oracle.pack_vec([K.from_int(1, 64)] * n, 64)
    H = CSR(64, rowptr, colidx, l64, e64, s64, transpose=True)
    with pytest.raises(MpspError):
        H.bicg(_vec([K.from_int(1, 64)] * n, 64), 10)   # p >= 128
    H.close()


def _dot_case(kind, n, p, rng):
    L = p // 32
    if kind == "random":
        return _rand_vals(rng, n, p, -30, 30, zeros=0.02), _rand_vals(rng, n, p, -30, 30)
    if kind == "growing":          # running sum's binade keeps changing across segments
        u = _rand_vals(rng, n, p, 0, 0)
        u = [(s, M, E + (k * 60) // n) for k, (s, M, E) in enumerate(u)]
        return u, _rand_vals(rng, n, p, 0, 2)
    if kind == "cancel":           # exact cancellation back to +0 mid-chain, then restart
        h = n // 2
        u = _rand_vals(rng, h, p, -5, 5)
        v = _rand_vals(rng, h, p, -5, 5)
        # second half: the negated products of the first half in REVERSE order do not
        # cancel exactly under rounding; instead repeat the first half with u negated
        return u + [K.neg(a) for a in u] + _rand_vals(rng, n - 2 * h, p, -5, 5), \
            v + v + _rand_vals(rng, n - 2 * h, p, -5, 5)
    if kind == "positive":         # monotone sum: binade changes only ~log2(n) times
        u = [(0, M, E) for (_, M, E) in _rand_vals(rng, n, p, -8, 8)]
        return u, [(0, M, E) for (_, M, E) in _rand_vals(rng, n, p, -8, 8)]
    if kind == "huge":             # fp64 estimates overflow: every guess invalid
        u = _rand_vals(rng, n, p, -(1 << 28), 1 << 28)
        return u, _rand_vals(rng, n, p, -10, 10)
    if kind == "ties":             # small gaps with 10..0 tails: grid ties everywhere
        one = K.from_int(1, p)
        u = [one] + [(rng.integers(0, 2), (1 << (p - 1)) | (1 << int(rng.integers(0, 3))), -p + 2)
                     for _ in range(n - 1)]
        return u, [one] * n
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["random", "positive", "growing", "cancel", "huge", "ties"])
@pytest.mark.parametrize("p,n", [(128, 20000), (256, 60000), (1024, 4000)])
def test_dot_segmented_paths(kind, p, n):
    """The segmented speculative dot (n > 256) must equal the ordered chain in
    every regime: stable binade (segments committed), drifting binade,
    exact cancellation to +0, fp64-overflowing guesses, grid ties."""
    import torch
    from paper_1411_2377_b200.csr import dot
    rng = np.random.default_rng(zlib.crc32(f"{kind}-{p}-{n}".encode()))
    from paper_1411_2377_b200._lib import dot_stats
    u, v = _dot_case(kind, n, p, rng)
    dot_stats()
    got = dot(p, _vec(u, p), _vec(v, p))
    torch.cuda.synchronize()
    st = dot_stats()
    assert_same(got.to_host(), oracle.pack_vec([K.dot(u, v, p)], p), f"dot {kind} p={p} n={n}")
    if kind == "huge":
        assert st["validated"] == 0              # overflowing guesses never commit
    if kind == "positive":
        assert st["validated"] > st["sequential"]   # the speculative path carries the chain


@pytest.mark.parametrize("kind,n,p,max_iter", [("band", 60, 128, 200), ("band", 150, 256, 300),
                                               ("random", 80, 128, 300), ("band", 40, 512, 100),
                                               ("band", 30, 1024, 4), ("random", 50, 256, 6)])
def test_gpbicg_parity(kind, n, p, max_iter):
    import torch
    from paper_1411_2377_b200 import CSR
    A, b = _system(kind, n, p, seed=3 * n + p)
    want = K.gpbicg(p, A, b, max_iter)
    H = CSR(p, *A)                                 # transpose-free: no A^T needed
    x, it, status = H.gpbicg(_vec(b, p), max_iter)
    torch.cuda.synchronize()
    assert (it, status) == (want["iters"], want["status"])
    assert_same(x.to_host(), oracle.pack_vec(want["x"], p), f"gpbicg {kind} n={n} p={p}")
    H.close()


def test_gpbicg_identity():
    import torch
    from paper_1411_2377_b200 import CSR
    p, n = 256, 33
    limbs, exps, signs = oracle.pack_vec([K.from_int(1, p)] * n, p)
    rowptr = np.arange(n + 1, dtype=np.int64)
    colidx = np.arange(n, dtype=np.int32)
    b = [K.from_int(i + 1, p) for i in range(n)]
    H = CSR(p, rowptr, colidx, limbs, exps, signs)
    x, it, status = H.gpbicg(_vec(b, p), 10)
    torch.cuda.synchronize()
    assert (it, status) == (1, "converged")
    assert_same(x.to_host(), oracle.pack_vec(b, p), "gpbicg identity")
    H.close()
