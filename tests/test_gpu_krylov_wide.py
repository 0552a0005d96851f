"""GPU parity of the solver path at p > 1024 (krylov_wide.cu; SURVEY.md 8(f)
ranks 1-3 - the paper's BiCG runs at >= 2048 bits) against
the CPU oracle (oracle/krylov.py), bit-exact: ordered-chain dot products,
axpy, and whole BiCG / GPBiCG solves (iterate, iteration count, status) whose
scalar steps use the warp-distributed division and square root."""
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
    l, e, s = gen.configs.rand_values(rng, n, p // 32, elo, ehi)
    if zeros:
        l[rng.random(n) < zeros] = 0
    return oracle.unpack_vec(l, e, s, p)


@pytest.mark.parametrize("p,n", [(2048, 1), (2048, 33), (2048, 700), (4096, 200), (8192, 40)])
def test_wide_dot_parity(p, n):
    import torch
    from paper_1411_2377_b200.csr import dot
    rng = np.random.default_rng(p + n)
    u = _rand_vals(rng, n, p, -30, 30, zeros=0.05)
    v = _rand_vals(rng, n, p, -30, 30)
    got = dot(p, _vec(u, p), _vec(v, p))
    torch.cuda.synchronize()
    assert_same(got.to_host(), oracle.pack_vec([K.dot(u, v, p)], p), f"dot p={p} n={n}")
    # exact cancellation: (u, -u) over ones = +0
    ones = [K.from_int(1, p)] * n
    both = u + [K.neg(a) for a in u]
    got = dot(p, _vec(both, p), _vec(ones + ones, p))
    torch.cuda.synchronize()
    assert_same(got.to_host(), oracle.pack_vec([K.dot(both, ones + ones, p)], p), "cancel")


@pytest.mark.parametrize("p", [2048, 8192])
@pytest.mark.parametrize("negate", [False, True])
def test_wide_axpy_parity(p, negate):
    import torch
    from paper_1411_2377_b200.csr import axpy
    rng = np.random.default_rng(p + int(negate))
    n = 300
    x = _rand_vals(rng, n, p, -10, 10, zeros=0.05)
    y = _rand_vals(rng, n, p, -10, 10, zeros=0.05)
    al = _rand_vals(rng, 1, p, -3, 3)
    got = axpy(p, _vec(al, p), _vec(x, p), _vec(y, p), negate=negate)
    torch.cuda.synchronize()
    assert_same(got.to_host(), oracle.pack_vec(K.axpy(al[0], x, y, p, negate=negate), p),
                f"axpy p={p} neg={negate}")


def _band(n, p, seed):
    rng = np.random.default_rng(seed)
    rowptr, colidx = gen.configs.pattern_band(n, 5)
    limbs, exps, signs = gen.configs.rand_values(rng, len(colidx), p // 32, -8, 0)
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    exps[colidx == rows] = 4
    xt = [K.from_int(i + 1, p) for i in range(n)]
    b = oracle.unpack_vec(*oracle.spmv(p, rowptr, colidx, limbs, exps, signs,
                                       *oracle.pack_vec(xt, p)), p)
    return (rowptr, colidx, limbs, exps, signs), b


@pytest.mark.parametrize("solver,n,p,max_iter", [("bicg", 30, 2048, 4), ("bicg", 12, 4096, 3),
                                                 ("gpbicg", 20, 2048, 3), ("bicg", 24, 2048, 80),
                                                 ("gpbicg", 24, 2048, 80)])
def test_wide_solver_parity(solver, n, p, max_iter):
    import torch
    from paper_1411_2377_b200 import CSR
    A, b = _band(n, p, seed=n + p)
    want = (K.bicg if solver == "bicg" else K.gpbicg)(p, A, b, max_iter)
    H = CSR(p, *A, transpose=(solver == "bicg"))
    x, it, status = (H.bicg if solver == "bicg" else H.gpbicg)(_vec(b, p), max_iter)
    torch.cuda.synchronize()
    assert (it, status) == (want["iters"], want["status"])
    assert_same(x.to_host(), oracle.pack_vec(want["x"], p), f"{solver} n={n} p={p}")
    H.close()


def test_wide_bicg_identity_converges():
    import torch
    from paper_1411_2377_b200 import CSR
    p, n = 2048, 10
    limbs, exps, signs = oracle.pack_vec([K.from_int(1, p)] * n, p)
    rowptr = np.arange(n + 1, dtype=np.int64)
    colidx = np.arange(n, dtype=np.int32)
    b = [K.from_int(3 * i + 1, p) for i in range(n)]
    H = CSR(p, rowptr, colidx, limbs, exps, signs, transpose=True)
    x, it, status = H.bicg(_vec(b, p), 5)
    torch.cuda.synchronize()
    assert (it, status) == (1, "converged")
    assert_same(x.to_host(), oracle.pack_vec(b, p), "identity")
    H.close()


@pytest.mark.parametrize("kind", ["random", "positive", "growing", "cancel", "huge", "ties"])
def test_wide_dot_segmented_paths(kind):
    """The segmented speculative dot at p = 2048 (64-element segments) must
    equal the ordered chain in every regime: committed segments, drifting
    binade, exact cancellation to +0, fp64-overflowing guesses, grid ties."""
    import zlib
    import torch
    from paper_1411_2377_b200.csr import dot
    from test_gpu_krylov import _dot_case
    p, n = 2048, 3000
    rng = np.random.default_rng(zlib.crc32(f"wide-{kind}".encode()))
    u, v = _dot_case(kind, n, p, rng)
    got = dot(p, _vec(u, p), _vec(v, p))
    torch.cuda.synchronize()
    assert_same(got.to_host(), oracle.pack_vec([K.dot(u, v, p)], p), f"dot {kind}")
