"""GPU dense MP MV (mpsp_dense_create)
on the sparsified Lotkin matrix: bit-exact against the oracle's dense_mv, and
bitwise equal to the sparse path on the CSR of the nonzeros (SPEC S:151,
S:522), for A x and A^T x, at p <= 1024 (warp-row kernel, no column
indices) and p = 2048 (warp-cooperative kernel)."""
import numpy as np
import pytest

import oracle
from gen import lotkin as LK
from gpu_util import assert_same

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    import __graft_entry__
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    __graft_entry__.build()


def _run(d, dense, op, rows=None):
    from paper_1411_2377_b200 import CSR, MPVec
    p, n = d["p"], d["n"]
    if dense:
        A = CSR.dense(p, n, d["dense_limbs"], d["dense_exps"], d["dense_signs"], rows=rows,
                      transpose=(op == "atx"))
    else:
        A = CSR(p, d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"], rows=rows,
                transpose=(op == "atx"))
    x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda:0")
    y = (A.spmv(x) if op == "ax" else A.spmv_t(x)).to_host()
    A.close()
    return y


@pytest.mark.parametrize("p", [128, 512, 1024, 2048])
@pytest.mark.parametrize("n,s", [(1, 0), (33, 0), (70, 50), (150, 90), (120, 99)])
def test_dense_vs_oracle_and_sparse(n, s, p):
    d = LK.make(n, s, p, seed=n + p)
    xa = (d["x_limbs"], d["x_exps"], d["x_signs"])
    for op in ("ax", "atx"):
        want = oracle.dense_mv(p, n, d["dense_limbs"], d["dense_exps"], d["dense_signs"], *xa,
                               transpose=(op == "atx"))
        got_dense = _run(d, True, op)
        assert_same(got_dense, want, f"dense n={n} s={s} p={p} {op}")
        assert_same(_run(d, False, op), want, f"sparse n={n} s={s} p={p} {op}")


def test_dense_row_block_and_errors():
    from paper_1411_2377_b200 import CSR, MpspError
    d = LK.make(90, 50, 256, seed=1)
    want = oracle.dense_mv(256, 90, d["dense_limbs"], d["dense_exps"], d["dense_signs"],
                           d["x_limbs"], d["x_exps"], d["x_signs"])
    got = _run(d, True, "ax", rows=(17, 61))
    assert_same(got, tuple(a[17:61] for a in want), "dense row block")
    bad = d["dense_limbs"].copy()
    bad[5, -1] = 1                                   # unnormalised nonzero
    with pytest.raises(MpspError):
        CSR.dense(256, 90, bad, d["dense_exps"], d["dense_signs"])
    with pytest.raises(MpspError):
        CSR.dense(256, 50000, np.zeros((1, 8), np.uint32), np.zeros(1, np.int32), np.zeros(1, np.uint8))


@pytest.mark.parametrize("p", [256, 2048])
def test_dense_empty_and_single(p):
    """n = 0 (nothing to do) and n = 1 (one product, RN(+0 + t) = t)."""
    from paper_1411_2377_b200 import CSR, MPVec
    L = p // 32
    D = CSR.dense(p, 0, np.zeros((0, L), np.uint32), np.zeros(0, np.int32), np.zeros(0, np.uint8))
    x = MPVec.from_host(np.zeros((0, L), np.uint32), np.zeros(0, np.int32), np.zeros(0, np.uint8),
                        device="cuda:0")
    y = D.spmv(x).to_host()
    assert y[0].size == 0
    D.close()
    d = LK.make(1, 0, p)
    D = CSR.dense(p, 1, d["dense_limbs"], d["dense_exps"], d["dense_signs"])
    x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda:0")
    want = oracle.dense_mv(p, 1, d["dense_limbs"], d["dense_exps"], d["dense_signs"],
                           d["x_limbs"], d["x_exps"], d["x_signs"])
    assert_same(D.spmv(x).to_host(), want, "n=1")
    D.close()
