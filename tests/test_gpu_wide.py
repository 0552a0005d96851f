"""GPU parity at p > 1024 (the paper's solver
precisions 2048-8192 bits): spmv_wide, one warp
per row with every MP value spread across the lanes, vs the CPU oracle,
bit-exact, for A x and A^T x - the stress corpus (ties, cancellation to +0,
carries through all-ones mantissas, zeros with junk fields, far-path
exponent gaps, huge/tiny exponents, empty and long rows) and config-shaped
random / stencil matrices."""
import numpy as np
import pytest

import gen
from gpu_util import assert_same, gpu_run, oracle_full

pytestmark = pytest.mark.gpu

PW = [2048, 4096, 8192]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    import __graft_entry__
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    __graft_entry__.build()


@pytest.mark.parametrize("op", ["ax", "atx"])
@pytest.mark.parametrize("p", PW)
def test_wide_stress_corpus(p, op):
    d = gen.stress(p, seed=0, long_len=700)
    assert_same(gpu_run(d, op), oracle_full(d, op), f"stress p={p} {op}")


@pytest.mark.parametrize("p", PW)
def test_wide_stress_other_seed(p):
    d = gen.stress(p, seed=1, long_len=300)
    for op in ("ax", "atx"):
        assert_same(gpu_run(d, op), oracle_full(d, op), f"stress seed1 p={p} {op}")


@pytest.mark.parametrize("cfg,n,p", [("C1", 600, 2048), ("C3", 400, 4096), ("C5", 400, 8192),
                                     ("C4", 800, 2048), ("C2", 300, 4096)])
def test_wide_config_shapes(cfg, n, p):
    d = gen.make(cfg, seed=3, n=n, p=p)
    for op in ("ax", "atx"):
        assert_same(gpu_run(d, op), oracle_full(d, op), f"{cfg} n={n} p={p} {op}")


def test_wide_row_block():
    """A row block at p = 2048 equals the same rows of the full result."""
    d = gen.stress(2048, seed=2, long_len=200)
    full = oracle_full(d, "ax")
    n = d["n"]
    rb, re = n // 3, n // 3 + 101
    got = gpu_run(d, "ax", rows=(rb, re))
    assert_same(got, tuple(a[rb:re] for a in full), "row block")


@pytest.mark.parametrize("p", [2048, 4096])
def test_wide_short_product_ambiguous_window(p):
    """The warp form's certificate window (bits 8 .. 30 - sh of the product's
    limb L-1: x's bits p-24 .. p-3 when a = 2^(p-1) + 1) all zeros / all
    ones with nonzero low limbs: every such product takes the full product."""
    import random
    rng = random.Random(p)
    n, per_row = 40, 4
    xs = []
    for i in range(n):
        M = (1 << (p - 1)) | rng.getrandbits(p - 1)
        win = ((1 << 22) - 1) << (p - 24)
        M = (M & ~win) | (win if i % 2 else 0) | 1
        xs.append((rng.getrandbits(1), M, rng.randint(-8, 8)))
    vals, cols, rowptr = [], [], [0]
    for r in range(n):
        for c in sorted(rng.sample(range(n), per_row)):
            Ma = (1 << (p - 1)) + 1 if rng.random() < 0.7 else (1 << (p - 1)) | rng.getrandbits(p - 1)
            vals.append((rng.getrandbits(1), Ma, rng.randint(-8, 8)))
            cols.append(c)
        rowptr.append(len(cols))
    al, ae, as_ = gen.pack_triples(vals, p)
    xl, xe, xsg = gen.pack_triples(xs, p)
    d = dict(p=p, n=n, rowptr=np.array(rowptr, np.int64), colidx=np.array(cols, np.int32),
             limbs=al, exps=ae, signs=as_, x_limbs=xl, x_exps=xe, x_signs=xsg)
    for op in ("ax", "atx"):
        assert_same(gpu_run(d, op), oracle_full(d, op), f"wide ambiguous window p={p} {op}")
