"""The section-3 workload and the dense MP MV (
PAPER.md:170-209; SPEC gen_lotkin / sparsify / dense_mv): the
Lotkin generator pinned against exact rationals, SplitMix64 against its
published seed-0 outputs, the sparsifier's counts and determinism, and the
oracle's dense_mv against closed forms and the bitwise dense == sparse
equivalence."""
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle
from gen import lotkin as LK


@pytest.mark.parametrize("p", [32, 64, 128])
def test_recip_is_correctly_rounded(p):
    """RN_p(1/k): normalised, within half an ulp of 1/k (exact rationals)."""
    for k in list(range(1, 400)) + [1 << 20, (1 << 20) + 1, 3 ** 15, 10 ** 9 + 7]:
        s, M, E = LK.recip(k, p)
        assert s == 0 and (1 << (p - 1)) <= M < (1 << p)
        v = Fraction(M, 1 << p) * Fraction(2) ** E
        ulp = Fraction(2) ** (E - p)
        assert abs(v - Fraction(1, k)) <= ulp / 2
        # and 1/k lies in v's binade [2^(E-1), 2^E) unless it rounded up to it
        assert Fraction(1, k) < Fraction(2) ** E


def test_lotkin_structure():
    n, p = 9, 64
    l, e, s = LK.lotkin(n, p)
    vals = oracle.unpack_vec(l, e, s, p)
    one = (0, 1 << (p - 1), 1)
    for j in range(n):
        assert vals[j] == one                              # row 1 all ones
    for i in range(1, n):
        for j in range(n):
            assert vals[i * n + j] == LK.recip(i + j + 1, p)   # 1/(i+j-1), 1-based
            if j >= 1:
                assert vals[i * n + j] == vals[j * n + i]       # symmetric trailing block
    # spot values against Fraction: a_22 = 1/3, a_33 = 1/5 (1-based)
    for (i, j, k) in ((1, 1, 3), (2, 2, 5), (8, 8, 17)):
        sg, M, E = vals[i * n + j]
        assert abs(Fraction(M, 1 << p) * Fraction(2) ** E - Fraction(1, k)) <= Fraction(2) ** (E - p - 1)


def test_splitmix64_published_outputs():
    """SplitMix64 from seed 0: the widely published first outputs."""
    g = LK.splitmix64(0)
    assert [next(g) for _ in range(3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                           0x06C45D188009454F]


@pytest.mark.parametrize("n,s", [(10, 0), (10, 50), (37, 90), (100, 99), (20, 99.9)])
def test_sparsify_counts_and_determinism(n, s):
    dense = LK.lotkin(n, 64)
    (dl, de, ds), csr = LK.sparsify(n, dense, s, seed=5)
    k = int(round(s / 100 * n * n))
    zeros = int(np.sum(~np.any(dl != 0, axis=1)))
    assert zeros == k and len(csr["colidx"]) == n * n - k
    (dl2, _, _), csr2 = LK.sparsify(n, dense, s, seed=5)
    assert np.array_equal(dl, dl2) and np.array_equal(csr["colidx"], csr2["colidx"])
    (dl3, _, _), _ = LK.sparsify(n, dense, s, seed=6)
    if 0 < k < n * n:
        assert not np.array_equal(dl, dl3)


def test_dense_mv_closed_forms():
    """Row 1 of Lotkin times [1..n] is n(n+1)/2 exactly; A e_j is column j."""
    n, p = 12, 128
    d = LK.make(n, 0, p)
    y = oracle.unpack_vec(*oracle.dense_mv(p, n, d["dense_limbs"], d["dense_exps"], d["dense_signs"],
                                           d["x_limbs"], d["x_exps"], d["x_signs"]), p)
    t = n * (n + 1) // 2
    assert y[0] == (0, t << (p - t.bit_length()), t.bit_length())
    L = p // 32
    for j in (0, 5, n - 1):
        ej = [oracle.ZERO] * n
        ej[j] = (0, 1 << (p - 1), 1)
        xl, xe, xs = oracle.pack_vec(ej, p)
        col = oracle.unpack_vec(*oracle.dense_mv(p, n, d["dense_limbs"], d["dense_exps"],
                                                 d["dense_signs"], xl, xe, xs), p)
        A = oracle.unpack_vec(d["dense_limbs"], d["dense_exps"], d["dense_signs"], p)
        assert col == [A[i * n + j] for i in range(n)]
        assert L == d["dense_limbs"].shape[1]


def test_dense_equals_sparse_bitwise():
    """SPEC's primary kernel equivalence, on the oracle: dense_mv of the
    sparsified Lotkin matrix == spmv of its CSR (and the transposes)."""
    rng = random.Random(7)
    for trial in range(12):
        n = rng.choice([1, 5, 23, 40])
        s = rng.choice([0, 50, 90, 99])
        p = rng.choice([32, 128, 512])
        d = LK.make(n, s, p, seed=trial)
        xa = (d["x_limbs"], d["x_exps"], d["x_signs"])
        dn = oracle.dense_mv(p, n, d["dense_limbs"], d["dense_exps"], d["dense_signs"], *xa)
        sp = oracle.spmv(p, d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"], *xa)
        for a, b in zip(dn, sp):
            assert np.array_equal(a, b), (trial, n, s, p)
        dt = oracle.dense_mv(p, n, d["dense_limbs"], d["dense_exps"], d["dense_signs"], *xa,
                             transpose=True)
        st = oracle.spmv_t(p, d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"], *xa)
        for a, b in zip(dt, st):
            assert np.array_equal(a, b), ("t", trial, n, s, p)
