"""Generator tests (CPU): closed-form nnz, CSR invariants, encodings, seeds."""
import numpy as np
import pytest

import gen
from gen import configs as C


def check_csr(d):
    rp, ci, n = d["rowptr"], d["colidx"], d["n"]
    assert rp[0] == 0 and np.all(np.diff(rp) >= 0) and rp[-1] == len(ci)
    assert ci.dtype == np.int32 and rp.dtype == np.int64
    if len(ci):
        assert ci.min() >= 0 and ci.max() < n
    rows = np.repeat(np.arange(n), np.diff(rp))
    same = rows[1:] == rows[:-1]
    assert np.all(ci[1:][same] > ci[:-1][same]), "strictly increasing columns per row"


def check_values(limbs, exps, signs):
    nz = np.any(limbs != 0, axis=1)
    assert np.all(limbs[nz, -1] >> 31 == 1), "nonzero values are normalised"
    assert np.all(np.abs(exps.astype(np.int64)) <= 2 ** 29)
    assert set(np.unique(signs)) <= {0, 1}


def test_closed_form_nnz():
    assert C.make("C1")["meta"]["nnz"] == 16_000                     # 8 per row
    assert C.pattern_band(100_000, 5)[0][-1] == 1_099_970           # 11n - 30
    rp, ci, dg = C.pattern_stencil5(2000)
    assert rp[-1] == 19_992_000                                     # 5 g^2 - 4 g
    assert dg.sum() == 4_000_000


@pytest.mark.parametrize("cfg,n", [("C1", None), ("C2", 3000), ("C3", 5000), ("C4", 20000), ("C5", 4900)])
def test_config_shapes(cfg, n):
    d = C.make(cfg, n=n)
    check_csr(d)
    check_values(d["limbs"], d["exps"], d["signs"])
    check_values(d["x_limbs"], d["x_exps"], d["x_signs"])
    L = d["p"] // 32
    assert d["limbs"].shape == (len(d["colidx"]), L)
    if cfg == "C1":
        assert (~np.any(d["x_limbs"] != 0, axis=1)).sum() == 100           # exactly 5 %
        rows = np.repeat(np.arange(d["n"]), 8)
        assert np.all(np.any(d["colidx"].reshape(-1, 8) == np.arange(d["n"])[:, None], axis=1))
    if cfg == "C3":
        rows = np.repeat(np.arange(d["n"]), np.diff(d["rowptr"]))
        assert np.all(np.bincount(rows[d["colidx"] == rows], minlength=d["n"]) == 1)  # diagonal
        assert abs(len(d["colidx"]) / d["n"] - 12.0) < 0.3
    if cfg == "C4":
        assert np.diff(d["rowptr"]).max() == 5000
        assert np.diff(d["rowptr"]).min() >= 1


def test_c5_values_encode_minus_one_plus_delta():
    d = C.make("C5", n=900)
    p, L = d["p"], d["p"] // 32
    rows = np.repeat(np.arange(d["n"]), np.diff(d["rowptr"]))
    diag = d["colidx"] == rows
    from fractions import Fraction
    for k in range(len(d["colidx"])):
        M = int.from_bytes(d["limbs"][k].tobytes(), "little")
        v = Fraction(M, 2 ** p) * Fraction(2) ** int(d["exps"][k]) * (-1 if d["signs"][k] else 1)
        if diag[k]:
            assert v == 4
        else:
            delta = v + 1
            assert abs(delta) <= Fraction(1, 2 ** 20)
            kk = delta * 2 ** (p - 1)
            assert kk.denominator == 1            # delta = k 2^(1-p), k integer


def test_determinism_and_seed_sensitivity():
    a = C.make("C4", n=5000, seed=3)
    b = C.make("C4", n=5000, seed=3)
    c = C.make("C4", n=5000, seed=4)
    assert C.sha256_arrays(a) == C.sha256_arrays(b) != C.sha256_arrays(c)


@pytest.mark.parametrize("p", [32, 64, 128, 256, 512, 1024])
def test_stress_corpus_valid(p):
    d = gen.stress(p, long_len=600, n_random_rows=30)
    check_csr(d)
    nz = np.any(d["limbs"] != 0, axis=1)
    assert np.all(d["limbs"][nz, -1] >> 31 == 1)
    assert (~nz).sum() > 0                       # explicit zeros present
    assert np.diff(d["rowptr"]).max() == 600
