"""Full-size parity (BASELINE.json configs C1..C5 at their real sizes, in the
launch configuration bench.py times): the whole result is computed on the
GPU, and sampled rows (random + first/last + the longest rows, i.e. the
5000-long chains of C4) are recomputed one by one by the oracle and compared
bit-exactly.  Plus an any-size property: two applications agree bitwise."""
import numpy as np
import pytest

import gen
from gpu_util import assert_same, oracle_rows

pytestmark = pytest.mark.gpu

OPS = {"C1": ["ax", "atx"], "C2": ["ax", "atx"], "C3": ["ax"], "C4": ["ax", "atx"], "C5": ["ax"]}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    import __graft_entry__
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    __graft_entry__.build()


def sample_rows(d, op, k=400, seed=0):
    n = d["n"]
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(n, size=min(k, n), replace=False).tolist())
    rows |= {0, 1, n - 2, n - 1}
    if op == "ax":
        lens = np.diff(d["rowptr"])
        rows |= set(np.argsort(-lens, kind="stable")[:6].tolist())     # longest chains
    return sorted(rows)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_fullsize_sampled(cfg):
    import torch
    from paper_1411_2377_b200 import CSR, MPVec
    d = gen.make(cfg, seed=0)
    ops = OPS[cfg]
    A = CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
            transpose=("atx" in ops))
    x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda:0")
    for op in ops:
        f = A.spmv if op == "ax" else A.spmv_t
        y1 = f(x)
        y2 = f(x)
        torch.cuda.synchronize()
        g1 = y1.to_host()
        g2 = y2.to_host()
        assert_same(g2, g1, f"{cfg} {op} repeat")
        rows = sample_rows(d, op, k=300 if cfg == "C4" else 400)
        want = oracle_rows(d, op, rows)
        got = tuple(a[rows] for a in g1)
        assert_same(got, want, f"{cfg} {op} sampled rows")
    A.close()
