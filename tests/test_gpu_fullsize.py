"""Full-size parity (BASELINE.json configs C1..C5 at their real sizes, in the
launch configuration bench.py times): the WHOLE result vector of every
config and operation is computed on the GPU and by the oracle on all host
cores (oracle/run_parallel.py: the serial oracle's row chains, unchanged,
over nnz-balanced row chunks; A^T through oracle.transpose_np), and compared
limb by limb, exponent and sign (BASELINE.json north_star: "bit-exact
agreement with the oracle on every config for both A x and A^T x";
PAPER.md:182-186 the product A^(s,p) b, PAPER.md:282-284 z = A p, z~ = A^T p~).
Plus an any-size property: repeated applications agree bitwise (C3's
"A x repeated 50 times", reading c20)."""
import numpy as np
import pytest

import gen
from gpu_util import assert_same, oracle_args
from oracle import run_parallel

pytestmark = pytest.mark.gpu

OPS = {"C1": ["ax", "atx"], "C2": ["ax", "atx"], "C3": ["ax"], "C4": ["ax", "atx"], "C5": ["ax"]}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    import __graft_entry__
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    __graft_entry__.build()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4", "C5"])
def test_fullsize_whole_vector(cfg):
    import torch
    from paper_1411_2377_b200 import CSR, MPVec
    d = gen.make(cfg, seed=0)
    ops = OPS[cfg]
    A = CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"],
            transpose=("atx" in ops))
    x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda:0")
    reps = 50 if cfg == "C3" else 2
    for op in ops:
        f = A.spmv if op == "ax" else A.spmv_t
        y1 = f(x)
        y2 = MPVec.empty(d["n"], d["p"] // 32, device="cuda:0")
        for _ in range(reps - 1):
            f(x, out=y2)
        torch.cuda.synchronize()
        g1 = y1.to_host()
        assert_same(y2.to_host(), g1, f"{cfg} {op} repeat")
        if op == "ax":
            want, _, _ = run_parallel.spmv_parallel(*oracle_args(d))
        else:
            want, _, _, _ = run_parallel.spmv_t_parallel(*oracle_args(d))
        assert_same(g1, want, f"{cfg} {op} whole vector ({d['n']} rows)")
    A.close()
