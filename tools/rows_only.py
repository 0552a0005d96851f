#!/usr/bin/env python
"""Run A x on a config with only the rows whose length is in [lo, hi] kept
(the others emptied) - a small command for ncu on one row class.
    python tools/rows_only.py C4 5000 5000 [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import gen  # noqa: E402
from paper_1411_2377_b200 import CSR, MPVec  # noqa: E402

cfg, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
d = gen.make(cfg, seed=0)
rp, ci = d["rowptr"], d["colidx"]
lens = np.diff(rp)
keep = (lens >= lo) & (lens <= hi)
kk = np.repeat(keep, lens)
nl = np.where(keep, lens, 0)
rp2 = np.zeros_like(rp)
np.cumsum(nl, out=rp2[1:])
A = CSR(d["p"], rp2, ci[kk], d["limbs"][kk], d["exps"][kk], d["signs"][kk])
x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda")
y = MPVec.empty(d["n"], d["p"] // 32, device="cuda")
for _ in range(reps):
    A.spmv(x, out=y)
torch.cuda.synchronize()
print("ok", int(keep.sum()), "rows", int(nl.sum()), "nnz")
A.close()
