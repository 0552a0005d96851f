#!/usr/bin/env python
"""Diagnostics: time the SpMV over row-length classes of a config separately
(rows kept by length range, the others emptied) to see which class bounds
the kernel time.   python tools/c4_parts.py [C4] [ranges...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import gen  # noqa: E402
from paper_1411_2377_b200 import CSR, MPVec  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
ranges = [tuple(int(v) for v in r.split("-")) for r in sys.argv[2:]] or \
    [(1, 32), (33, 128), (129, 999), (1000, 4999), (5000, 5000), (1, 5000)]
d = gen.make(cfg, seed=0)
rp, ci = d["rowptr"], d["colidx"]
lens = np.diff(rp)
x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda")
for lo, hi in ranges:
    keep = (lens >= lo) & (lens <= hi)
    kk = np.repeat(keep, lens)
    nl = np.where(keep, lens, 0)
    rp2 = np.zeros_like(rp)
    np.cumsum(nl, out=rp2[1:])
    A = CSR(d["p"], rp2, ci[kk], d["limbs"][kk], d["exps"][kk], d["signs"][kk])
    y = MPVec.empty(d["n"], d["p"] // 32, device="cuda")
    for _ in range(3):
        A.spmv(x, out=y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        A.spmv(x, out=y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    nnz = int(nl.sum())
    print(f"rows {lo}-{hi}: {int(keep.sum())} rows {nnz} nnz  {ms:.4f} ms  "
          f"{nnz / ms / 1e6:.3f} G-nnz/s", flush=True)
    A.close()
