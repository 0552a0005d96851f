#!/usr/bin/env python
"""Diagnostics: SpMV kernel time of a config generated at several sizes n
(same structure), to tell a latency-bound kernel (flat in n) from a
throughput-bound one (linear in n).   python tools/scale_n.py C2 25000 50000 ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import gen  # noqa: E402
from paper_1411_2377_b200 import CSR, MPVec  # noqa: E402

cfg = sys.argv[1]
p = None
for n in [int(v) for v in sys.argv[2:]]:
    d = gen.make(cfg, seed=0, n=n)
    A = CSR(d["p"], d["rowptr"], d["colidx"], d["limbs"], d["exps"], d["signs"])
    x = MPVec.from_host(d["x_limbs"], d["x_exps"], d["x_signs"], device="cuda")
    y = MPVec.empty(d["n"], d["p"] // 32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(13):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A.spmv(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    ts.sort()
    nnz = int(d["rowptr"][-1])
    print(f"{cfg} n={n} nnz={nnz} p={d['p']} ms_med={ts[len(ts)//2]:.4f} ns_per_nnz={ts[len(ts)//2]*1e6/nnz:.3f}")
    A.close()
