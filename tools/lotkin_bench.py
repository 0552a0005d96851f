#!/usr/bin/env python
"""The paper's section-3 study on the GPU (Fig. 3; SPEC
spmv_bench S:421-427): dense MP MV vs sparse MP SpMV on the Lotkin matrix
with s% of its entries zeroed, "Speedup Ratio" = dense time / sparse time.
Both paths are verified bitwise equal before timing.  One JSON line per
(n, s, p).   python tools/lotkin_bench.py [n ...] [--p 128,512,1024] [--s 0,50,90,99]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
from gen import lotkin as LK  # noqa: E402
from paper_1411_2377_b200 import CSR, MPVec  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("n", type=int, nargs="*", default=[1000, 2000])
ap.add_argument("--p", default="128,512,1024")
ap.add_argument("--s", default="0,50,90,99")
ap.add_argument("--trials", type=int, default=10)
args = ap.parse_args()


def timed(A, x, y, trials):
    for _ in range(3):
        A.spmv(x, out=y)
    ts = []
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A.spmv(x, out=y)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


for n in args.n:
    for p in [int(v) for v in args.p.split(",")]:
        base = LK.lotkin(n, p)
        for s in [float(v) for v in args.s.split(",")]:
            dense, csr = LK.sparsify(n, base, s, seed=1)
            X = MPVec.from_host(*LK.xvec(n, p), device="cuda:0")
            D = CSR.dense(p, n, *dense)
            S = CSR(p, csr["rowptr"], csr["colidx"], csr["limbs"], csr["exps"], csr["signs"])
            yd = MPVec.empty(n, p // 32, device="cuda:0")
            ys = MPVec.empty(n, p // 32, device="cuda:0")
            D.spmv(X, out=yd)
            S.spmv(X, out=ys)
            a, b = yd.to_host(), ys.to_host()
            same = all(bool((u == v).all()) for u, v in zip(a, b))
            td, ts = timed(D, X, yd, args.trials), timed(S, X, ys, args.trials)
            print(json.dumps({"workload": f"Lotkin n={n} s={s}% p={p}", "nnz": int(len(csr["colidx"])),
                              "dense_ms": td, "sparse_ms": ts, "speedup_ratio": td / ts,
                              "bitwise_equal": same}), flush=True)
            D.close()
            S.close()
