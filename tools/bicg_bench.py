#!/usr/bin/env python
"""Time BiCG (mpsp_bicg) on a synthetic diagonally dominant system shaped like
C2 (band +-5, off-diagonal exponents U[-8, 0], diagonal exponent 4; SURVEY.md
8(f)), b = A [1..n]^T computed by the library's SpMV, and the pieces of one
iteration (dot, SpMV, A^T SpMV, axpy) with CUDA events.
    python tools/bicg_bench.py [n] [p] [iters]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import gen  # noqa: E402
from paper_1411_2377_b200 import CSR, MPVec  # noqa: E402
from paper_1411_2377_b200.csr import axpy, dot  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 256
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
L = p // 32
rng = np.random.default_rng(2)
rowptr, colidx = gen.configs.pattern_band(n, 5)
limbs, exps, signs = gen.configs.rand_values(rng, len(colidx), L, -8, 0)
rows = np.repeat(np.arange(n), np.diff(rowptr))
exps[colidx == rows] = 4
A = CSR(p, rowptr, colidx, limbs, exps, signs, transpose=True)
# b = A [1..n]: integers i+1 encoded exactly (MSB-normalised)
xi = np.arange(1, n + 1, dtype=np.uint64)
bl = np.zeros((n, L), np.uint32)
bits = np.floor(np.log2(xi)).astype(np.int64) + 1
top = (xi << (32 - bits).astype(np.uint64)).astype(np.uint32)
bl[:, L - 1] = top
xt = MPVec.from_host(bl, bits.astype(np.int32), np.zeros(n, np.uint8), device="cuda")
b = A.spmv(xt)
torch.cuda.synchronize()


def timed(f, reps=3):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


t_dot = timed(lambda: dot(p, b, b))
t_spmv = timed(lambda: A.spmv(b))
t_spmvt = timed(lambda: A.spmv_t(b))
al = dot(p, b, b)
t_axpy = timed(lambda: axpy(p, al, b, b))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
x, it, status = A.bicg(b, iters)
e1.record()
torch.cuda.synchronize()
t_total = e0.elapsed_time(e1)
import ctypes  # noqa: E402
from paper_1411_2377_b200 import _lib  # noqa: E402
st = (ctypes.c_ulonglong * 2)()
_lib.lib().mpsp_debug_dot_stats(st)
print("dot segments over the run: sequential", st[0], "validated", st[1])
A.gpbicg(b, 2)                              # warm-up (kernel loading, clocks)
torch.cuda.synchronize()
e0.record()
xg, itg, statusg = A.gpbicg(b, iters)
e1.record()
torch.cuda.synchronize()
t_gp = e0.elapsed_time(e1)
print(json.dumps({"workload": f"GPBiCG band+-5 n={n} p={p}", "iters": itg, "status": statusg,
                  "ms_total": t_gp, "ms_per_iter": t_gp / max(itg, 1)}))
print(json.dumps({"workload": f"BiCG band+-5 n={n} p={p}", "iters": it, "status": status,
                  "ms_total": t_total, "ms_per_iter": t_total / max(it, 1),
                  "ms_dot": t_dot, "ms_spmv": t_spmv, "ms_spmv_t": t_spmvt, "ms_axpy": t_axpy,
                  "per_iter_model_ms": 3 * t_dot + t_spmv + t_spmvt + 5 * t_axpy}))
