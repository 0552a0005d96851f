#!/usr/bin/env python
"""Randomised parity sweep (GPU vs oracle, bit-exact) over precisions
32 ... 8192, row-length mixes, value mixes (random, powers of two, all-ones
runs, tie-prone, wide exponent spreads, zeros, cancellation pairs), A x /
A^T x, sparse / dense handles, and the dot product.  Reports the first
mismatch with its seed.   python tools/fuzz.py [seconds] [first_seed]"""
import os
import random
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import oracle  # noqa: E402
from oracle import krylov as K  # noqa: E402
from paper_1411_2377_b200 import CSR, MPVec  # noqa: E402
from paper_1411_2377_b200.csr import dot  # noqa: E402

PS = [int(v) for v in os.environ.get("FUZZ_P", "32,64,128,256,512,1024,2048,4096,8192").split(",")]


def value(R, p, e0):
    top = 1 << (p - 1)
    k = R.random()
    if k < 0.08:
        return (0, 0, 0)
    s = R.getrandbits(1)
    if k < 0.2:
        M = top
    elif k < 0.3:
        M = (1 << p) - 1
    elif k < 0.4:
        M = top | ((1 << R.randrange(1, p)) - 1)
    elif k < 0.5:
        M = top | (1 << R.randrange(0, p - 1))
    else:
        M = top | R.getrandbits(p - 1)
    return (s, M, e0 + R.randint(-R.choice([2, 8, 40, 200]), R.choice([2, 8, 40, 200])))


def case(seed):
    R = random.Random(seed)
    p = R.choice(PS)
    n = R.choice([1, 2, 7, 33, 100, 250])
    e0 = R.randint(-50, 50)
    rows, cols, vals = [], [], []
    for i in range(n):
        ln = R.choice([0, 1, 3, 8, 20, 40, 100, 300]) if R.random() < 0.9 else R.choice([600, 1000])
        ln = min(ln, n)
        cs = sorted(R.sample(range(n), ln))
        for j in cs:
            rows.append(i)
            cols.append(j)
            v = value(R, p, e0)
            if R.random() < 0.05 and vals:                 # cancellation partner
                s_, M_, E_ = vals[-1]
                v = (s_ ^ 1, M_, E_)
            vals.append(v)
    rowptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(np.array(rows, np.int64), minlength=n), out=rowptr[1:])
    colidx = np.array(cols, np.int32)
    limbs, exps, signs = oracle.pack_vec(vals, p)
    xv = [value(R, p, R.randint(-20, 20)) for _ in range(n)]
    xl, xe, xs = oracle.pack_vec(xv, p)
    return R, p, n, rowptr, colidx, limbs, exps, signs, xl, xe, xs


def same(a, b):
    return all(np.array_equal(np.asarray(u).reshape(np.asarray(v).shape), v) for u, v in zip(a, b))


def run(seed):
    R, p, n, rowptr, colidx, limbs, exps, signs, xl, xe, xs = case(seed)
    x = MPVec.from_host(xl, xe, xs, device="cuda:0")
    op = R.choice(["ax", "atx"])
    args = (p, rowptr, colidx, limbs, exps, signs, xl, xe, xs)
    want = oracle.spmv(*args) if op == "ax" else oracle.spmv_t(*args)
    A = CSR(p, rowptr, colidx, limbs, exps, signs, transpose=(op == "atx"))
    got = (A.spmv(x) if op == "ax" else A.spmv_t(x)).to_host()
    A.close()
    if not same(got, want):
        return f"spmv {op} p={p} n={n}"
    if R.random() < 0.3:                                # host-buffer entry point
        A = CSR(p, rowptr, colidx, limbs, exps, signs, transpose=(op == "atx"))
        got = (A.spmv_host if op == "ax" else A.spmv_t_host)(xl, xe, xs)
        A.close()
        if not same(got, want):
            return f"spmv_host {op} p={p} n={n}"
    if R.random() < 0.3 and n <= 120:                   # dense handle of the same matrix
        L = p // 32
        dl = np.zeros((n * n, L), np.uint32)
        de = np.zeros(n * n, np.int32)
        ds = np.zeros(n * n, np.uint8)
        rr = np.repeat(np.arange(n), np.diff(rowptr))
        dl[rr * n + colidx] = limbs
        de[rr * n + colidx] = exps
        ds[rr * n + colidx] = signs
        D = CSR.dense(p, n, dl, de, ds, transpose=(op == "atx"))
        got = (D.spmv(x) if op == "ax" else D.spmv_t(x)).to_host()
        D.close()
        if not same(got, want):
            return f"dense {op} p={p} n={n}"
    if R.random() < 0.3:
        m = R.choice([5, 300, 3000])
        u = [value(R, p, 0) for _ in range(m)]
        v = [value(R, p, 0) for _ in range(m)]
        g = dot(p, MPVec.from_host(*oracle.pack_vec(u, p), device="cuda:0"),
                MPVec.from_host(*oracle.pack_vec(v, p), device="cuda:0"))
        if not same(g.to_host(), oracle.pack_vec([K.dot(u, v, p)], p)):
            return f"dot p={p} m={m}"
    if R.random() < 0.1 and p >= 128:                  # a few solver iterations
        m = R.choice([5, 12, 30])
        sets = [sorted({i, (i + 1) % m, (i + R.randrange(1, m)) % m}) for i in range(m)]
        rp = np.zeros(m + 1, np.int64)
        np.cumsum([len(c) for c in sets], out=rp[1:])
        ci = [j for c in sets for j in c]
        vl = [(0, 1 << (p - 1), 5) if j == i else value(R, p, 0)     # dominant diagonal 16
              for i, c in enumerate(sets) for j in c]
        A = (rp, np.array(ci, np.int32), *oracle.pack_vec(vl, p))
        b = [value(R, p, 0) for _ in range(m)]
        solver = R.choice(["bicg", "gpbicg"])
        it = R.choice([1, 3, 5])
        want = (K.bicg if solver == "bicg" else K.gpbicg)(p, A, b, it)
        H = CSR(p, *A, transpose=(solver == "bicg"))
        bv = MPVec.from_host(*oracle.pack_vec(b, p), device="cuda:0")
        xg, itg, st = (H.bicg if solver == "bicg" else H.gpbicg)(bv, it)
        torch.cuda.synchronize()
        H.close()
        if (itg, st) != (want["iters"], want["status"]) or \
                not same(xg.to_host(), oracle.pack_vec(want["x"], p)):
            return f"{solver} p={p} m={m} it={it}"
    return None


seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 60
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t0 = time.time()
done = 0
while time.time() - t0 < seconds:
    bad = run(seed)
    if bad:
        print(f"MISMATCH seed={seed}: {bad}", flush=True)
        sys.exit(1)
    seed += 1
    done += 1
print(f"fuzz ok: {done} cases (seeds up to {seed - 1})", flush=True)
