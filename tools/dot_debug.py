#!/usr/bin/env python
"""Debug: first prefix length where the GPU dot differs from the oracle chain
for the failing segmented-dot test case, and the model's transition stats."""
import os
import sys
import zlib

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import oracle  # noqa: E402
from oracle import krylov as K  # noqa: E402
import test_gpu_krylov as TG  # noqa: E402
import test_kernel_algorithms as TA  # noqa: E402
from paper_1411_2377_b200.csr import dot  # noqa: E402

kind, p, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(zlib.crc32(f"{kind}-{p}-{n}".encode()))
u, v = TG._dot_case(kind, n, p, rng)


def gpu(m):
    r = dot(p, TG._vec(u[:m], p), TG._vec(v[:m], p))
    torch.cuda.synchronize()
    return r.to_host()


def ok(m):
    g = gpu(m)
    w = oracle.pack_vec([K.dot(u[:m], v[:m], p)], p)
    return all(np.array_equal(a, b) for a, b in zip(g, w))


print("full ok:", ok(n))
lo, hi = 1, n
while lo < hi:
    m = (lo + hi) // 2
    if ok(m):
        lo = m + 1
    else:
        hi = m
print("first failing prefix", lo)
ts = [oracle.mul(a, b, p) for a, b in zip(u[:lo], v[:lo])]
st = {}
got, _ = TA.block_sum_chain(ts, p, transitions=True, stats=st)
print("model ok:", got == TA.oracle_chain(ts, p), st)
st2 = {}
TA.block_sum_chain(ts[:-1], p, transitions=True, stats=st2)
print("model stats without the last step", st2)
print("last product", ts[-1], "chain before", TA.oracle_chain(ts[:-1], p))
