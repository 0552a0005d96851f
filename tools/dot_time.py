#!/usr/bin/env python
"""Diagnostics: time the exact ordered-chain dot (mpsp_dot) on random-sign
(random walk) and positive vectors, and report the segment statistics.
    python tools/dot_time.py [n] [p]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import gen  # noqa: E402
from paper_1411_2377_b200 import MPVec  # noqa: E402
from paper_1411_2377_b200.csr import dot  # noqa: E402
from paper_1411_2377_b200._lib import dot_stats  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 84617
p = int(sys.argv[2]) if len(sys.argv) > 2 else 256
rng = np.random.default_rng(5)
L = p // 32
for kind in ("random-walk", "positive"):
    l1, e1, s1 = gen.configs.rand_values(rng, n, L, -4, 4)
    l2, e2, s2 = gen.configs.rand_values(rng, n, L, -4, 4)
    if kind == "positive":
        s1[:] = 0
        s2[:] = 0
    u = MPVec.from_host(l1, e1, s1, device="cuda:0")
    v = MPVec.from_host(l2, e2, s2, device="cuda:0")
    for _ in range(2):
        dot(p, u, v)
    torch.cuda.synchronize()
    dot_stats()
    ts = []
    for _ in range(5):
        e0, e1_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dot(p, u, v)
        e1_.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1_))
    st = dot_stats()
    print(f"{kind} n={n} p={p}: ms median {sorted(ts)[2]:.3f} (all {[round(t, 3) for t in ts]}) "
          f"segments/5 calls: {st}", flush=True)
