#!/usr/bin/env python
"""Debug: GPU dot vs oracle chain on random walks (binade crossings) per p."""
import os
import random
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import __graft_entry__  # noqa: E402

__graft_entry__.build()
import oracle  # noqa: E402
from oracle import krylov as K  # noqa: E402
import test_gpu_krylov as TG  # noqa: E402
from paper_1411_2377_b200.csr import dot  # noqa: E402

for p in (64, 128, 256, 512, 1024):
    rng = random.Random(p)
    bad = 0
    for trial in range(30):
        n = rng.choice([20, 100, 300, 1000])
        u = [(rng.getrandbits(1), (1 << (p - 1)) | rng.getrandbits(p - 1), rng.randint(-3, 3))
             for _ in range(n)]
        one = [K.from_int(1, p)] * n
        r = dot(p, TG._vec(u, p), TG._vec(one, p))
        torch.cuda.synchronize()
        g = r.to_host()
        w = oracle.pack_vec([K.dot(u, one, p)], p)
        if not all(np.array_equal(a, b) for a, b in zip(g, w)):
            bad += 1
    print("p", p, "bad", bad, "of 30", flush=True)
