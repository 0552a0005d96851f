import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
import gen
from paper_1411_2377_b200 import MPVec
from paper_1411_2377_b200.csr import dot
n, p = 84617, 256
rng = np.random.default_rng(5)
l1, e1, s1 = gen.configs.rand_values(rng, n, 8, -4, 4)
l2, e2, s2 = gen.configs.rand_values(rng, n, 8, -4, 4)
u = MPVec.from_host(l1, e1, s1, device="cuda:0"); v = MPVec.from_host(l2, e2, s2, device="cuda:0")
for _ in range(3):
    dot(p, u, v)
torch.cuda.synchronize()
