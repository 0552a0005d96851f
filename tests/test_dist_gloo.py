"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the row-block
partition and the x all-gather that precede every multi-GPU application
(paper_1411_2377_b200/dist.py; BASELINE.json north_star (4)).  The SpMV itself
needs a GPU; here the exchanged x must be bit-identical to the global x, the
row blocks must tile [0, n), and the exchange must work for ragged n."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1411_2377_b200.csr import MPVec
from paper_1411_2377_b200.dist import allgather_x, block_range, block_size


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, L, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(seed)
        xl = rng.integers(0, 2 ** 32, size=(n, L), dtype=np.uint32)
        xe = rng.integers(-100, 100, size=n).astype(np.int32)
        xs = rng.integers(0, 2, size=n).astype(np.uint8)
        rb, re = block_range(n, world, rank)
        xloc = MPVec(torch.from_numpy(xl[rb:re].view(np.int32).copy()),
                     torch.from_numpy(xe[rb:re].copy()), torch.from_numpy(xs[rb:re].copy()))
        full = allgather_x(xloc, n)
        gl = full.limbs.numpy().view(np.uint32)[:n]
        ok = (np.array_equal(gl, xl) and np.array_equal(full.exps.numpy()[:n], xe)
              and np.array_equal(full.signs.numpy()[:n], xs)
              and full.limbs.shape[0] == world * block_size(n, world))
        q.put((rank, ok, rb, re))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,L", [(2, 1001, 4), (3, 10, 8), (2, 2, 1), (3, 7, 32)])
def test_allgather_x_gloo(world, n, L):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, L, 7, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _, _ in res)
    # row blocks tile [0, n) in rank order
    bounds = [(rb, re) for _, _, rb, re in res]
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    for (a, b), (c, d) in zip(bounds, bounds[1:]):
        assert b == c


def test_block_range_properties():
    for n in (0, 1, 7, 100, 4_000_000):
        for G in (1, 2, 3, 4, 8):
            blocks = [block_range(n, G, r) for r in range(G)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(b[0] <= b[1] for b in blocks)
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(G - 1))
            assert max(b[1] - b[0] for b in blocks) == (block_size(n, G) if n else 0)
