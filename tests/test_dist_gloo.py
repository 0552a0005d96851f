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


def _window_worker(rank, world, port, kind, n, L, transpose, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        from paper_1411_2377_b200.dist import WindowExchange, needed_window
        if kind == "stencil":
            g = int(round(n ** 0.5))
            rowptr, colidx, _ = gen.configs.pattern_stencil5(g)
            n = g * g
        elif kind == "band":
            rowptr, colidx = gen.configs.pattern_band(n, 5)
        else:
            rng = np.random.default_rng(3)
            rowptr, colidx = gen.configs.pattern_random_rows(rng, n, rng.integers(0, 6, size=n))
        rng = np.random.default_rng(11)
        xl = rng.integers(0, 2 ** 32, size=(n, L), dtype=np.uint32)
        xe = rng.integers(-100, 100, size=n).astype(np.int32)
        xs = rng.integers(0, 2, size=n).astype(np.uint8)
        rb, re = block_range(n, world, rank)
        lo, hi = needed_window(rowptr, colidx, rb, re, transpose=transpose)
        # the window really covers every x index the rows read
        if transpose:
            k = np.flatnonzero((colidx >= rb) & (colidx < re))
            idx = np.searchsorted(rowptr, k, side="right") - 1
        else:
            idx = colidx[rowptr[rb]:rowptr[re]]
        covered = bool(len(idx) == 0 or (idx.min() >= lo and idx.max() < hi))
        X = WindowExchange(n, L, (lo, hi))
        xloc = MPVec(torch.from_numpy(xl[rb:re].view(np.int32).copy()),
                     torch.from_numpy(xe[rb:re].copy()), torch.from_numpy(xs[rb:re].copy()))
        full = X.exchange(xloc)
        gl = full.limbs.numpy().view(np.uint32)
        ok = (np.array_equal(gl[lo:hi], xl[lo:hi]) and np.array_equal(full.exps.numpy()[lo:hi], xe[lo:hi])
              and np.array_equal(full.signs.numpy()[lo:hi], xs[lo:hi]))
        # second exchange through the local view (no copy) gives the same
        v = X.local_view()
        v.limbs.copy_(xloc.limbs); v.exps.copy_(xloc.exps); v.signs.copy_(xloc.signs)
        full2 = X.exchange(v)
        ok = ok and np.array_equal(full2.limbs.numpy().view(np.uint32)[lo:hi], xl[lo:hi])
        q.put((rank, ok and covered, X.bytes_in, hi - lo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,n,L,transpose", [
    (2, "stencil", 400, 4, False), (3, "stencil", 900, 8, False), (2, "band", 1001, 2, False),
    (3, "band", 100, 1, True), (2, "random", 300, 4, False), (3, "random", 200, 2, True),
    (4, "stencil", 64, 32, False)])
def test_window_exchange_gloo(world, kind, n, L, transpose):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_window_worker, args=(r, world, port, kind, n, L, transpose, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res)
    if kind == "stencil":
        g = int(round(n ** 0.5))
        # halo only: each rank receives at most two grid lines per neighbour
        assert all(b <= 2 * g * (4 * L + 5) for _, _, b, _ in res)
