"""Multi-process (world_size 2-4, gloo, CPU) tests of the row-block partition
and the x exchange that precedes every multi-GPU application
(paper_1411_2377_b200/dist.py; BASELINE.json north_star (4)).
The SpMV itself needs a GPU; here the exchanged x must be bit-identical to
the global x wherever a rank's rows read it, for the all-gather and the
needed-window exchange of (L+1)-word records, the automatic choice between
them must agree on every rank, and the interior-row split (rows overlapped
with the exchange) must contain only rows that read the rank's own block.

On the CPU the record packing is done by TorchPacker below (test side); the
product path packs with the library kernels (mpsp_vec_pack / unpack, tested
on the GPU in test_gpu_abi.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
from paper_1411_2377_b200.csr import MPVec
from paper_1411_2377_b200.dist import (XExchange, block_range, block_size, choose_exchange,
                                       interior_mask, interior_run, needed_window)


class TorchPacker:
    """(L limbs, (sign << 31) | (exp & 0x7fffffff)) records with torch CPU ops."""

    def pack(self, v, rec, stream=None):
        L = v.limbs.shape[1]
        rec[:, :L] = v.limbs
        rec[:, L] = (v.exps & 0x7fffffff) | (v.signs.to(torch.int32) << 31)

    def unpack(self, rec, v, stream=None):
        L = v.limbs.shape[1]
        v.limbs.copy_(rec[:, :L])
        w = rec[:, L]
        v.exps.copy_((w << 1) >> 1)
        v.signs.copy_(((w >> 31) & 1).to(torch.uint8))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _pattern(kind, n):
    if kind == "stencil":
        g = int(round(n ** 0.5))
        rowptr, colidx, _ = gen.configs.pattern_stencil5(g)
    elif kind == "band":
        rowptr, colidx = gen.configs.pattern_band(n, 5)
    else:
        rng = np.random.default_rng(3)
        rowptr, colidx = gen.configs.pattern_random_rows(rng, n, rng.integers(0, 6, size=n))
    return rowptr, colidx


def _worker(rank, world, port, kind, n, L, transpose, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rowptr, colidx = _pattern(kind, n)
        n = len(rowptr) - 1
        rng = np.random.default_rng(11)
        xl = rng.integers(0, 2 ** 32, size=(n, L), dtype=np.uint32)
        xe = rng.integers(-(2 ** 29), 2 ** 29 + 1, size=n).astype(np.int32)
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
        X = XExchange(n, L, (lo, hi), mode=mode, packer=TorchPacker())
        X.set_local(xl[rb:re], xe[rb:re], xs[rb:re])
        full = X.exchange()
        a, b = (0, n) if X.mode == "allgather" else (lo, hi)
        gl = full.limbs.numpy().view(np.uint32)
        ok = (np.array_equal(gl[a:b], xl[a:b]) and np.array_equal(full.exps.numpy()[a:b], xe[a:b])
              and np.array_equal(full.signs.numpy()[a:b], xs[a:b]))
        # a second application with a new x block (as in BiCG) refreshes it
        xl2 = xl ^ np.uint32(0x5A5A5A5A)
        xl2[:, -1] |= np.uint32(0x80000000)
        X.set_local(xl2[rb:re], xe[rb:re], xs[rb:re])
        full2 = X.exchange()
        ok = ok and np.array_equal(full2.limbs.numpy().view(np.uint32)[a:b], xl2[a:b])
        # interior rows read only the own block
        m = interior_mask(rowptr, colidx, rb, re, transpose=transpose)
        ia, ib = interior_run(m)
        inner_ok = True
        for r in range(rb + ia, rb + ib):
            if transpose:
                kk = np.flatnonzero(colidx == r)
                rr = np.searchsorted(rowptr, kk, side="right") - 1
            else:
                rr = colidx[rowptr[r]:rowptr[r + 1]]
            inner_ok &= bool(np.all((rr >= rb) & (rr < re)))
        q.put((rank, ok and covered and inner_ok, X.bytes_in, X.mode, ib - ia, re - rb))
    finally:
        dist.destroy_process_group()


def _run(world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, *args, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res)


@pytest.mark.parametrize("world,kind,n,L,transpose,mode", [
    (2, "stencil", 400, 4, False, "auto"), (3, "stencil", 900, 8, False, "window"),
    (2, "band", 1001, 2, False, "auto"), (3, "band", 100, 1, True, "window"),
    (2, "random", 300, 4, False, "auto"), (3, "random", 200, 2, True, "window"),
    (4, "stencil", 64, 32, False, "allgather"), (3, "band", 10, 8, False, "allgather"),
    (2, "random", 7, 1, True, "allgather"), (4, "band", 3, 4, False, "auto")])
def test_exchange_gloo(world, kind, n, L, transpose, mode):
    res = _run(world, kind, n, L, transpose, mode)
    assert all(ok for _, ok, *_ in res)
    modes = {m for _, _, _, m, _, _ in res}
    assert len(modes) == 1                          # every rank took the same exchange
    if mode != "auto":
        assert modes == {mode}
    if kind in ("stencil", "band") and mode == "auto" and n >= 100:
        assert modes == {"window"}
    if kind == "random" and mode == "auto":
        assert modes == {"allgather"}
    if kind == "stencil" and modes == {"window"}:
        g = int(round(n ** 0.5))
        # halo only: each rank receives at most two grid lines per neighbour
        assert all(b <= 2 * g * 4 * (L + 1) for _, _, b, *_ in res)
        # stencil blocks are mostly interior rows
        assert all(inner >= rows - 2 * g for *_, inner, rows in res)


def test_block_range_properties():
    for n in (0, 1, 7, 100, 4_000_000):
        for G in (1, 2, 3, 4, 8):
            blocks = [block_range(n, G, r) for r in range(G)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(b[0] <= b[1] for b in blocks)
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(G - 1))
            assert max(b[1] - b[0] for b in blocks) == (block_size(n, G) if n else 0)


def test_choose_exchange_rule():
    # G = 2, blocks [0, 50) and [50, 100): receives 5 and 20 of 50
    assert choose_exchange("auto", [(0, 55), (30, 100)], 100) == "window"
    # rank 1 would receive 26 of 50
    assert choose_exchange("auto", [(0, 55), (24, 100)], 100) == "allgather"
    assert choose_exchange("window", [(0, 100), (0, 100)], 100) == "window"
    assert choose_exchange("auto", [(0, 0)], 0) == "window"


@pytest.mark.parametrize("transpose", [False, True])
def test_interior_mask_brute_force(transpose):
    rng = np.random.default_rng(2)
    for kind, n in (("band", 60), ("stencil", 100), ("random", 50)):
        rowptr, colidx = _pattern(kind, n)
        n = len(rowptr) - 1
        for G in (2, 3):
            for r in range(G):
                rb, re = block_range(n, G, r)
                m = interior_mask(rowptr, colidx, rb, re, transpose=transpose)
                for i in range(rb, re):
                    if transpose:
                        reads = [a for a in range(n) if i in colidx[rowptr[a]:rowptr[a + 1]]]
                    else:
                        reads = list(colidx[rowptr[i]:rowptr[i + 1]])
                    assert m[i - rb] == all(rb <= c < re for c in reads)
    a, b = interior_run(np.array([0, 1, 1, 0, 1, 1, 1, 0], bool))
    assert (a, b) == (4, 7)
    assert interior_run(np.zeros(3, bool)) == (0, 0)
