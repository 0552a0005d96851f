"""Row-block multi-GPU SpMV: one process per GPU, x replicated by an all-gather
before each application (BASELINE.json north_star (4)).

Rank r owns rows [r*blk, min((r+1)*blk, n)) of A (blk = ceil(n/G)) and the
same block of x.  apply(x_local) all-gathers x (limbs, exps, signs) into a
padded x_full of G*blk elements, then runs the local handle over it.  No
reduction collective exists on this path: each row's ordered chain runs
entirely on one GPU, so the result is bit-identical to one GPU.

The partition / exchange logic is plain torch.distributed and works with
gloo (CPU tensors) for tests; the SpMV itself is the CUDA library.
"""
from __future__ import annotations

import numpy as np

from .csr import CSR, MPVec

try:
    import torch
    import torch.distributed as dist
except ImportError:  # pragma: no cover
    torch = None
    dist = None


def block_range(n: int, G: int, r: int) -> tuple[int, int]:
    blk = (n + G - 1) // G if G else 0
    return min(r * blk, n), min((r + 1) * blk, n)


def block_size(n: int, G: int) -> int:
    return (n + G - 1) // G


def allgather_x(x_local: MPVec, n: int, group=None) -> MPVec:
    """Replicate x: every rank passes its block (padded to blk rows by this
    function) and receives the G*blk-row concatenation (first n rows valid)."""
    G = dist.get_world_size(group)
    blk = block_size(n, G)
    L = x_local.limbs.shape[1]
    dev = x_local.limbs.device
    m = x_local.limbs.shape[0]
    if m != blk:  # pad the (last) short block
        pl = torch.zeros((blk, L), dtype=x_local.limbs.dtype, device=dev)
        pe = torch.zeros((blk,), dtype=x_local.exps.dtype, device=dev)
        ps = torch.zeros((blk,), dtype=x_local.signs.dtype, device=dev)
        pl[:m] = x_local.limbs
        pe[:m] = x_local.exps
        ps[:m] = x_local.signs
        x_local = MPVec(pl, pe, ps)
    out = MPVec(torch.empty((G * blk, L), dtype=x_local.limbs.dtype, device=dev),
                torch.empty((G * blk,), dtype=x_local.exps.dtype, device=dev),
                torch.empty((G * blk,), dtype=x_local.signs.dtype, device=dev))
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out.limbs, x_local.limbs.contiguous(), group=group)
        dist.all_gather_into_tensor(out.exps, x_local.exps.contiguous(), group=group)
        dist.all_gather_into_tensor(out.signs, x_local.signs.contiguous(), group=group)
    else:  # gloo (tests): list form
        for dst, src in ((out.limbs, x_local.limbs), (out.exps, x_local.exps),
                         (out.signs, x_local.signs)):
            dist.all_gather(list(dst.chunk(G)), src.contiguous(), group=group)
    return out


class DistCSR:
    """Rank-local row block of A (and optionally A^T) plus the x exchange."""

    def __init__(self, p, rowptr, colidx, limbs, exps, signs, group=None, transpose=False):
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = len(rowptr) - 1
        self.rows = block_range(self.n, self.G, self.rank)
        self.local = CSR(p, rowptr, colidx, limbs, exps, signs, rows=self.rows, transpose=transpose)

    def apply(self, x_local: MPVec, out: MPVec | None = None, transpose=False) -> MPVec:
        x_full = allgather_x(x_local, self.n, self.group)
        f = self.local.spmv_t if transpose else self.local.spmv
        return f(x_full, out=out)

    def close(self):
        self.local.close()
