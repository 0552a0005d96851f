"""Row-block multi-GPU SpMV: one process per GPU (BASELINE.json north_star (4);
SURVEY.md 8(e)).

Rank r owns rows [r*blk, min((r+1)*blk, n)) of A (blk = ceil(n/G)) and the
same block of x.  Before each application x must be present on every rank
wherever the rank's rows read it.  Two exchanges:

* ``allgather``: x replicated everywhere by NCCL all_gather_into_tensor (the
  literal north_star step);
* ``window`` (default, "needed-window exchange", SURVEY.md 8(e)
  recommendation 2): each rank's rows read only columns in [lo, hi) (computed
  once from the CSR); every rank sends each peer the part of its own block
  that lies in the peer's window, as NCCL point-to-point sends in one batch.
  For banded / stencil patterns (C2, C5) that is two halos of a few hundred
  KB; for random patterns (C3, C4) the windows span [0, n) and the exchange
  moves the same bytes as the all-gather.

No reduction collective exists on this path: each row's ordered chain runs
entirely on one GPU, so results are bit-identical to one GPU for either
exchange (the exchanged x elements are copied bit for bit).

The partition / exchange logic is plain torch.distributed and works with gloo
(CPU tensors) for tests; the SpMV itself is the CUDA library.
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


def needed_window(rowptr, colidx, rb: int, re: int, transpose: bool = False) -> tuple[int, int]:
    """[lo, hi) of the x indices read by rows [rb, re) of A (or of A^T: the
    row indices i of A's entries whose column lies in [rb, re)).  (0, 0) if
    the rows read nothing."""
    rowptr = np.asarray(rowptr)
    colidx = np.asarray(colidx)
    if not transpose:
        c = colidx[rowptr[rb]:rowptr[re]]
        return (int(c.min()), int(c.max()) + 1) if len(c) else (0, 0)
    hit = (colidx >= rb) & (colidx < re)
    if not hit.any():
        return (0, 0)
    k = np.flatnonzero(hit)
    rows = np.searchsorted(rowptr, k, side="right") - 1
    return int(rows.min()), int(rows.max()) + 1


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


class WindowExchange:
    """Needed-window exchange of x into a rank-local full-length buffer.

    Setup (collective, once): every rank contributes its window [lo, hi); the
    plan sends peer q the intersection of this rank's block with q's window
    and receives from q the intersection of q's block with this window."""

    def __init__(self, n: int, L: int, window: tuple[int, int], group=None, device=None):
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = n
        self.rb, self.re = block_range(n, self.G, self.rank)
        dev = torch.device(device) if device is not None else torch.device("cpu")
        nccl = dist.get_backend(group) == "nccl"
        w = torch.tensor([window[0], window[1]], dtype=torch.int64,
                         device=dev if nccl else "cpu")
        allw = [torch.empty_like(w) for _ in range(self.G)]
        dist.all_gather(allw, w, group=group)
        self.windows = [(int(t[0]), int(t[1])) for t in allw]
        self.sends, self.recvs = [], []
        lo, hi = self.windows[self.rank]
        for q in range(self.G):
            if q == self.rank:
                continue
            qlo, qhi = self.windows[q]
            s0, s1 = max(self.rb, qlo), min(self.re, qhi)
            if s0 < s1:
                self.sends.append((q, s0, s1))
            qb, qe = block_range(n, self.G, q)
            r0, r1 = max(qb, lo), min(qe, hi)
            if r0 < r1:
                self.recvs.append((q, r0, r1))
        self.x = MPVec(torch.zeros((n, L), dtype=torch.int32, device=dev),
                       torch.zeros((n,), dtype=torch.int32, device=dev),
                       torch.zeros((n,), dtype=torch.uint8, device=dev))
        self.bytes_in = sum((r1 - r0) * (4 * L + 5) for _, r0, r1 in self.recvs)

    def local_view(self) -> MPVec:
        """This rank's block of the buffer (write x_local here to skip a copy)."""
        return MPVec(self.x.limbs[self.rb:self.re], self.x.exps[self.rb:self.re],
                     self.x.signs[self.rb:self.re])

    def exchange(self, x_local: MPVec | None = None) -> MPVec:
        """Copy x_local into the buffer (unless it is the local view) and fill
        this rank's window from its peers.  Returns the full-length buffer
        (valid inside the window)."""
        if x_local is not None and self.re > self.rb and \
                x_local.limbs.data_ptr() != self.x.limbs[self.rb:self.re].data_ptr():
            self.x.limbs[self.rb:self.re].copy_(x_local.limbs)
            self.x.exps[self.rb:self.re].copy_(x_local.exps)
            self.x.signs[self.rb:self.re].copy_(x_local.signs)
        ops = []
        for t in (self.x.limbs, self.x.exps, self.x.signs):
            for q, s0, s1 in self.sends:
                ops.append(dist.P2POp(dist.isend, t[s0:s1], q, group=self.group))
            for q, r0, r1 in self.recvs:
                ops.append(dist.P2POp(dist.irecv, t[r0:r1], q, group=self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        return self.x


class DistCSR:
    """Rank-local row block of A (and optionally A^T) plus the x exchange."""

    def __init__(self, p, rowptr, colidx, limbs, exps, signs, group=None, transpose=False,
                 exchange: str = "window", device=None):
        if exchange not in ("window", "allgather"):
            raise ValueError("exchange must be 'window' or 'allgather'")
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = len(rowptr) - 1
        self.L = p // 32
        self.rows = block_range(self.n, self.G, self.rank)
        self.exchange_kind = exchange
        self.local = CSR(p, rowptr, colidx, limbs, exps, signs, rows=self.rows, transpose=transpose)
        self.xchg = {}
        if exchange == "window":
            for t in ((False, True) if transpose else (False,)):
                win = needed_window(rowptr, colidx, *self.rows, transpose=t)
                self.xchg[t] = WindowExchange(self.n, self.L, win, group, device)

    def apply(self, x_local: MPVec, out: MPVec | None = None, transpose=False) -> MPVec:
        if self.exchange_kind == "allgather":
            x_full = allgather_x(x_local, self.n, self.group)
        else:
            x_full = self.xchg[transpose].exchange(x_local)
        f = self.local.spmv_t if transpose else self.local.spmv
        return f(x_full, out=out)

    def close(self):
        self.local.close()
