"""Row-block multi-GPU SpMV: one process per GPU (BASELINE.json north_star (4);
SURVEY.md 8(a) row a4, 8(e)).

Rank r owns rows [r*blk, min((r+1)*blk, n)) of A (blk = ceil(n/G)) and the
same block of x.  Before each application x must be present on every rank
wherever the rank's rows read it.  Each x element travels as ONE record of
L + 1 words (L limbs, then the exponent word with the sign in bit 31;
mpsp_vec_pack / mpsp_vec_unpack, csrc/xchg.cu), so an exchange is one NCCL
call per peer (or one all-gather), not three.  Two exchanges:

* ``allgather``: x replicated everywhere by one NCCL all_gather_into_tensor
  of records (the literal north_star step);
* ``window`` ("needed-window exchange", SURVEY.md 8(e) recommendation 2):
  each rank's rows read only columns in [lo, hi) (computed once from the
  CSR); every rank sends each peer the records of its own block that lie in
  the peer's window, as NCCL point-to-point sends in one batch.  For banded /
  stencil patterns (C2, C5) that is two halos of a few hundred KB.

``auto`` (default) takes the window exchange unless some rank would receive
more than half of what the all-gather brings it (random patterns, C3 / C4:
every window is [0, n) and the P2P batch would move the all-gather's bytes
in 2 (G-1) messages).  The
decision is made from all ranks' windows, so every rank takes the same one.

Overlap (SURVEY.md 8(e) recommendation 3): ``DistCSR`` splits the rank's rows
into boundary rows and one contiguous run of INTERIOR rows that read only the
rank's own block of x.  Each application starts the exchange, runs the
interior rows' kernels while the records are in flight, then unpacks the
received records and runs the boundary rows.  Stencils (C5) are almost all
interior; random patterns have no interior rows and run after the exchange.

No reduction collective exists on this path: each row's ordered chain runs
entirely on one GPU, so results are bit-identical to one GPU for either
exchange (the exchanged x elements are copied bit for bit).

The partition / exchange logic is plain torch.distributed and also runs
under gloo (CPU tensors) in the tests, with a test-side record packer; the
product path packs with the library's kernels and the SpMV is the CUDA
library.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .csr import CSR, MPVec, _ptr

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


def interior_mask(rowptr, colidx, rb: int, re: int, transpose: bool = False) -> np.ndarray:
    """Boolean per row of [rb, re): True if the row reads x only inside the
    rank's own block [rb, re) (empty rows included)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colidx = np.asarray(colidx)
    m = re - rb
    if not transpose:
        seg = colidx[rowptr[rb]:rowptr[re]]
        outside = ((seg < rb) | (seg >= re)).astype(np.int64)
        row_of = np.repeat(np.arange(m), np.diff(rowptr[rb:re + 1]))
        bad = np.bincount(row_of, weights=outside, minlength=m) if m else np.zeros(0)
        return bad == 0
    k = np.flatnonzero((colidx >= rb) & (colidx < re))
    i = np.searchsorted(rowptr, k, side="right") - 1          # row of A of entry k
    out = (i < rb) | (i >= re)
    mask = np.ones(m, dtype=bool)
    mask[colidx[k[out]] - rb] = False
    return mask


def interior_run(mask: np.ndarray) -> tuple[int, int]:
    """The longest run [a, b) of True in mask (relative indices); (0, 0) if none."""
    if not mask.any():
        return (0, 0)
    d = np.diff(np.concatenate([[0], mask.astype(np.int8), [0]]))
    starts, ends = np.flatnonzero(d == 1), np.flatnonzero(d == -1)
    j = int(np.argmax(ends - starts))
    return int(starts[j]), int(ends[j])


def choose_exchange(kind: str, windows, n: int) -> str:
    """'window' or 'allgather' from every rank's window (same on all ranks):
    the window exchange unless some rank would receive more than half of
    what the all-gather brings it (x outside its own block)."""
    if kind != "auto":
        return kind
    G = len(windows)
    worst = 0.0
    for r, (lo, hi) in enumerate(windows):
        rb, re = block_range(n, G, r)
        recv = max(0, min(hi, rb) - lo) + max(0, hi - max(lo, re))
        worst = max(worst, recv / max(1, n - (re - rb)))
    return "window" if worst <= 0.5 else "allgather"


class LibPacker:
    """Record pack / unpack with the library's kernels (csrc/xchg.cu) on the
    current CUDA stream."""

    def __init__(self, L: int):
        self.p = 32 * L

    def pack(self, v: MPVec, rec, stream=None) -> None:
        st = ctypes.c_void_p(stream if stream is not None else
                             torch.cuda.current_stream(rec.device).cuda_stream)
        _lib.check(_lib.lib().mpsp_vec_pack(self.p, v.n, _ptr(v.limbs), _ptr(v.exps), _ptr(v.signs),
                                            _ptr(rec), st), "mpsp_vec_pack")

    def unpack(self, rec, v: MPVec, stream=None) -> None:
        st = ctypes.c_void_p(stream if stream is not None else
                             torch.cuda.current_stream(rec.device).cuda_stream)
        _lib.check(_lib.lib().mpsp_vec_unpack(self.p, v.n, _ptr(rec), _ptr(v.limbs), _ptr(v.exps),
                                              _ptr(v.signs), st), "mpsp_vec_unpack")


def _default_device(group):
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _slice(v: MPVec, a: int, b: int) -> MPVec:
    return MPVec(v.limbs[a:b], v.exps[a:b], v.signs[a:b])


class XExchange:
    """The x exchange into a rank-local full-length vector ``self.x`` (ABI
    layout), valid wherever this rank's rows read it.

    Setup (collective, once): the windows of all ranks are all-gathered, the
    exchange kind is chosen (``choose_exchange``) and the send / receive
    plans are fixed.  ``start`` packs and issues the NCCL calls
    asynchronously; ``finish`` waits for them and unpacks the received
    records; ``exchange`` = both."""

    def __init__(self, n: int, L: int, window: tuple[int, int], group=None, device=None,
                 mode: str = "auto", packer=None):
        if mode not in ("auto", "window", "allgather"):
            raise ValueError("mode must be 'auto', 'window' or 'allgather'")
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n, self.L = n, L
        self.rb, self.re = block_range(n, self.G, self.rank)
        self.nccl = dist.get_backend(group) == "nccl"
        dev = torch.device(device) if device is not None else _default_device(group)
        self.device = dev
        self.packer = packer if packer is not None else LibPacker(L)
        w = torch.tensor([window[0], window[1]], dtype=torch.int64,
                         device=dev if self.nccl else "cpu")
        allw = [torch.empty_like(w) for _ in range(self.G)]
        dist.all_gather(allw, w, group=group)
        self.windows = [(int(t[0]), int(t[1])) for t in allw]
        self.mode = choose_exchange(mode, self.windows, n)
        self.x = MPVec(torch.zeros((n, L), dtype=torch.int32, device=dev),
                       torch.zeros((n,), dtype=torch.int32, device=dev),
                       torch.zeros((n,), dtype=torch.uint8, device=dev))
        R = L + 1
        if self.mode == "allgather":
            blk = block_size(n, self.G)
            self.send_rec = torch.zeros((blk, R), dtype=torch.int32, device=dev)
            self.recv_rec = torch.zeros((self.G * blk, R), dtype=torch.int32, device=dev)
            self.sends = [(q, self.rb, self.re) for q in range(self.G) if q != self.rank]
            self.recvs = [(q, *block_range(n, self.G, q)) for q in range(self.G) if q != self.rank]
            self.bytes_in = (n - (self.re - self.rb)) * 4 * R
            return
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
        ns = sum(s1 - s0 for _, s0, s1 in self.sends)
        nr = sum(r1 - r0 for _, r0, r1 in self.recvs)
        self.send_rec = torch.zeros((max(ns, 1), R), dtype=torch.int32, device=dev)
        self.recv_rec = torch.zeros((max(nr, 1), R), dtype=torch.int32, device=dev)
        self.bytes_in = nr * 4 * R

    def local_view(self) -> MPVec:
        """This rank's block of the buffer (write x_local here to skip a copy)."""
        return _slice(self.x, self.rb, self.re)

    def set_local(self, limbs, exps, signs) -> None:
        """Copy this rank's block of x (host numpy or tensors) into the buffer."""
        v = self.local_view()
        for dst, src, dt in ((v.limbs, limbs, np.uint32), (v.exps, exps, np.int32),
                             (v.signs, signs, np.uint8)):
            if isinstance(src, np.ndarray):
                a = np.ascontiguousarray(src, dtype=dt)
                src = torch.from_numpy(a.view(np.int32) if dt == np.uint32 else a)
            dst.copy_(src.reshape(dst.shape))

    def start(self, stream=None):
        """Pack the outgoing records and issue the NCCL calls (asynchronous
        w.r.t. the host; under NCCL the transfers wait for the pack on the
        current stream).  Returns the pending works for ``finish``."""
        if self.G == 1:
            return []
        if self.mode == "allgather":
            m = self.re - self.rb
            if m:
                self.packer.pack(self.local_view(), self.send_rec[:m], stream)
            if self.nccl:
                return [dist.all_gather_into_tensor(self.recv_rec, self.send_rec, group=self.group,
                                                    async_op=True)]
            return [dist.all_gather(list(self.recv_rec.chunk(self.G)), self.send_rec,
                                    group=self.group, async_op=True)]
        ops, off = [], 0
        for q, s0, s1 in self.sends:
            seg = self.send_rec[off:off + s1 - s0]
            self.packer.pack(_slice(self.x, s0, s1), seg, stream)
            ops.append(dist.P2POp(dist.isend, seg, q, group=self.group))
            off += s1 - s0
        off = 0
        for q, r0, r1 in self.recvs:
            ops.append(dist.P2POp(dist.irecv, self.recv_rec[off:off + r1 - r0], q, group=self.group))
            off += r1 - r0
        return dist.batch_isend_irecv(ops) if ops else []

    def finish(self, works, stream=None) -> MPVec:
        """Wait for the transfers (under NCCL: the current stream waits) and
        unpack the received records into ``self.x``."""
        for w in works:
            w.wait()
        if self.G == 1:
            return self.x
        if self.mode == "allgather":
            for a, b in ((0, self.rb), (self.re, self.n)):
                if b > a:
                    self.packer.unpack(self.recv_rec[a:b], _slice(self.x, a, b), stream)
            return self.x
        off = 0
        for q, r0, r1 in self.recvs:
            self.packer.unpack(self.recv_rec[off:off + r1 - r0], _slice(self.x, r0, r1), stream)
            off += r1 - r0
        return self.x

    def exchange(self, stream=None) -> MPVec:
        return self.finish(self.start(stream), stream)

    def close(self):
        self.x = self.send_rec = self.recv_rec = None


class DistCSR:
    """Rank-local row block of A (and optionally A^T) plus the x exchange,
    with the interior rows overlapped with the exchange."""

    def __init__(self, p, rowptr, colidx, limbs, exps, signs, group=None, transpose=False,
                 exchange: str = "auto", device=None, overlap: bool = True, packer=None,
                 min_interior: float = 0.25):
        if exchange not in ("auto", "window", "allgather"):
            raise ValueError("exchange must be 'auto', 'window' or 'allgather'")
        self.group = group
        self.G = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.n = len(rowptr) - 1
        self.p, self.L = int(p), int(p) // 32
        self.rows = block_range(self.n, self.G, self.rank)
        rb, re = self.rows
        self.device = torch.device(device) if device is not None else _default_device(group)
        self.parts, self.xchg = {}, {}
        for t in ((False, True) if transpose else (False,)):
            win = needed_window(rowptr, colidx, rb, re, transpose=t)
            self.xchg[t] = XExchange(self.n, self.L, win, group, self.device, exchange, packer)
            a, b = (0, 0)
            if overlap and self.G > 1 and re > rb:
                a, b = interior_run(interior_mask(rowptr, colidx, rb, re, transpose=t))
                if b - a < min_interior * (re - rb):
                    a, b = (0, 0)
            cuts = [(rb, rb + a, False), (rb + a, rb + b, True), (rb + b, re, False)] if b > a \
                else [(rb, re, False)]
            self.parts[t] = [(CSR(p, rowptr, colidx, limbs, exps, signs, rows=(c0, c1),
                                  transpose=t), c0 - rb, c1 - rb, inner)
                             for c0, c1, inner in cuts if c1 > c0]
        self.exchange_kind = self.xchg[False].mode

    def interior_rows(self, transpose=False) -> int:
        return sum(h.rows for h, _, _, inner in self.parts[transpose] if inner)

    def apply(self, x_local: MPVec | None, out: MPVec | None = None, transpose=False,
              stream=None) -> MPVec:
        """y_local = the rank's rows of A x (A^T x).  x_local: this rank's block
        of x (None: already in ``xchg[transpose].local_view()``)."""
        X = self.xchg[transpose]
        if x_local is not None:
            v = X.local_view()
            if x_local.limbs.data_ptr() != v.limbs.data_ptr() and v.n:
                v.limbs.copy_(x_local.limbs)
                v.exps.copy_(x_local.exps)
                v.signs.copy_(x_local.signs)
        if out is None:
            out = MPVec.empty(self.rows[1] - self.rows[0], self.L, device=X.x.limbs.device)
        works = X.start()
        for h, a, b, inner in self.parts[transpose]:          # overlaps the transfers
            if inner:
                (h.spmv_t if transpose else h.spmv)(X.x, out=_slice(out, a, b), stream=stream)
        X.finish(works)
        for h, a, b, inner in self.parts[transpose]:
            if not inner:
                (h.spmv_t if transpose else h.spmv)(X.x, out=_slice(out, a, b), stream=stream)
        return out

    def close(self):
        for parts in self.parts.values():
            for h, _, _, _ in parts:
                h.close()
        for X in self.xchg.values():
            X.close()
