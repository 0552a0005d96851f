"""Python face of the C ABI: CSR handles and device MP vectors.

Argument marshalling only - every step of the SpMV runs in libmpsp's CUDA
kernels.  torch provides device memory and streams (plumbing).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def check_vec(v: "MPVec", n: int, L: int, name: str, device=None) -> None:
    """Raise ValueError unless v is an n-element, L-limb MPVec of int32 /
    int32 / uint8 contiguous CUDA tensors (on `device` if given): the C ABI
    takes raw pointers and cannot check sizes itself."""
    if not isinstance(v, MPVec):
        raise ValueError(f"{name}: expected an MPVec, got {type(v).__name__}")
    l, e, s = v.limbs, v.exps, v.signs
    if l.dim() != 2 or tuple(l.shape) != (n, L) or tuple(e.shape) != (n,) or tuple(s.shape) != (n,):
        raise ValueError(f"{name}: shape limbs {tuple(l.shape)} exps {tuple(e.shape)} signs "
                         f"{tuple(s.shape)}, expected ({n}, {L}) / ({n},) / ({n},)")
    if l.dtype != torch.int32 or e.dtype != torch.int32 or s.dtype != torch.uint8:
        raise ValueError(f"{name}: dtypes {l.dtype}/{e.dtype}/{s.dtype}, expected int32/int32/uint8")
    if not (l.is_contiguous() and e.is_contiguous() and s.is_contiguous()):
        raise ValueError(f"{name}: tensors must be contiguous")
    devs = {l.device, e.device, s.device}
    if len(devs) != 1 or next(iter(devs)).type != "cuda":
        raise ValueError(f"{name}: tensors must live on one CUDA device, got {devs}")
    if device is not None and l.device != torch.device(device):
        raise ValueError(f"{name}: on {l.device}, expected {device}")


def _ptr(a) -> int:
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


@dataclass
class MPVec:
    """A p-bit vector on the GPU: limbs int32 [n, L] (uint32 bit patterns),
    exps int32 [n], signs uint8 [n].  Packed format of include/mpsp.h."""
    limbs: "torch.Tensor"
    exps: "torch.Tensor"
    signs: "torch.Tensor"

    @property
    def n(self) -> int:
        return int(self.exps.shape[0])

    @property
    def L(self) -> int:
        return int(self.limbs.shape[1])

    @classmethod
    def empty(cls, n: int, L: int, device="cuda") -> "MPVec":
        return cls(torch.empty((n, L), dtype=torch.int32, device=device),
                   torch.empty((n,), dtype=torch.int32, device=device),
                   torch.empty((n,), dtype=torch.uint8, device=device))

    @classmethod
    def from_host(cls, limbs: np.ndarray, exps: np.ndarray, signs: np.ndarray, device="cuda",
                  L: int | None = None) -> "MPVec":
        L = L or (limbs.shape[1] if limbs.ndim == 2 else None)
        l = np.ascontiguousarray(limbs, dtype=np.uint32).reshape(-1, L).view(np.int32)
        return cls(torch.from_numpy(l.copy()).to(device),
                   torch.from_numpy(np.ascontiguousarray(exps, dtype=np.int32).copy()).to(device),
                   torch.from_numpy(np.ascontiguousarray(signs, dtype=np.uint8).copy()).to(device))

    def to_host(self):
        l = self.limbs.cpu().numpy().view(np.uint32)
        return l, self.exps.cpu().numpy(), self.signs.cpu().numpy()


class CSR:
    """Handle on rows [row_begin, row_end) of an n x n p-bit CSR matrix on the
    current CUDA device (mpsp_csr_create).  Inputs are host numpy arrays in
    the packed format; the handle copies them."""

    def __init__(self, p: int, rowptr, colidx, limbs, exps, signs, rows=None,
                 transpose: bool = False):
        self.p = int(p)
        self.L = self.p // 32
        self.n = int(len(rowptr) - 1)
        rb, re = (0, self.n) if rows is None else (int(rows[0]), int(rows[1]))
        self.row_begin, self.row_end = rb, re
        self._keep = [np.ascontiguousarray(rowptr, dtype=np.int64),
                      np.ascontiguousarray(colidx, dtype=np.int32),
                      np.ascontiguousarray(limbs, dtype=np.uint32),
                      np.ascontiguousarray(exps, dtype=np.int32),
                      np.ascontiguousarray(signs, dtype=np.uint8)]
        rp, ci, li, ex, sg = self._keep
        h = ctypes.c_void_p()
        rc = _lib.lib().mpsp_csr_create(ctypes.byref(h), self.p, self.n, _ptr(rp), _ptr(ci),
                                        _ptr(li), _ptr(ex), _ptr(sg), rb, re,
                                        _lib.MPSP_WITH_TRANSPOSE if transpose else 0)
        self._keep = None
        _lib.check(rc, "mpsp_csr_create")
        self._h = h
        self.transpose = transpose

    @classmethod
    def dense(cls, p: int, n: int, limbs, exps, signs, rows=None, transpose: bool = False):
        """Handle on a DENSE row-major n x n matrix (entry (i, j) at i*n + j,
        zeros stored as all-zero limbs): mpsp_dense_create.  spmv / spmv_t then
        run the dense MP MV - every row's chain over all n columns."""
        self = cls.__new__(cls)
        self.p, self.L, self.n = int(p), int(p) // 32, int(n)
        rb, re = (0, self.n) if rows is None else (int(rows[0]), int(rows[1]))
        self.row_begin, self.row_end = rb, re
        li = np.ascontiguousarray(limbs, dtype=np.uint32)
        ex = np.ascontiguousarray(exps, dtype=np.int32)
        sg = np.ascontiguousarray(signs, dtype=np.uint8)
        h = ctypes.c_void_p()
        rc = _lib.lib().mpsp_dense_create(ctypes.byref(h), self.p, self.n, _ptr(li), _ptr(ex),
                                          _ptr(sg), rb, re,
                                          _lib.MPSP_WITH_TRANSPOSE if transpose else 0)
        _lib.check(rc, "mpsp_dense_create")
        self._h = h
        self.transpose = transpose
        return self

    @property
    def rows(self) -> int:
        return self.row_end - self.row_begin

    def info(self) -> dict:
        arr = (ctypes.c_int64 * 10)()
        _lib.check(_lib.lib().mpsp_csr_info(self._h, arr), "mpsp_csr_info")
        keys = ("p", "n", "row_begin", "row_end", "nnz", "nnz_t", "device_bytes", "device",
                "slots", "max_row")
        return dict(zip(keys, [int(v) for v in arr]))

    def _apply(self, fn, x: MPVec, out: MPVec | None, stream) -> MPVec:
        check_vec(x, self.n, self.L, "x")
        if out is None:
            out = MPVec.empty(self.rows, self.L, device=x.limbs.device)
        check_vec(out, self.rows, self.L, "out", device=x.limbs.device)
        if stream is None:
            stream = torch.cuda.current_stream(x.limbs.device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        rc = fn(self._h, _ptr(x.limbs), _ptr(x.exps), _ptr(x.signs),
                _ptr(out.limbs), _ptr(out.exps), _ptr(out.signs), ctypes.c_void_p(stream))
        _lib.check(rc, fn.__name__)
        return out

    def spmv(self, x: MPVec, out: MPVec | None = None, stream=None) -> MPVec:
        """y = A x for the handle's rows (async on `stream`, default: torch's current)."""
        return self._apply(_lib.lib().mpsp_spmv, x, out, stream)

    def spmv_t(self, x: MPVec, out: MPVec | None = None, stream=None) -> MPVec:
        """y = A^T x for the handle's rows of A^T (needs transpose=True)."""
        return self._apply(_lib.lib().mpsp_spmv_t, x, out, stream)

    def _host(self, fn, xl, xe, xs, out=None):
        xl = np.ascontiguousarray(xl, dtype=np.uint32).reshape(-1)
        xe = np.ascontiguousarray(xe, dtype=np.int32)
        xs = np.ascontiguousarray(xs, dtype=np.uint8)
        if xl.size != self.n * self.L or xe.shape != (self.n,) or xs.shape != (self.n,):
            raise ValueError(f"x: expected {self.n} elements of {self.L} limbs")
        if out is None:
            out = (np.empty((self.rows, self.L), np.uint32), np.empty(self.rows, np.int32),
                   np.empty(self.rows, np.uint8))
        yl, ye, ys = out
        for a, dt, size in ((yl, np.uint32, self.rows * self.L), (ye, np.int32, self.rows),
                            (ys, np.uint8, self.rows)):
            if not isinstance(a, np.ndarray) or a.dtype != dt or a.size != size or \
                    not a.flags.c_contiguous:
                raise ValueError(f"out: expected contiguous {np.dtype(dt).name} arrays of "
                                 f"{self.rows} rows x {self.L} limbs")
        rc = fn(self._h, _ptr(xl), _ptr(xe), _ptr(xs), _ptr(yl), _ptr(ye), _ptr(ys))
        _lib.check(rc, fn.__name__)
        return out

    def spmv_host(self, xl, xe, xs, out=None):
        """y = A x with HOST buffers (copies inside the call; synchronous)."""
        return self._host(_lib.lib().mpsp_spmv_host, xl, xe, xs, out)

    def spmv_t_host(self, xl, xe, xs, out=None):
        return self._host(_lib.lib().mpsp_spmv_t_host, xl, xe, xs, out)

    def gpbicg(self, b: MPVec, max_iter: int, x: MPVec | None = None, stream=None):
        """Solve A x = b by GPBiCG (Fig. 4 right, K = I; mpsp_gpbicg).
        Transpose-free; full-matrix handle, p >= 128.  Returns (x, iterations,
        status)."""
        return self._solve(_lib.lib().mpsp_gpbicg, b, max_iter, x, stream)

    def bicg(self, b: MPVec, max_iter: int, x: MPVec | None = None, stream=None):
        """Solve A x = b by BiCG (Fig. 4, K = I; mpsp_bicg).  Needs a
        full-matrix handle built with transpose=True and p >= 128.  Returns
        (x, iterations, status) with status "converged" | "breakdown" |
        "max_iter"."""
        return self._solve(_lib.lib().mpsp_bicg, b, max_iter, x, stream)

    def _solve(self, fn, b, max_iter, x, stream):
        check_vec(b, self.n, self.L, "b")
        if x is None:
            x = MPVec.empty(self.n, self.L, device=b.limbs.device)
        check_vec(x, self.n, self.L, "x", device=b.limbs.device)
        if stream is None:
            stream = torch.cuda.current_stream(b.limbs.device).cuda_stream
        it, st = ctypes.c_int(0), ctypes.c_int(0)
        rc = fn(self._h, _ptr(b.limbs), _ptr(b.exps), _ptr(b.signs), _ptr(x.limbs),
                _ptr(x.exps), _ptr(x.signs), int(max_iter), ctypes.byref(it), ctypes.byref(st),
                ctypes.c_void_p(stream))
        _lib.check(rc, fn.__name__)
        return x, it.value, _lib.BICG_STATUS[st.value]

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            _lib.lib().mpsp_destroy(h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def _stream(dev, stream):
    if stream is None:
        return torch.cuda.current_stream(dev).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else stream


def dot(p: int, u: MPVec, v: MPVec, out: MPVec | None = None, stream=None) -> MPVec:
    """(u, v) as the ordered rounded chain (mpsp_dot); a 1-element MPVec."""
    L = p // 32
    check_vec(u, u.n, L, "u")
    check_vec(v, u.n, L, "v", device=u.limbs.device)
    if out is None:
        out = MPVec.empty(1, L, device=u.limbs.device)
    check_vec(out, 1, L, "out", device=u.limbs.device)
    rc = _lib.lib().mpsp_dot(int(p), u.n, _ptr(u.limbs), _ptr(u.exps), _ptr(u.signs),
                             _ptr(v.limbs), _ptr(v.exps), _ptr(v.signs), _ptr(out.limbs),
                             _ptr(out.exps), _ptr(out.signs),
                             ctypes.c_void_p(_stream(u.limbs.device, stream)))
    _lib.check(rc, "mpsp_dot")
    return out


def axpy(p: int, alpha: MPVec, x: MPVec, y: MPVec, negate: bool = False,
         out: MPVec | None = None, stream=None) -> MPVec:
    """out_k = RN(y_k + RN(+-alpha x_k)) (mpsp_axpy); alpha a 1-element MPVec."""
    L = p // 32
    check_vec(alpha, 1, L, "alpha", device=x.limbs.device)
    check_vec(x, x.n, L, "x")
    check_vec(y, x.n, L, "y", device=x.limbs.device)
    if out is None:
        out = MPVec.empty(x.n, L, device=x.limbs.device)
    check_vec(out, x.n, L, "out", device=x.limbs.device)
    rc = _lib.lib().mpsp_axpy(int(p), x.n, _ptr(alpha.limbs), _ptr(alpha.exps), _ptr(alpha.signs),
                              1 if negate else 0, _ptr(x.limbs), _ptr(x.exps), _ptr(x.signs),
                              _ptr(y.limbs), _ptr(y.exps), _ptr(y.signs), _ptr(out.limbs),
                              _ptr(out.exps), _ptr(out.signs),
                              ctypes.c_void_p(_stream(x.limbs.device, stream)))
    _lib.check(rc, "mpsp_axpy")
    return out
