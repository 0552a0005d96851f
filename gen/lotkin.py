"""The paper's section-3 workload: the Lotkin matrix "randomly filled with
zeros" (SPEC gen_lotkin / sparsify).

  lotkin(n, p)            dense n x n: row 1 all ones, a_ij = RN_p(1/(i+j-1))
                          for i >= 2 (1-based), correctly rounded to nearest
                          even.  This is INPUT generation (the reciprocal is
                          the matrix definition, not the SpMV method), done
                          by exact integer division; tests/test_gen.py pins it
                          against Fraction.
  splitmix64(seed)        the exact SplitMix64 stream (constants
                          0x9E3779B97F4A7C15, 0xBF58476D1CE4E5B9,
                          0x94D049BB133111EB).
  sparsify(D, s, seed)    zero exactly k = round(s/100 n^2) distinct positions,
                          chosen by a partial Fisher-Yates shuffle of the n^2
                          linear indices driven by SplitMix64(seed); returns
                          the dense matrix with those zeros and its CSR
                          (exact zeros dropped).
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1


def recip(k: int, p: int):
    """(sign, M, E) of RN_p(1/k), k >= 1: value M 2^(E-p), M in [2^(p-1), 2^p)."""
    b = k.bit_length()
    if k == 1 << (b - 1):                      # 1/2^(b-1) = 2^(p-1) 2^((2-b)-p)
        return 0, 1 << (p - 1), 2 - b
    E = 1 - b                                  # 2^(E-1) < 1/k < 2^E
    q, r = divmod(1 << (p - E), k)             # 1/k = (q + r/k) 2^(E-p)
    if 2 * r > k:                              # 2r == k is impossible (k not a power of 2)
        q += 1
    if q == 1 << p:
        q, E = 1 << (p - 1), E + 1
    return 0, q, E


def lotkin(n: int, p: int):
    """Dense Lotkin matrix as packed arrays: limbs [n*n, L], exps, signs (row-major)."""
    L = p // 32
    # entry (i, j) (0-based) is 1/k with k = 1 on row 0, else i + j + 1
    tl = np.zeros((2 * n + 1, L), dtype=np.uint32)
    te = np.zeros(2 * n + 1, dtype=np.int32)
    for k in range(1, 2 * n + 1):
        _, M, e = recip(k, p)
        tl[k] = np.frombuffer(M.to_bytes(4 * L, "little"), dtype="<u4")
        te[k] = e
    K = np.add.outer(np.arange(n), np.arange(n)) + 1
    K[0, :] = 1
    K = K.ravel()
    return tl[K], te[K], np.zeros(n * n, dtype=np.uint8)


def splitmix64(seed: int):
    """Infinite SplitMix64 stream (python ints in [0, 2^64))."""
    x = seed & M64
    while True:
        x = (x + 0x9E3779B97F4A7C15) & M64
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        yield z ^ (z >> 31)


def zero_positions(n: int, s: float, seed: int) -> np.ndarray:
    """The k = round(s/100 n^2) linear indices zeroed: the first k slots of a
    partial Fisher-Yates shuffle (slot t swaps with t + (r mod (N - t)))."""
    N = n * n
    k = int(round(s / 100.0 * N))
    perm = np.arange(N, dtype=np.int64)
    g = splitmix64(seed)
    for t in range(k):
        u = t + next(g) % (N - t)
        perm[t], perm[u] = perm[u], perm[t]
    return np.sort(perm[:k])


def sparsify(n: int, dense, s: float, seed: int):
    """(dense arrays with the zeros, CSR dict) of the Lotkin matrix with s% zeros."""
    limbs, exps, signs = (a.copy() for a in dense)
    z = zero_positions(n, s, seed)
    limbs[z] = 0
    exps[z] = 0
    signs[z] = 0
    keep = np.any(limbs != 0, axis=1)
    rows = np.repeat(np.arange(n), n)
    cols = np.tile(np.arange(n, dtype=np.int32), n)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=rowptr[1:])
    csr = dict(rowptr=rowptr, colidx=cols[keep].astype(np.int32), limbs=limbs[keep],
               exps=exps[keep], signs=signs[keep])
    return (limbs, exps, signs), csr


def xvec(n: int, p: int):
    """x = [1, 2, ..., n] packed (exact: every k < 2^p is representable)."""
    L = p // 32
    xl = np.zeros((n, L), dtype=np.uint32)
    xe = np.zeros(n, dtype=np.int32)
    xs = np.zeros(n, dtype=np.uint8)
    for i in range(n):
        v = i + 1
        b = v.bit_length()
        xl[i] = np.frombuffer((v << (p - b)).to_bytes(4 * L, "little"), dtype="<u4")
        xe[i] = b
    return xl, xe, xs


def make(n: int, s: float, p: int, seed: int = 0) -> dict:
    """Sparsified Lotkin workload with x = [1..n] (SPEC spmv_bench: b = A [1..n]^T)."""
    dense, csr = sparsify(n, lotkin(n, p), s, seed)
    xl, xe, xs = xvec(n, p)
    return dict(p=p, n=n, s=s, seed=seed, dense_limbs=dense[0], dense_exps=dense[1],
                dense_signs=dense[2], x_limbs=xl, x_exps=xe, x_signs=xs, **csr)
