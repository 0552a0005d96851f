"""Seeded synthetic inputs for multiple-precision CSR SpMV (C1..C5, stress).

This module is shared by the oracle side (tests) and the CUDA side (tests,
bench); it holds NO arithmetic of the method (no rounding, no products, no
sums of values) - only pattern and bit-pattern construction.

Recipes follow BASELINE.json `configs` (C1..C5) with the readings of
DESIGN.md and the seeds of SURVEY.md 8(d):
``np.random.SeedSequence([14112377, k, seed])`` for config k, spawned into
three children (pattern, A values, x values).

Value encoding: a nonzero is (-1)^sign * M/2^p * 2^exp with
M in [2^(p-1), 2^p) stored as L = p/32 uint32 limbs, limb 0 least
significant; zero = all limbs 0 (exp = sign = 0).

The paper's own workloads are UF-collection matrices (cavity04 n=317,
nnz=7327; epb3 n=84617, nnz=463,625) and
the sparsified Lotkin matrix.  They are not in this
container; these synthetic configs stand in for their shapes.
"""
from __future__ import annotations

import hashlib

import numpy as np

ROOT_SEED = 14112377
CONFIG_IDS = ("C1", "C2", "C3", "C4", "C5")

# p (bits) and default n per config (BASELINE.json configs[0..4])
SPEC = {
    "C1": dict(p=128, n=2000),
    "C2": dict(p=256, n=100_000),
    "C3": dict(p=512, n=500_000),
    "C4": dict(p=256, n=1_000_000),
    "C5": dict(p=1024, n=4_000_000),   # 2000 x 2000 grid
}


# ------------------------------------------------------------------ values
def rand_mantissas(rng: np.random.Generator, count: int, L: int) -> np.ndarray:
    """count x L uint32 limbs, top bit set, other p-1 bits uniform (c22)."""
    m = rng.integers(0, 1 << 32, size=(count, L), dtype=np.uint32)
    if count:
        m[:, L - 1] |= np.uint32(0x80000000)
    return m


def rand_values(rng, count, L, elo, ehi):
    """Random full mantissas, exponent uniform in [elo, ehi], random sign."""
    limbs = rand_mantissas(rng, count, L)
    exps = rng.integers(elo, ehi + 1, size=count, dtype=np.int64).astype(np.int32)
    signs = rng.integers(0, 2, size=count, dtype=np.uint8)
    return limbs, exps, signs


def pack_triples(vals, p):
    """[(sign, M, exp)] python ints -> packed arrays (plain bit copy)."""
    L = p // 32
    n = len(vals)
    limbs = np.zeros((n, L), dtype=np.uint32)
    exps = np.zeros(n, dtype=np.int32)
    signs = np.zeros(n, dtype=np.uint8)
    for i, (s, M, e) in enumerate(vals):
        if M == 0:
            continue
        limbs[i] = np.frombuffer(int(M).to_bytes(4 * L, "little"), dtype="<u4")
        exps[i] = e
        signs[i] = s
    return limbs, exps, signs


# ------------------------------------------------------------------ patterns
def _dedupe_sorted(rng, rows, cols, lo, hi, skip_diag):
    """Make columns distinct within each row (resample duplicates), sorted.

    Entries are ordered by the single key row * K + col (K > every column):
    the same order as lexsort((cols, rows)), one int64 sort per round."""
    K = np.int64(max(int(hi), int(cols.max()) + 1 if len(cols) else 1))
    key = np.sort(rows * K + cols)
    while True:
        dup = np.zeros(len(key), dtype=bool)
        if len(key) > 1:
            dup[1:] = key[1:] == key[:-1]
        nd = int(dup.sum())
        if nd == 0:
            return key // K, key % K
        r = key[dup] // K
        new = rng.integers(lo, hi, size=nd, dtype=np.int64)
        if skip_diag:
            new = new + (new >= r)
        key = key.copy()
        key[dup] = r * K + new
        key = np.sort(key)


def pattern_diag_plus_random(rng, n, k_off):
    """Row i = {i} U k_off[i] distinct uniform off-diagonal columns, sorted."""
    k_off = np.asarray(k_off, dtype=np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), k_off)
    cols = rng.integers(0, max(n - 1, 1), size=len(rows), dtype=np.int64)
    cols = cols + (cols >= rows)                      # skip the diagonal
    rows, cols = _dedupe_sorted(rng, rows, cols, 0, max(n - 1, 1), True)
    rows = np.concatenate([rows, np.arange(n, dtype=np.int64)])
    cols = np.concatenate([cols, np.arange(n, dtype=np.int64)])
    order = np.lexsort((cols, rows))
    return _to_csr(n, rows[order], cols[order])


def pattern_random_rows(rng, n, k):
    """Row i = k[i] distinct uniform columns (no forced diagonal), sorted."""
    k = np.asarray(k, dtype=np.int64)
    dense = k > n // 4              # near-full rows (small n only): sample w/o replacement
    kk = np.where(dense, 0, k)
    rows = np.repeat(np.arange(n, dtype=np.int64), kk)
    cols = rng.integers(0, n, size=len(rows), dtype=np.int64)
    rows, cols = _dedupe_sorted(rng, rows, cols, 0, n, False)
    for i in np.flatnonzero(dense):
        rows = np.concatenate([rows, np.full(k[i], i, dtype=np.int64)])
        cols = np.concatenate([cols, rng.choice(n, size=k[i], replace=False).astype(np.int64)])
    if dense.any():
        order = np.lexsort((cols, rows))
        rows, cols = rows[order], cols[order]
    return _to_csr(n, rows, cols)


def pattern_band(n, w):
    """Columns max(0, i-w) .. min(n-1, i+w)."""
    i = np.arange(n, dtype=np.int64)
    lo = np.maximum(0, i - w)
    hi = np.minimum(n - 1, i + w)
    cnt = hi - lo + 1
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rowptr[1:])
    rows = np.repeat(i, cnt)
    cols = rows * 0 + (np.arange(rowptr[-1], dtype=np.int64) - np.repeat(rowptr[:-1], cnt)) + np.repeat(lo, cnt)
    return rowptr, cols.astype(np.int32)


def pattern_stencil5(g):
    """2-D 5-point stencil on a g x g grid, row-major idx = gy*g + gx,
    Dirichlet truncation (c21).  Columns ascending per row."""
    n = g * g
    idx = np.arange(n, dtype=np.int64)
    gy, gx = idx // g, idx % g
    nb = [(idx - g, gy > 0), (idx - 1, gx > 0), (idx, np.ones(n, bool)),
          (idx + 1, gx < g - 1), (idx + g, gy < g - 1)]
    cnt = sum(m.astype(np.int64) for _, m in nb)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rowptr[1:])
    cols = np.empty(rowptr[-1], dtype=np.int32)
    pos = rowptr[:-1].copy()
    is_diag = np.zeros(rowptr[-1], dtype=bool)
    for c, m in nb:                                   # ascending column order
        cols[pos[m]] = c[m]
        if c is idx:
            is_diag[pos[m]] = True
        pos[m] += 1
    return rowptr, cols, is_diag


def _to_csr(n, rows, cols):
    cnt = np.bincount(rows, minlength=n).astype(np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rowptr[1:])
    return rowptr, cols.astype(np.int32)


# ------------------------------------------------------------------ configs
def _seeds(cfg_index, seed):
    ss = np.random.SeedSequence([ROOT_SEED, cfg_index, seed])
    return [np.random.default_rng(s) for s in ss.spawn(3)]


def make(cfg: str, seed: int = 0, n: int | None = None, p: int | None = None) -> dict:
    """Build config `cfg` (C1..C5).  `n` / `p` override the size / precision
    (same recipe) for oracle-sized parity cases.  Returns a dict of packed
    host arrays: p, n, rowptr (int64), colidx (int32), limbs (uint32 [nnz, L]),
    exps (int32), signs (uint8), x_limbs, x_exps, x_signs, plus `meta`."""
    k = CONFIG_IDS.index(cfg) + 1
    spec = SPEC[cfg]
    p = p or spec["p"]
    n = n or spec["n"]
    L = p // 32
    r_pat, r_a, r_x = _seeds(k, seed)
    if cfg == "C1":
        rowptr, colidx = pattern_diag_plus_random(r_pat, n, np.full(n, min(7, n - 1)))
        limbs, exps, signs = rand_values(r_a, len(colidx), L, -4, 4)
        xl, xe, xs = rand_values(r_x, n, L, -4, 4)
        nz = r_x.permutation(n)[: int(round(0.05 * n))]    # exactly 5% zeros
        xl[nz] = 0
        xe[nz] = 0
        xs[nz] = 0
    elif cfg == "C2":
        rowptr, colidx = pattern_band(n, 5)
        limbs, exps, signs = rand_values(r_a, len(colidx), L, -8, 8)
        rows = np.repeat(np.arange(n), np.diff(rowptr))
        exps[colidx == rows] = 4                           # c18: literal
        xl, xe, xs = rand_values(r_x, n, L, -8, 8)
    elif cfg == "C3":
        kk = np.maximum(1, r_pat.poisson(12, size=n))
        rowptr, colidx = pattern_diag_plus_random(r_pat, n, np.minimum(kk - 1, n - 1))
        limbs, exps, signs = rand_values(r_a, len(colidx), L, -16, 16)
        xl, xe, xs = rand_values(r_x, n, L, -16, 16)
    elif cfg == "C4":
        kk = np.minimum(r_pat.zipf(1.8, size=n), min(5000, n)).astype(np.int64)
        rowptr, colidx = pattern_random_rows(r_pat, n, kk)
        limbs, exps, signs = rand_values(r_a, len(colidx), L, -32, 32)
        xl, xe, xs = rand_values(r_x, n, L, -32, 32)
    elif cfg == "C5":
        g = int(round(np.sqrt(n)))
        assert g * g == n, "C5 needs a square grid"
        rowptr, colidx, is_diag = pattern_stencil5(g)
        limbs, exps, signs = stencil_values(r_a, is_diag, L)
        xl, xe, xs = rand_values(r_x, n, L, -2, 2)
    else:
        raise KeyError(cfg)
    d = dict(cfg=cfg, seed=seed, p=p, n=n, rowptr=rowptr, colidx=colidx,
             limbs=limbs, exps=exps, signs=signs,
             x_limbs=xl, x_exps=xe, x_signs=xs)
    d["meta"] = dict(cfg=cfg, seed=seed, p=p, n=n, nnz=int(rowptr[-1]),
                     max_row=int(np.diff(rowptr).max()) if n else 0)
    return d


def stencil_values(rng, is_diag, L):
    """C5 values (c21): diagonal exactly 4; off-diagonal -1 + delta with
    delta = k * 2^(1-p), k = +-m, m uniform in [0, 2^(p-21)).

    Encodings (no arithmetic, bit patterns only):
      k > 0 : M = 2^p - 2m  = top 20 bits ones | random even low field, exp 0
      k <= 0: M = 2^(p-1) + m = 1, 20 zero bits, random (p-21)-bit field, exp 1
      diag  : M = 2^(p-1), exp 3, sign 0.
    """
    nnz = len(is_diag)
    limbs = rng.integers(0, 1 << 32, size=(nnz, L), dtype=np.uint32)
    pos = rng.integers(0, 2, size=nnz, dtype=np.uint8).astype(bool)   # k > 0
    top20 = np.uint32(0xFFFFF000)
    # --- k > 0: top 20 bits ones, bit 0 cleared, low field nonzero
    limbs[pos, L - 1] |= top20
    limbs[pos, 0] &= np.uint32(0xFFFFFFFE)
    # --- k <= 0: MSB set, next 20 bits zero
    neg = ~pos
    limbs[neg, L - 1] &= np.uint32(0x000007FF)
    limbs[neg, L - 1] |= np.uint32(0x80000000)
    exps = np.where(pos, 0, 1).astype(np.int32)
    signs = np.ones(nnz, dtype=np.uint8)
    # a k>0 low field of all zeros would be M = 2^p - 0: not representable
    low_zero = pos & np.all(limbs[:, :] == np.where(np.arange(L) == L - 1, top20, 0), axis=1)
    limbs[low_zero, 0] |= np.uint32(2)
    limbs[is_diag] = 0
    limbs[is_diag, L - 1] = np.uint32(0x80000000)
    exps[is_diag] = 3
    signs[is_diag] = 0
    return limbs, exps, signs


def sha256_arrays(d: dict) -> str:
    h = hashlib.sha256()
    for key in ("rowptr", "colidx", "limbs", "exps", "signs", "x_limbs", "x_exps", "x_signs"):
        h.update(np.ascontiguousarray(d[key]).tobytes())
    return h.hexdigest()
