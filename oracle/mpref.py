"""Plain, slow, obviously-correct CPU oracle for multiple-precision CSR SpMV.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product path (``paper_1411_2377_b200``) never imports it, and this
module imports nothing from the product path: the two share no code.

What it computes (arXiv 1411.2377, "A Highly Efficient Implementation of
Multiple Precision Sparse Matrix-Vector Multiplication ..."):

* PAPER.md:119-133 (Sec. 2): the matrix is stored in CSR form, one array of
  nonzero elements plus per-row column indices.
* PAPER.md:81-85 (Sec. 2): MPFR arithmetic, IEEE-754-style correctly rounded
  p-bit operations; the rounding mode used is RN (reading c1 in DESIGN.md).
* PAPER.md:182-186 (Sec. 3): the product A^(s,p) b; PAPER.md:282-284 (Fig. 4,
  BiCG): z = A p and z~ = A^T p~ (the paper typesets the second "A", reading
  c3: it is the transpose).
* BASELINE.json north_star: rounding to nearest-even after every multiply and
  every add, each row's products summed in ascending column order; the A^T
  order is ascending row index of A.

Representation: a nonzero value is a triple (s, M, E) with value
(-1)^s * M * 2^(E-p) and 2^(p-1) <= M < 2^p (MPFR exponent convention,
reading c7).  Zero is (0, 0, 0).  No NaN/Inf/subnormals (reading c8).

Every arithmetic step uses Python integers, no floats anywhere.  Each
function follows SURVEY.md section 8(c) "Algorithm, step by step" in order.

Parity status: ``rn``/``mul``/``add`` are pinned by tests/test_oracle_pins.py
against MPFR (library routine, via ctypes), mpmath.libmp, exact Fraction
arithmetic with a single rounding, hand-worked examples and brute force.
``spmv``/``spmv_t`` are pinned by the invariants listed in DESIGN.md (identity,
permutation, transpose, small-integer exactness, scaling, negation,
densification) and by the 1-nnz-row == single rounding property.  The paper
prints no SpMV values to store as a fixture: whole-config outputs are pinned
through the pieces above and the hand-worked SpMV examples of tests/golden/
(every function of this module has a pin).  ``dense_mv`` (the paper's
section-3 dense MP MV) is pinned by closed forms (Lotkin
row 1 times [1..n] = n(n+1)/2 exactly; A e_j = column j) and by dense ==
sparse bitwise (tests/test_lotkin.py).  Every function works at any p that is
a multiple of 32 (the GPU path: 32 ... 8192).
"""
from __future__ import annotations

import numpy as np

ZERO = (0, 0, 0)

# Threshold above which add() uses the far-path lemma instead of exact
# alignment (exact alignment of a 2^30-bit shift would need a 128 MB integer).
# The lemma (checked in tests) holds for d >= p + 2; it is only
# applied when d also exceeds this threshold so the boundary region is always
# computed by exact alignment.
FAR_THRESHOLD = 4096


# --------------------------------------------------------------------------
# Scalar arithmetic
# --------------------------------------------------------------------------

def rn(N: int, f: int, p: int) -> tuple[int, int]:
    """Round the positive integer N (value N * 2^f) to p bits, ties to even.

    Returns (M, E) with value M * 2^(E-p), 2^(p-1) <= M < 2^p.
    Step 1 of SURVEY 8(c); RN = round-to-nearest of PAPER.md:84-85.
    """
    assert N > 0
    b = N.bit_length()
    if b <= p:
        return (N << (p - b), f + b)
    sh = b - p
    q = N >> sh
    r = N & ((1 << sh) - 1)
    h = 1 << (sh - 1)
    if r > h or (r == h and (q & 1)):
        q += 1
    E = f + b
    if q == (1 << p):
        q = 1 << (p - 1)
        E += 1
    return (q, E)


def mul(a: tuple, x: tuple, p: int) -> tuple:
    """t = RN_p(a * x).  A zero operand gives +0 (reading c5)."""
    sa, Ma, Ea = a
    sx, Mx, Ex = x
    if Ma == 0 or Mx == 0:
        return ZERO
    M, E = rn(Ma * Mx, Ea + Ex - 2 * p, p)
    return (sa ^ sx, M, E)


def add(u: tuple, v: tuple, p: int) -> tuple:
    """RN_p(u + v).  An exact zero sum is +0 (reading c5)."""
    su, Mu, Eu = u
    sv, Mv, Ev = v
    if Mu == 0:
        return v
    if Mv == 0:
        return u
    d = abs(Eu - Ev)
    if d > FAR_THRESHOLD and d >= p + 2:
        # far-path lemma: |small| < ulp(big)/4, so RN(big + small) = big
        return u if Eu > Ev else v
    f = min(Eu, Ev) - p
    S = (-1 if su else 1) * (Mu << (Eu - p - f)) + (-1 if sv else 1) * (Mv << (Ev - p - f))
    if S == 0:
        return ZERO
    M, E = rn(abs(S), f, p)
    return (1 if S < 0 else 0, M, E)


# --------------------------------------------------------------------------
# Packed <-> triple conversion (SURVEY.md 8(b) value encoding, 8(c) step 6)
# --------------------------------------------------------------------------

def unpack(limbs_row: np.ndarray, e: int, s: int, p: int) -> tuple:
    """(L uint32 limbs, limb 0 least significant) + exp + sign -> triple."""
    M = int.from_bytes(np.ascontiguousarray(limbs_row, dtype='<u4').tobytes(), 'little')
    if M == 0:
        return ZERO  # any all-zero mantissa is zero, whatever exp/sign (c25)
    if M.bit_length() != p:
        raise ValueError("unnormalised nonzero input (MSB of top limb not set)")
    return (int(s) & 1, M, int(e))


def unpack_vec(limbs: np.ndarray, exps: np.ndarray, signs: np.ndarray, p: int) -> list:
    L = p // 32
    limbs = np.asarray(limbs, dtype=np.uint32).reshape(-1, L)
    return [unpack(limbs[i], int(exps[i]), int(signs[i]), p) for i in range(limbs.shape[0])]


def pack_vec(vals: list, p: int):
    """list of triples -> (limbs uint32 [n, L], exps int32 [n], signs uint8 [n])."""
    L = p // 32
    n = len(vals)
    limbs = np.zeros((n, L), dtype=np.uint32)
    exps = np.zeros(n, dtype=np.int32)
    signs = np.zeros(n, dtype=np.uint8)
    for i, (s, M, E) in enumerate(vals):
        if M == 0:
            continue
        limbs[i] = np.frombuffer(M.to_bytes(4 * L, 'little'), dtype='<u4')
        exps[i] = E
        signs[i] = s
    return limbs, exps, signs


# --------------------------------------------------------------------------
# SpMV
# --------------------------------------------------------------------------

def row_chain(p: int, entries) -> tuple:
    """s = +0; for (a, x) in order: s = RN(s + RN(a * x))."""
    s = ZERO
    for a, x in entries:
        s = add(s, mul(a, x, p), p)
    return s


def spmv_rows(p, rowptr, colidx, limbs, exps, signs, x_limbs, x_exps, x_signs, rows):
    """y_i for the listed rows i of y = A x (ascending column order per row).

    Inputs are the packed host format of SURVEY 8(b); returns a list of triples.
    """
    L = p // 32
    limbs = np.asarray(limbs, dtype=np.uint32).reshape(-1, L)
    x_limbs = np.asarray(x_limbs, dtype=np.uint32).reshape(-1, L)
    out = []
    for i in rows:
        entries = []
        for k in range(int(rowptr[i]), int(rowptr[i + 1])):
            j = int(colidx[k])
            a = unpack(limbs[k], int(exps[k]), int(signs[k]), p)
            x = unpack(x_limbs[j], int(x_exps[j]), int(x_signs[j]), p)
            entries.append((a, x))
        out.append(row_chain(p, entries))
    return out


def spmv(p, rowptr, colidx, limbs, exps, signs, x_limbs, x_exps, x_signs):
    """y = A x for all rows; returns packed (limbs [n, L], exps, signs)."""
    n = len(rowptr) - 1
    vals = spmv_rows(p, rowptr, colidx, limbs, exps, signs,
                     x_limbs, x_exps, x_signs, range(n))
    return pack_vec(vals, p)


def transpose(n, rowptr, colidx):
    """Independent transpose by sorting (col, row, k) triples (step 5).

    Returns (rowptr_t, colidx_t, perm) where perm[k_t] = k, the index of the
    entry of A stored at position k_t of A^T.  Within each transposed row the
    order is ascending row index of A (BASELINE.json north_star (3)).
    """
    triples = []
    for i in range(n):
        for k in range(int(rowptr[i]), int(rowptr[i + 1])):
            triples.append((int(colidx[k]), i, k))
    triples = sorted(triples)
    rowptr_t = [0] * (n + 1)
    for (j, _, _) in triples:
        rowptr_t[j + 1] += 1
    for j in range(n):
        rowptr_t[j + 1] += rowptr_t[j]
    colidx_t = [i for (_, i, _) in triples]
    perm = [k for (_, _, k) in triples]
    return (np.array(rowptr_t, dtype=np.int64), np.array(colidx_t, dtype=np.int32),
            np.array(perm, dtype=np.int64))


def transpose_np(n, rowptr, colidx):
    """The same transpose as ``transpose`` (step 5) with numpy's stable sort.

    A stable argsort of the entries by column keeps, inside each column, the
    CSR storage order - ascending row index of A (BASELINE.json north_star
    (3)).  A library sort primitive, for full-size inputs where sorting
    Python tuples would take minutes; pinned against ``transpose`` in
    tests/test_oracle_invariants.py.  Returns (rowptr_t, colidx_t, perm).
    """
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colidx = np.asarray(colidx, dtype=np.int64)
    perm = np.argsort(colidx, kind='stable').astype(np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))   # row i of entry k
    rowptr_t = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(colidx, minlength=n), out=rowptr_t[1:])
    return rowptr_t, rows[perm].astype(np.int32), perm


def spmv_t(p, rowptr, colidx, limbs, exps, signs, x_limbs, x_exps, x_signs):
    """y = A^T x: y_j = chain over i ascending with (i, j) stored of RN(A_ij x_i)."""
    n = len(rowptr) - 1
    L = p // 32
    rowptr_t, colidx_t, perm = transpose(n, rowptr, colidx)
    limbs = np.asarray(limbs, dtype=np.uint32).reshape(-1, L)
    return spmv(p, rowptr_t, colidx_t, limbs[perm], np.asarray(exps)[perm],
                np.asarray(signs)[perm], x_limbs, x_exps, x_signs)


def spmv_t_cols(p, rowptr, colidx, limbs, exps, signs, x_limbs, x_exps, x_signs, cols):
    """(A^T x)_j for the listed j, for sampled checks at full size.

    Column j's entries are located with numpy (a search primitive); their
    order is ascending row index of A because CSR rows are visited in order.
    """
    L = p // 32
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colidx = np.asarray(colidx)
    limbs = np.asarray(limbs, dtype=np.uint32).reshape(-1, L)
    x_limbs = np.asarray(x_limbs, dtype=np.uint32).reshape(-1, L)
    out = []
    for j in cols:
        ks = np.flatnonzero(colidx == j)
        rows = np.searchsorted(rowptr, ks, side='right') - 1  # row i of entry k
        order = np.argsort(rows, kind='stable')
        entries = []
        for k, i in zip(ks[order], rows[order]):
            a = unpack(limbs[k], int(exps[k]), int(signs[k]), p)
            x = unpack(x_limbs[i], int(x_exps[i]), int(x_signs[i]), p)
            entries.append((a, x))
        out.append(row_chain(p, entries))
    return out


# --------------------------------------------------------------------------
# Dense MP MV (the section-3 dense
# vs sparse comparison; SPEC dense_mv): y_i = the ordered chain over
# ALL n columns j of row i, zeros included.
# --------------------------------------------------------------------------

def dense_mv(p, n, limbs, exps, signs, x_limbs, x_exps, x_signs, transpose=False):
    """y = A x (or A^T x) for a dense row-major n x n A (entry (i, j) at i*n + j)."""
    L = p // 32
    limbs = np.asarray(limbs, dtype=np.uint32).reshape(-1, L)
    x = unpack_vec(x_limbs, x_exps, x_signs, p)
    out = []
    for i in range(n):
        entries = []
        for j in range(n):
            k = j * n + i if transpose else i * n + j
            entries.append((unpack(limbs[k], int(exps[k]), int(signs[k]), p), x[j]))
        out.append(row_chain(p, entries))
    return pack_vec(out, p)
