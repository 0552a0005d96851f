"""Stress corpus: CSR inputs that force the rounding corners (SURVEY.md 8(c)
"Stress corpus" items 1-9).  Pure input construction - no method arithmetic.

Most corner rows multiply by x = 1 exactly (unit columns, x = (+, 2^(p-1), 1)),
so each product equals its A entry and the row is a pure rounded add chain
whose operands (and therefore exponent gaps, signs, tie patterns) are chosen
here.  Product corners use dedicated x columns.
"""
from __future__ import annotations

import numpy as np

from .configs import pack_triples, ROOT_SEED


def _val(s, M, e):
    return (int(s), int(M), int(e))


def stress(p: int, seed: int = 0, long_len: int = 5000, n_random_rows: int = 300) -> dict:
    L = p // 32
    rng = np.random.default_rng(np.random.SeedSequence([ROOT_SEED, 99, p, seed]))
    import random
    R = random.Random(int(rng.integers(0, 2**62)))
    top = 1 << (p - 1)
    full = (1 << p) - 1

    def rmant():
        return top | R.getrandbits(p - 1)

    # ---------------------------------------------------------------- x
    U = 72                                      # unit columns 0..U-1: x = 1
    xs = [_val(0, top, 1) for _ in range(U)]
    SPECIAL = {}

    def add_x(v, name):
        SPECIAL[name] = len(xs)
        xs.append(v)

    add_x(_val(0, top | 1, 0), "1p")              # (2^(p-1)+1)/2^p
    add_x(_val(0, full, 0), "ones")               # 1 - 2^-p
    add_x(_val(1, top, 1), "minus1")
    add_x(_val(0, top | (top >> 1), 2), "three")  # 3
    add_x(_val(0, top | (1 << (p // 2)), 1), "halfbit")
    add_x(_val(1, 0, 12345), "zero_junk")         # zero with junk sign/exp
    add_x(_val(0, 0, 0), "zero")
    add_x(_val(0, top, (1 << 29)), "hugeexp")
    add_x(_val(1, rmant(), -(1 << 29)), "tinyexp")
    nx_special = len(xs)

    rows = []                                    # list of [(col, a_triple)]

    def unit_row(vals):
        assert len(vals) <= U
        rows.append([(j, v) for j, v in enumerate(vals)])

    # 1-2. product ties and carry-outs (a * special x)
    for _ in range(12):
        nb = R.randint(1, min(p, 8))
        Ma = (((1 << (nb - 1)) | R.getrandbits(nb - 1)) if nb > 1 else 1) << (p - nb)
        rows.append([(SPECIAL["1p"], _val(R.getrandbits(1), Ma, R.randint(-5, 5)))])
        rows.append([(SPECIAL["halfbit"], _val(R.getrandbits(1), Ma | (1 << (p // 2)), R.randint(-5, 5)))])
    rows.append([(SPECIAL["1p"], _val(0, full - 1, 0))])              # carry-out (A.3)
    rows.append([(SPECIAL["ones"], _val(0, full, 0))])
    rows.append([(SPECIAL["ones"], _val(1, top | 1, 3)), (SPECIAL["three"], _val(0, full, -2))])
    rows.append([(SPECIAL["three"], _val(0, top | (top >> 2), 1))])

    # 3. adds with chosen exponent gaps d, both sign combos, mantissa patterns
    mpat = [top, full, top | 1, full ^ (1 << (p - 2)), rmant()]
    for k in range(1, L):
        mpat.append(top | ((1 << (32 * k)) - 1))     # low limbs all ones
    gaps = sorted({0, 1, 2, 3, 31, 32, 33, p - 1, p, p + 1, p + 2, p + 3, 2 * p, 5000})
    for d in gaps:
        for sa in (0, 1):
            for sb in (0, 1):
                Ma, Mb = R.choice(mpat), R.choice(mpat)
                unit_row([_val(sa, Ma, 10), _val(sb, Mb, 10 - d)])
                unit_row([_val(sb, Mb, 10 - d), _val(sa, Ma, 10)])
    # 4. power-of-two boundaries: down (A.3) and up
    for e in (0, 7, -9):
        unit_row([_val(0, top, e), _val(1, top, e - p - 1)])                  # tie below
        unit_row([_val(0, top, e), _val(1, top | 1, e - p - 1)])              # just past tie
        unit_row([_val(0, top, e), _val(1, top, e - p - 2)])
        unit_row([_val(1, top, e), _val(0, top, e - p)])
        unit_row([_val(0, full, e), _val(0, top, e - p)])                      # up to 2^e: tie
        unit_row([_val(0, full, e), _val(0, top | 1, e - p)])
        unit_row([_val(0, full, e), _val(0, top, e - p - 1)])
        unit_row([_val(1, full, e), _val(1, full, e - p + 1)])
    # 5. cancellation: exact, +-1 ulp, massive, then continue
    for _ in range(6):
        M = rmant()
        e = R.randint(-20, 20)
        unit_row([_val(0, M, e), _val(1, M, e), _val(0, rmant(), e - 3)])
        unit_row([_val(0, M, e), _val(1, min(M + 1, full), e)])
        unit_row([_val(0, M, e), _val(1, max(M - 1, top), e), _val(1, rmant(), e - p - 4)])
        unit_row([_val(0, top, e), _val(1, full, e - 1)])                    # 1-bit result
        Mlow = M ^ (R.getrandbits(3) + 1)
        if Mlow < top:
            Mlow = M
        unit_row([_val(0, M, e), _val(1, Mlow, e), _val(0, rmant(), e - 2 * p)])
    # partial sums passing through zero repeatedly
    M = rmant()
    unit_row([_val(i % 2, M, 4) for i in range(12)] + [_val(0, rmant(), -3)])
    # 6. row lengths 0, 1, 2, 31, 32, 33 over random columns
    for ln in (0, 1, 2, 31, 32, 33):
        rows.append(("rand", ln))
    # 7. rows of explicit zero entries (junk sign/exp) and zero x
    rows.append([(0, _val(1, 0, 77)), (1, _val(0, 0, -5)), (2, _val(1, 0, 0))])
    rows.append([(0, _val(0, rmant(), 1)), (SPECIAL["zero_junk"], _val(0, rmant(), 2)),
                 (SPECIAL["zero"], _val(1, rmant(), 3))])
    rows.append([(SPECIAL["zero_junk"], _val(1, rmant(), 0))])
    # 8. exponent extremes |exp| = 2^29
    big, sm = 1 << 29, -(1 << 29)
    unit_row([_val(0, rmant(), big), _val(1, rmant(), sm)])
    unit_row([_val(1, rmant(), sm), _val(0, rmant(), big), _val(0, rmant(), sm)])
    rows.append([(SPECIAL["hugeexp"], _val(0, rmant(), big)), (SPECIAL["tinyexp"], _val(1, rmant(), sm))])
    rows.append([(SPECIAL["tinyexp"], _val(0, rmant(), sm))])
    # 9. limb-boundary carry ripple: all-ones mantissa + half-ulp tie (odd -> up)
    unit_row([_val(0, full, 3), _val(0, top, 3 - p)])
    unit_row([_val(0, full ^ 2, 3), _val(0, top, 3 - p), _val(0, top, 3 - p)])
    # a long row (critical-path case) and random rows
    rows.append(("rand", long_len))
    for _ in range(n_random_rows):
        rows.append(("rand", R.randint(0, 40)))

    n = max(len(rows), long_len + nx_special + 8, nx_special + 64)
    # random x for the remaining columns (some zeros)
    while len(xs) < n:
        if R.random() < 0.03:
            xs.append(_val(R.getrandbits(1), 0, R.randint(-9, 9)))
        else:
            xs.append(_val(R.getrandbits(1), rmant(), R.randint(-40, 40)))
    # materialise rows, pad with empty rows up to n
    cols_all, vals_all, rowptr = [], [], [0]
    for r in rows:
        if isinstance(r, tuple):
            ln = r[1]
            cols = sorted(R.sample(range(nx_special, n), ln))
            ent = []
            for c in cols:
                u = R.random()
                if u < 0.05:
                    ent.append((c, _val(R.getrandbits(1), 0, R.randint(-3, 3))))
                elif u < 0.15:
                    nb = min(R.randint(1, 6), p - 1)    # few significant bits: tie-prone
                    ent.append((c, _val(R.getrandbits(1), top | (R.getrandbits(nb) << (p - 1 - nb)),
                                        R.randint(-8, 8))))
                else:
                    ent.append((c, _val(R.getrandbits(1), rmant(), R.randint(-40, 40))))
            r = ent
        r = sorted(r, key=lambda t: t[0])
        assert all(r[i][0] < r[i + 1][0] for i in range(len(r) - 1))
        for c, v in r:
            cols_all.append(c)
            vals_all.append(v)
        rowptr.append(len(cols_all))
    while len(rowptr) < n + 1:
        rowptr.append(len(cols_all))
    limbs, exps, signs = pack_triples(vals_all, p)
    xl, xe, xs_ = pack_triples(xs, p)
    # zero entries keep their junk sign/exp (they must read as zero)
    for k, (s, M, e) in enumerate(vals_all):
        if M == 0:
            exps[k], signs[k] = e, s
    for j, (s, M, e) in enumerate(xs):
        if M == 0:
            xe[j], xs_[j] = e, s
    rowptr = np.array(rowptr, dtype=np.int64)
    d = dict(cfg=f"stress{p}", seed=seed, p=p, n=n, rowptr=rowptr,
             colidx=np.array(cols_all, dtype=np.int32), limbs=limbs, exps=exps, signs=signs,
             x_limbs=xl, x_exps=xe, x_signs=xs_)
    d["meta"] = dict(cfg=d["cfg"], seed=seed, p=p, n=n, nnz=int(rowptr[-1]),
                     max_row=int(np.diff(rowptr).max()))
    return d
