"""CPU models of the two non-obvious algorithms inside the CUDA kernels,
checked against the oracle on adversarial and random inputs.

These are test-side restatements (Python ints) of the REASONING the kernels
rely on - not of their code - so a flaw in the argument shows up here at CPU
speed over many more cases than the GPU parity tests run:

1. the short product with an exactness certificate (mp_device.cuh mp_mul):
   only Comba columns k >= L-3 are formed; if the bits of that partial sum
   between B = 32(L-2)+5 and the round bit are neither all 0 nor all 1, the
   rounded product equals RN(a*x) with sticky = 1;
2. the speculative exact block sum of spmv_wrow.cu: steps of the chain
   s = RN(s + t_k) whose partial sums provably stay in s's binade are integer
   additions on the grid u = ulp(s), with ties resolved from the running
   parity; everything else goes through the exact adder.

Both models are compared bit for bit with oracle.mul / oracle.add chains.
"""
import random

import pytest

import oracle

M32 = (1 << 32) - 1


# ---------------------------------------------------------------- 1. product
def short_product(Ma, Mx, p, D=None):
    """Model of mp_mul: returns (M, dE, certified) or None when the
    certificate fails (the kernel then forms the full product).  Columns
    k >= K0 = L - D are formed: D = 2 in mp_mul (L <= 32, MPSP_SHORT_D) and
    in the warp form for L = 64..256 (wide_mp.cuh wmul); D = 3 models round
    1's kernels."""
    L = p // 32
    if D is None:
        D = 2
    a = [(Ma >> (32 * i)) & M32 for i in range(L)]
    x = [(Mx >> (32 * i)) & M32 for i in range(L)]
    K0 = L - D
    T = sum(a[i] * x[j] << (32 * (i + j)) for i in range(L) for j in range(L) if i + j >= K0)
    N = Ma * Mx - T
    # K0 < 32 terms per omitted column (L <= 32, mp_mul): +37 over column K0;
    # the warp form for L = 64..256 has K0 < 256 terms: +40
    B = 32 * K0 + (37 if L <= 32 else 40)
    assert 0 <= N < (1 << B)                      # the bound the certificate uses
    sh = 0 if (T >> (64 * L - 1)) & 1 else 1
    rpos = 32 * L - 1 - sh                        # round bit position
    if D == 2 and L <= 32:
        B += 1 - sh                               # mp_mul's window: bits 6..30 of T[1] << sh
    # (wmul's window at D = 2: bits 8 .. 30-sh of limb L-1, i.e. [B, rpos))
    W = (T >> B) & ((1 << (rpos - B)) - 1)
    if W == 0 or W == (1 << (rpos - B)) - 1:
        return None
    q = T >> (rpos + 1)
    rb = (T >> rpos) & 1
    q += rb                                       # sticky = 1: round up iff rb
    dE = -sh
    if q == 1 << p:
        q >>= 1
        dE += 1
    return q, dE


@pytest.mark.parametrize("p,D", [(128, 2), (256, 2), (512, 2), (1024, 2), (2048, 2), (8192, 2),
                                 (256, 3), (1024, 3), (2048, 3), (8192, 3)])
def test_short_product_certificate_random(p, D):
    rng = random.Random(p)
    hits = 0
    for _ in range(3000 if p <= 1024 else 300):
        Ma = (1 << (p - 1)) | rng.getrandbits(p - 1)
        Mx = (1 << (p - 1)) | rng.getrandbits(p - 1)
        r = short_product(Ma, Mx, p, D)
        if r is None:
            continue
        hits += 1
        s, M, E = oracle.mul((0, Ma, 0), (0, Mx, 0), p)
        assert (M, E) == (r[0], r[1])
    assert hits == (3000 if p <= 1024 else 300)   # random mantissas never need the full product


@pytest.mark.parametrize("p,D", [(128, 2), (256, 2), (512, 2), (2048, 2), (256, 3), (2048, 3)])
def test_short_product_certificate_adversarial(p, D):
    """Structured mantissas (powers of two, all-ones runs, carries rippling
    into the round bit, exact ties): whenever the certificate passes the
    result is exact; ambiguous cases must be rejected, never mis-rounded."""
    rng = random.Random(7 * p)
    top = 1 << (p - 1)
    corpus = [top, (1 << p) - 1, top | 1, top | (1 << (p // 2)), top + (1 << 32) - 1,
              (1 << p) - (1 << (p // 2)), top | ((1 << (p // 2)) - 1)]
    for _ in range(200):
        corpus.append(top | rng.getrandbits(p - 1))
        k = rng.randrange(1, p - 1)
        corpus.append(top | ((1 << k) - 1))             # long runs of ones
        corpus.append(((1 << p) - 1) ^ (1 << rng.randrange(p - 1)))
    rejected = 0
    for Ma in corpus:
        for Mx in corpus[:60]:
            r = short_product(Ma, Mx, p, D)
            s, M, E = oracle.mul((0, Ma, 0), (0, Mx, 0), p)
            if r is None:
                rejected += 1
                continue
            assert (M, E) == (r[0], r[1]), (hex(Ma), hex(Mx))
    assert rejected > 0           # the corpus does exercise the fallback


def test_short_product_tie_is_never_certified():
    """An exact tie has all-zero bits below the round bit: W == 0, so the
    certificate must reject it (the kernel then rounds the exact product)."""
    p = 128
    a = (0, 3 << (p - 2), 2)                 # 3
    x = (0, (1 << (p - 1)) | 1, 1)           # 1 + 2^-(p-1)
    assert short_product(a[1], x[1], p) is None


# ---------------------------------------------------------------- 2. block sum
HB = 26


def block_sum_chain(ts, p, G=32, ties_exact=False, transitions=False, stats=None, herr2=False):
    """Model of spmv_wrow's chain over the products ts (oracle triples),
    G steps per block.  ties_exact=True models a chain that sends a grid tie
    through the exact path instead of resolving its parity (the U-steps-per-
    lane variant measured in round 2, G = 32U).
    transitions=True models WChain's one-binade transitions: a failing step
    whose exact sum provably crosses 2^p (same signs) or provably drops to
    [2^(p-2), 2^(p-1)) (opposite signs) is rounded on the new grid directly
    (2u or u/2) from W's low bits and the step's fraction bits, without the
    exact adder.  herr2=True models WChain::consume as of round 2: the high
    part of a step is taken from P = Y (plus sign) or ~Y (minus sign) - the
    rounding / two's-complement carry is added later by the commit's carry
    chain - so Q/H lies in [h, h + 2) and the bounds count two units of error
    per step (the transitions' bounds widened by one unit).
    Returns (result, n_fast_steps)."""
    L = p // 32
    S, E, sg, zero = 0, 0, 0, True         # exact S (grid integer), exponent, sign
    Shi, err, par = 0, 0, 0
    nfast = 0
    H = p - HB                             # log2 of the high-part unit in grid units
    M1 = 1                                 # one grid unit u <= one H unit (p >= HB)

    def hi(v):                             # floor(v / 2^H) (v may be negative)
        return v >> H if H >= 0 else v << (-H)

    for b0 in range(0, len(ts), G):
        blk = ts[b0:b0 + G]
        start = 0
        while start < len(blk):
            if zero:
                nz = [k for k in range(start, len(blk)) if blk[k][1] != 0]
                if not nz:
                    break
                f = nz[0]
                sg, S, E = blk[f]
                zero = False
                Shi, err, par = hi(S), 1, S & 1
                start = f + 1
                continue
            Q, ties, bad = [], [], []
            for k in range(len(blk)):
                st, Mt, Et = blk[k]
                act = k >= start and Mt != 0
                if not act:
                    Q.append(0); ties.append(False); bad.append(False)
                    continue
                d = E - Et
                if d < 1:
                    Q.append(0); ties.append(False); bad.append(True)
                    continue
                d = min(d, 32 * L + 32)
                Y = Mt >> d
                rem = Mt & ((1 << d) - 1)
                half = 1 << (d - 1)
                tie = rem == half
                inc = 1 if rem > half else 0
                Q.append((Y, inc, st != sg))
                ties.append(tie)
                bad.append(tie and ties_exact)
            # tie parity, then signed Q, then the conservative checks
            p_run = par
            PH = {}
            for k in range(len(blk)):
                if not isinstance(Q[k], tuple):
                    continue
                Y, inc, neg = Q[k]
                if ties[k]:
                    inc = p_run ^ (Y & 1)
                    p_run = 0
                else:
                    p_run ^= (Y + inc) & 1
                q = Y + inc
                Q[k] = -q if neg else q
                if herr2:
                    PH[k] = hi(-Y - 1 if neg else Y)
            EU = 2 if herr2 else 1               # bound error units per step

            def hq(k):
                return PH[k] if herr2 and k in PH else hi(Q[k])
            LB, cnt, fail = Shi, 0, None
            for k in range(len(blk)):
                h = hq(k)
                act = k >= start and blk[k][1] != 0
                if act:
                    # the kernel bounds the floor errors before step k by EU k
                    ok = (not bad[k]) and LB + h - M1 >= (1 << (HB - 1)) and \
                        LB + err + EU * k + h + EU <= (1 << HB)
                    if not ok:
                        fail = k
                        break
                    cnt += 1
                LB += h
            if fail is None:
                S += sum(Q[start:])
                Shi, err, par = LB, min(err + EU * G, 1 << 28), p_run
                nfast += cnt
                assert (1 << (p - 1)) <= S < (1 << p)
                break
            S += sum(Q[start:fail])
            nfast += cnt
            assert (1 << (p - 1)) <= S < (1 << p)
            st_, Mt_, Et_ = blk[fail]
            if transitions and E - Et_ < 1 and Et_ - E <= 27:
                # dominant product (|t| >= 2^(E-1)): V = S u + t lies in a binade
                # E + k (1 <= k <= 26) certified from the high-part bounds and
                # t's top 32 bits; W = S +- t/u is an integer (t is on a grid
                # >= u) and RN(V) = RN_int(W / 2^k) on the grid 2^k u
                dd = Et_ - E
                LBf = Shi + sum(hq(k) for k in range(start, fail))
                ek = err + EU * fail
                mt = Mt_ >> (p - 32)
                tl = mt << (dd - 6) if dd >= 6 else mt >> (6 - dd)
                th = tl + ((1 << (dd - 6)) if dd >= 6 else 1)
                if st_ == sg:
                    vlo, vhi = LBf + tl, LBf + ek + th
                else:
                    vlo, vhi = tl - LBf - ek, th - LBf + 1
                k = vlo.bit_length() - HB if vlo > 0 else 0
                if 1 <= k <= 26 and vhi <= (1 << (HB + k)) - 1:
                    W = S + (Mt_ << dd) if st_ == sg else (Mt_ << dd) - S
                    q = W >> k
                    rb = (W >> (k - 1)) & 1
                    sticky = (W & ((1 << (k - 1)) - 1)) != 0
                    S = q + (rb & (1 if sticky else (q & 1)))
                    sg, E = st_, E + k
                    Shi, err = (vlo >> k) - 1, (vhi >> k) - (vlo >> k) + 3
                    par = S & 1
                    assert (1 << (p - 1)) <= S < (1 << p)
                    assert Shi <= hi(S) < Shi + err
                    if stats is not None:
                        stats["dom"] = stats.get("dom", 0) + 1
                    start = fail + 1
                    continue
            if transitions and not bad[fail]:
                LBf = Shi + sum(hq(k) for k in range(start, fail))
                hf = hq(fail)
                ek = err + EU * fail
                st, Mt, Et = blk[fail]
                d = min(E - Et, 32 * L + 32)
                Y, rem = Mt >> d, Mt & ((1 << d) - 1)
                LO, HI = 1 << (HB - 1), 1 << HB
                if st == sg and LBf + hf - M1 >= HI:             # up: grid 2u
                    W = S + Y
                    inc = (W & 1) & (1 if (rem != 0 or (W >> 1) & 1) else 0)
                    S = (W >> 1) + inc
                    E += 1
                    Shi, err = (LBf + hf - 1) >> 1, ((ek + 2 + EU) >> 1) + 2
                    par = S & 1                                  # (the kernel reads it off R)
                    assert (1 << (p - 1)) <= S < (1 << p)
                    assert Shi <= hi(S) and hi(S) < Shi + err
                    if stats is not None:
                        stats["up"] = stats.get("up", 0) + 1
                    start = fail + 1
                    continue
                if st != sg and LBf + ek + hf + 1 + EU <= LO and LBf + hf - M1 >= LO // 2:   # down: u/2
                    b1 = (rem >> (d - 1)) & 1
                    b2 = (rem >> (d - 2)) & 1 if d >= 2 else 0
                    low = rem & ((1 << (d - 1)) - 1)
                    I = 2 * S - (2 * Y + b1)
                    if low == 0:
                        S = I
                    else:
                        tie2 = b2 == 1 and (low & ((1 << max(d - 2, 0)) - 1)) == 0
                        up = (b2 == 0) or (tie2 and b1 == 0)
                        S = I - 1 + (1 if up else 0)
                    E -= 1
                    Shi, err = 2 * (LBf + hf - M1) - 2, 2 * (ek + 1 + EU) + 4
                    par = S & 1
                    assert (1 << (p - 1)) <= S < (1 << p)
                    assert Shi <= hi(S) and hi(S) < Shi + err
                    if stats is not None:
                        stats["down"] = stats.get("down", 0) + 1
                    start = fail + 1
                    continue
            if stats is not None:
                stats["exact"] = stats.get("exact", 0) + 1
            r = oracle.add((sg, S, E), blk[fail], p)
            sg, S, E = r
            zero = S == 0
            Shi, err, par = (hi(S) if not zero else 0), 1, S & 1
            start = fail + 1
    return ((0, 0, 0) if zero else (sg, S, E)), nfast


def oracle_chain(ts, p):
    s = oracle.ZERO
    for t in ts:
        s = oracle.add(s, t, p)
    return s


def _rand_t(rng, p, elo, ehi):
    return (rng.getrandbits(1), (1 << (p - 1)) | rng.getrandbits(p - 1), rng.randint(elo, ehi))


@pytest.mark.parametrize("p", [32, 64, 256])
def test_block_sum_random_rows(p):
    rng = random.Random(p + 1)
    tot_fast = tot = 0
    for trial in range(40):
        n = rng.choice([1, 5, 31, 32, 33, 200, 700])
        ts = [_rand_t(rng, p, -64, 64) for _ in range(n)]
        got, nf = block_sum_chain(ts, p)
        assert got == oracle_chain(ts, p), (trial, n)
        tot_fast += nf
        tot += n
    assert tot_fast > 0.8 * tot        # the fast path carries the long rows


@pytest.mark.parametrize("p", [32, 64, 128])
def test_block_sum_ties_cancellation_and_zeros(p):
    """Products engineered to tie on the accumulator's grid (d small, low bits
    10...0), to cancel the accumulator exactly mid-row, zero products, and
    binade crossings in both directions."""
    rng = random.Random(3 * p)
    for trial in range(150):
        ts = []
        s_e = rng.randint(0, 8)
        for k in range(rng.choice([8, 40, 100])):
            kind = rng.random()
            if kind < 0.25:        # tie-prone: few low bits set, exponent just below
                d = rng.randint(1, 4)
                M = (1 << (p - 1)) | (1 << (d - 1)) | (rng.getrandbits(p - 1 - d) << d)
                ts.append((rng.getrandbits(1), M, s_e - d + rng.randint(-1, 1)))
            elif kind < 0.35:
                ts.append((0, 0, 0))                      # zero product
            elif kind < 0.45 and ts:
                prev = oracle_chain(ts, p)                # exact cancellation
                if prev[1]:
                    ts.append((prev[0] ^ 1, prev[1], prev[2]))
                    continue
                ts.append(_rand_t(rng, p, s_e - 3, s_e + 3))
            else:
                ts.append(_rand_t(rng, p, s_e - 6, s_e + 2))
        got, _ = block_sum_chain(ts, p, G=rng.choice([4, 32]))
        assert got == oracle_chain(ts, p), trial
        got, _ = block_sum_chain(ts, p, G=rng.choice([64, 128]), ties_exact=True)
        assert got == oracle_chain(ts, p), ("ties exact", trial)


@pytest.mark.parametrize("p", [32, 64, 128, 256])
def test_block_sum_one_binade_transitions(p):
    """Random walks (random signs, similar magnitudes) cross binade boundaries
    all the time: most crossings must be taken by the one-binade transitions,
    and every result must still be the ordered chain's."""
    rng = random.Random(11 * p)
    st = {}
    for trial in range(30):
        n = rng.choice([200, 600, 1500])
        ts = [_rand_t(rng, p, -3, 3) for _ in range(n)]
        got, _ = block_sum_chain(ts, p, transitions=True, stats=st)
        assert got == oracle_chain(ts, p), trial
        got, _ = block_sum_chain(ts, p, G=rng.choice([4, 32]), transitions=True, ties_exact=True,
                                 stats=st)
        assert got == oracle_chain(ts, p), ("ties exact", trial)
        got, _ = block_sum_chain(ts, p, transitions=True, herr2=True)   # round-2 consume
        assert got == oracle_chain(ts, p), ("herr2", trial)
    assert st.get("up", 0) > 0 and st.get("down", 0) > 0
    assert 2 * (st.get("up", 0) + st.get("down", 0)) > st.get("exact", 0)


@pytest.mark.parametrize("p", [32, 64])
def test_block_sum_transitions_adversarial(p):
    """Tie-prone products and exact cancellations with the transitions on."""
    rng = random.Random(5 * p)
    for trial in range(120):
        ts = []
        s_e = rng.randint(0, 8)
        for k in range(rng.choice([8, 40, 100])):
            kind = rng.random()
            if kind < 0.3:
                d = rng.randint(1, 4)
                M = (1 << (p - 1)) | (1 << (d - 1)) | (rng.getrandbits(p - 1 - d) << d)
                ts.append((rng.getrandbits(1), M, s_e - d + rng.randint(-1, 1)))
            elif kind < 0.4:
                ts.append((0, 0, 0))
            else:
                ts.append(_rand_t(rng, p, s_e - 3, s_e + 1))
        got, _ = block_sum_chain(ts, p, G=rng.choice([4, 32]), transitions=True)
        assert got == oracle_chain(ts, p), trial
        got, _ = block_sum_chain(ts, p, transitions=True, herr2=True)
        assert got == oracle_chain(ts, p), ("herr2", trial)
        # 64 steps per warp pass, grid ties sent to the exact path,
        # transitions on (the U = 2 variant)
        got, _ = block_sum_chain(ts, p, G=64, transitions=True, ties_exact=True)
        assert got == oracle_chain(ts, p), ("U=2", trial)


@pytest.mark.parametrize("p", [32, 64, 256])
def test_block_sum_dominant_transitions(p):
    """Wide exponent ranges (C4: products of exponents U[-32,32]): most exact-
    path steps are a new product that dominates the running sum (|t| >=
    2^(E-1)); they must be taken by the dominant-product transition, and every
    result must be the ordered chain's - including near-cancelling opposite
    products, exact ties on the coarser grid and jumps of up to 30 binades."""
    rng = random.Random(17 * p)
    st = {}
    for trial in range(40):
        n = rng.choice([50, 300, 900])
        ts = []
        for k in range(n):
            kind = rng.random()
            if kind < 0.08 and ts:
                s = oracle_chain(ts, p)
                if s[1]:
                    # opposite sign, slightly larger: |V| small or a binade down
                    M = s[1] + rng.randint(1, 1 << max(p - 8, 1))
                    if M < (1 << p):
                        ts.append((s[0] ^ 1, M, s[2]))
                        continue
            if kind < 0.14 and ts:
                s = oracle_chain(ts, p)
                if s[1]:
                    # same or opposite sign, 2..30 binades up, low bits 0 or 10..0
                    dd = rng.randint(2, 30)
                    M = (1 << (p - 1)) | (rng.getrandbits(p - 1) & ~((1 << rng.randint(0, 6)) - 1))
                    ts.append((rng.getrandbits(1), M, s[2] + dd))
                    continue
            ts.append(_rand_t(rng, p, -40, 40))
        got, _ = block_sum_chain(ts, p, G=rng.choice([4, 32]), transitions=True, stats=st)
        assert got == oracle_chain(ts, p), trial
        got, _ = block_sum_chain(ts, p, G=64, transitions=True, ties_exact=True)
        assert got == oracle_chain(ts, p), ("U=2", trial)
        got, _ = block_sum_chain(ts, p, transitions=True, herr2=True)
        assert got == oracle_chain(ts, p), ("herr2", trial)
    assert st.get("dom", 0) > 0
    # C4-like rows (products of values with exponents U[-32, 32]): the
    # dominant transition takes most of what used to be exact-path steps
    st = {}
    for trial in range(6):
        ts = [oracle.mul(_rand_t(rng, p, -32, 32), _rand_t(rng, p, -32, 32), p)
              for _ in range(rng.choice([300, 1000]))]
        got, _ = block_sum_chain(ts, p, transitions=True, stats=st)
        assert got == oracle_chain(ts, p), ("c4-like", trial)
    assert st.get("dom", 0) > 2 * st.get("exact", 0)


@pytest.mark.parametrize("p,D", [(128, 2), (256, 2), (1024, 2), (256, 3), (1024, 3)])
def test_short_product_zero_low_limbs_is_exact(p, D):
    """mp_mul's exact case: when either operand's limbs 0 .. K0-1 (K0 = L-D)
    are all zero, every omitted Comba term a_i x_j (i + j < K0) is zero, so
    the upper columns T are the exact product and rounding T directly (round
    bit and sticky read from T) equals RN(a*x) - e.g. C5's diagonal 4
    (M = 2^(p-1)), whose products the certificate cannot decide (all-zero
    bits below the round bit)."""
    L = p // 32
    K0 = L - D
    rng = random.Random(p + 99)
    for _ in range(400):
        hi_bits = 32 * (L - K0)
        Ma = ((1 << (hi_bits - 1)) | rng.getrandbits(hi_bits - 1)) << (32 * K0)
        if rng.random() < 0.3:
            Ma = 1 << (p - 1)
        Mx = (1 << (p - 1)) | rng.getrandbits(p - 1)
        if rng.random() < 0.5:
            Ma, Mx = Mx, Ma
        a = [(Ma >> (32 * i)) & M32 for i in range(L)]
        x = [(Mx >> (32 * i)) & M32 for i in range(L)]
        T = sum(a[i] * x[j] << (32 * (i + j)) for i in range(L) for j in range(L) if i + j >= K0)
        assert T == Ma * Mx
        sh = 0 if (T >> (2 * p - 1)) & 1 else 1
        q = T >> (p - sh)
        rb = (T >> (p - sh - 1)) & 1
        sticky = (T & ((1 << (p - sh - 1)) - 1)) != 0
        q += rb & (1 if sticky else (q & 1))
        dE = -sh
        if q == 1 << p:
            q >>= 1
            dE += 1
        s, M, E = oracle.mul((0, Ma, 0), (0, Mx, 0), p)
        assert (M, E) == (q, dE)
