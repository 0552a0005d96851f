"""CPU oracle for the MP BiCG solver.

TEST INFRASTRUCTURE ONLY (same rules as oracle/mpref.py: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may use
it; it shares no code with the CUDA path).

What it computes - PAPER.md:249-297 (Fig. 4, BiCG), without preconditioning
(K = I, so w = r and w~ = r~), and PAPER.md:375-380 (b = A [1..n]^T computed in
multiple precision; convergence test ||r_k||_2 <= 1e-20 ||r_0||_2 + 1e-50):

    x_0 = 0, r_0 = b - A x_0 = b, r~_0 = r_0
    for i = 1, 2, ...
        rho_{i-1} = (r~_{i-1}, r_{i-1});  rho = 0 -> breakdown exit
        i = 1: p_1 = r_0, p~_1 = r~_0
        else:  beta = rho_{i-1} / rho_{i-2}
               p_i = r_{i-1} + beta p_{i-1};  p~_i = r~_{i-1} + beta p~_{i-1}
        z_i = A p_i;  z~_i = A^T p~_i                     (reading c3)
        sigma = (p~_i, z_i);  sigma = 0 -> breakdown exit
        alpha = rho_{i-1} / sigma
        x_i = x_{i-1} + alpha p_i;  r_i = r_{i-1} - alpha z_i;  r~_i = r~_{i-1} - alpha z~_i
        converged iff ||r_i|| <= c1 ||r_0|| + c2

Readings (c26-c31): every operation is one p-bit RN
operation in the order written; a dot product (u, v) is the ordered chain
s = RN(s + RN(u_k v_k)), k ascending, from +0 (BNCpack-style loop, like a
matrix row); "a + beta b" is RN(a + RN(beta b)) and "a - alpha b" is
RN(a + RN(-(alpha b))); ||v|| = RN(sqrt((v, v))); c1 = RN(10^-20),
c2 = RN(10^-50) (correctly rounded constants); the test is
||r_i|| <= RN(RN(c1 ||r_0||) + c2); the paper's "p~_i = w~_i + ..." is read as
w~_{i-1} (index typo).
"""
from __future__ import annotations

import math

from .mpref import ZERO, add, mul, rn, spmv, spmv_t, unpack_vec, pack_vec


def neg(a):
    s, M, E = a
    return ZERO if M == 0 else (s ^ 1, M, E)


def from_int(k: int, p: int):
    """RN_p of an integer."""
    if k == 0:
        return ZERO
    M, E = rn(abs(k), 0, p)
    return (1 if k < 0 else 0, M, E)


def div(a, b, p: int):
    """RN_p(a / b); b must be nonzero.  Exact integer quotient with p+3 bits
    and a sticky bit, then one rounding (the definition of correct rounding)."""
    sa, Ma, Ea = a
    sb, Mb, Eb = b
    if Mb == 0:
        raise ZeroDivisionError("MP division by zero")
    if Ma == 0:
        return ZERO
    K = p + 3
    q, r = divmod(Ma << K, Mb)                  # Ma/Mb in (1/2, 2): q has K or K+1 bits
    N = (q << 1) | (1 if r else 0)
    M, E = rn(N, Ea - Eb - K - 1, p)
    return (sa ^ sb, M, E)


def sqrt(a, p: int):
    """RN_p(sqrt(a)), a >= 0.  Exact integer square root with p+3 bits and a
    sticky bit, then one rounding."""
    s, M, E = a
    if M == 0:
        return ZERO
    if s:
        raise ValueError("MP sqrt of a negative number")
    e = E - p                                   # value = M * 2^e
    if e & 1:
        M <<= 1
        e -= 1
    K = p // 2 + 3
    X = M << (2 * K)                            # value = X * 2^(e - 2K)
    N = math.isqrt(X)
    N2 = (N << 1) | (1 if N * N != X else 0)
    Mr, Er = rn(N2, e // 2 - K - 1, p)
    return (0, Mr, Er)


def recip_pow10(k: int, p: int):
    """RN_p(10^-k), correctly rounded."""
    K = p + 3 + 4 * k
    q, r = divmod(1 << K, 10 ** k)
    N = (q << 1) | (1 if r else 0)
    M, E = rn(N, -K - 1, p)
    return (0, M, E)


def cmp(a, b) -> int:
    """Exact comparison of two values: -1, 0 or 1 (normalised mantissas, so
    (E, M) orders magnitudes lexicographically)."""
    def sgn(v):
        return 0 if v[1] == 0 else (-1 if v[0] else 1)
    ga, gb = sgn(a), sgn(b)
    if ga != gb:
        return -1 if ga < gb else 1
    if ga == 0:
        return 0
    ka, kb = (a[2], a[1]), (b[2], b[1])
    c = (ka > kb) - (ka < kb)
    return c if ga > 0 else -c


def le(a, b) -> bool:
    return cmp(a, b) <= 0


def dot(u, v, p: int):
    """(u, v) = ordered chain s = RN(s + RN(u_k v_k)), k ascending, from +0."""
    s = ZERO
    for a, b in zip(u, v):
        s = add(s, mul(a, b, p), p)
    return s


def axpy(alpha, x, y, p: int, negate: bool = False):
    """y_k + alpha x_k (negate: y_k - alpha x_k), each as RN(y + RN(+-alpha x))."""
    al = neg(alpha) if negate else alpha
    return [add(yk, mul(al, xk, p), p) for xk, yk in zip(x, y)]


def norm2(v, p: int):
    return sqrt(dot(v, v, p), p)


def _spmv_list(p, A, vec, transpose=False):
    rowptr, colidx, limbs, exps, signs = A
    xl, xe, xs = pack_vec(vec, p)
    f = spmv_t if transpose else spmv
    yl, ye, ys = f(p, rowptr, colidx, limbs, exps, signs, xl, xe, xs)
    return unpack_vec(yl, ye, ys, p)


def bicg(p: int, A, b, max_iter: int, trace: bool = False):
    """Fig. 4 BiCG (K = I) from x_0 = 0.  A = (rowptr, colidx, limbs, exps,
    signs) packed; b = list of triples.  Returns a dict with x (triples), the
    iteration count, the status ("converged" | "breakdown" | "max_iter"), the
    residual norms, and (trace=True) every iteration's rho, alpha, beta."""
    n = len(b)
    c1, c2 = recip_pow10(20, p), recip_pow10(50, p)
    x = [ZERO] * n
    r = list(b)
    rt = list(r)
    nrm0 = norm2(r, p)
    thr = add(mul(c1, nrm0, p), c2, p)
    norms = [nrm0]
    hist = []
    rho_prev = None
    pv = pt = None
    status = "max_iter"
    it = 0
    for i in range(1, max_iter + 1):
        rho = dot(rt, r, p)
        if rho[1] == 0:
            status = "breakdown"
            break
        if i == 1:
            pv, pt = list(r), list(rt)
            beta = None
        else:
            beta = div(rho, rho_prev, p)
            pv = axpy(beta, pv, r, p)
            pt = axpy(beta, pt, rt, p)
        z = _spmv_list(p, A, pv)
        zt = _spmv_list(p, A, pt, transpose=True)
        sigma = dot(pt, z, p)
        if sigma[1] == 0:
            status = "breakdown"
            break
        alpha = div(rho, sigma, p)
        x = axpy(alpha, pv, x, p)
        r = axpy(alpha, z, r, p, negate=True)
        rt = axpy(alpha, zt, rt, p, negate=True)
        nrm = norm2(r, p)
        norms.append(nrm)
        it = i
        if trace:
            hist.append(dict(rho=rho, beta=beta, sigma=sigma, alpha=alpha, nrm=nrm))
        rho_prev = rho
        if le(nrm, thr):
            status = "converged"
            break
    return dict(x=x, iters=it, status=status, norms=norms, thr=thr, hist=hist)


# --------------------------------------------------------------------------
# GPBiCG (Fig. 4 right), K = I, over the reals (mu4-bar =
# mu4).  Readings (DESIGN.md c32-c35): u = z = 0, x_0 = 0, r~ = r_0 = b;
# every compound update is evaluated left to right as a chain of single RN
# operations (sub(a, b) = RN(a - b), scal(c, a) = RN(c a), axpy as above):
#   beta = RN(RN(rho/rho_prev) * RN(alpha_prev/zeta))
#   w = v + beta q;  p = r + beta (p - u);  s = t - r;  t = r - alpha q
#   y = s - alpha (w - q)    (i = 1: y = RN(alpha q) - r)
#   tau = RN(RN(mu5 mu1) - RN(mu4 mu4))
#   zeta = RN(RN(RN(mu1 mu2) - RN(mu3 mu4)) / tau)
#   eta  = RN(RN(RN(mu5 mu3) - RN(mu4 mu2)) / tau)
#   (i = 1: zeta = mu2/mu5, or 0 when mu5 = 0 (then t = 0), eta = 0)
#   u = RN(RN(zeta q) + RN(eta RN(s + RN(beta u))))   (i = 1: u = RN(zeta q))
#   z = RN(RN(RN(zeta r) + RN(eta z)) - RN(alpha u))
#   x = RN(RN(x + RN(alpha p)) + z)
#   r = RN(RN(t - RN(eta y)) - RN(zeta v))
# The figure prints "z = zeta r + zeta z - alpha u" and "r = t - eta y -
# zeta u"; read literally the method does not converge (a diagonally dominant
# band where BiCG converges in 39 iterations stalls for 200); these are read as
# the typos of Zhang's GPBiCG (1997), which the paper implements: eta z and
# zeta v (v = A t).
# The figure's convergence check (*) sits before r_i is formed; it is applied
# to r_i (the residual it tests).  Breakdown: rho = 0, (r~, q) = 0, tau = 0,
# or zeta = 0 for an iteration that did not converge.
# --------------------------------------------------------------------------

def sub(a, b, p):
    return [add(x, neg(y), p) for x, y in zip(a, b)]


def scal(c, a, p):
    return [mul(c, x, p) for x in a]


def vadd(a, b, p):
    return [add(x, y, p) for x, y in zip(a, b)]


def gpbicg(p: int, A, b, max_iter: int, trace: bool = False):
    n = len(b)
    c1, c2 = recip_pow10(20, p), recip_pow10(50, p)
    x = [ZERO] * n
    r = list(b)
    rt = list(r)
    u = [ZERO] * n
    z = [ZERO] * n
    nrm0 = norm2(r, p)
    thr = add(mul(c1, nrm0, p), c2, p)
    norms = [nrm0]
    hist = []
    status, it = "max_iter", 0
    rho_prev = alpha_prev = zeta = beta = None
    pv = t = w = q = v = s = y = None
    for i in range(1, max_iter + 1):
        rho = dot(rt, r, p)
        if rho[1] == 0:
            status = "breakdown"
            break
        if i == 1:
            pv = list(r)
            q = _spmv_list(p, A, pv)
            sq = dot(rt, q, p)
            if sq[1] == 0:
                status = "breakdown"
                break
            alpha = div(rho, sq, p)
            t = axpy(alpha, q, r, p, negate=True)
            v = _spmv_list(p, A, t)
            y = sub(scal(alpha, q, p), r, p)
            mu2, mu5 = dot(v, t, p), dot(v, v, p)
            zeta = ZERO if mu5[1] == 0 else div(mu2, mu5, p)
            eta = ZERO
            u = scal(zeta, q, p)
        else:
            beta = mul(div(rho, rho_prev, p), div(alpha_prev, zeta, p), p)
            w = axpy(beta, q, v, p)
            pv = axpy(beta, sub(pv, u, p), r, p)
            q = _spmv_list(p, A, pv)
            sq = dot(rt, q, p)
            if sq[1] == 0:
                status = "breakdown"
                break
            alpha = div(rho, sq, p)
            s = sub(t, r, p)
            t = axpy(alpha, q, r, p, negate=True)
            v = _spmv_list(p, A, t)
            y = axpy(alpha, sub(w, q, p), s, p, negate=True)
            mu1, mu2, mu3 = dot(y, y, p), dot(v, t, p), dot(y, t, p)
            mu4, mu5 = dot(v, y, p), dot(v, v, p)
            tau = add(mul(mu5, mu1, p), neg(mul(mu4, mu4, p)), p)
            if tau[1] == 0:
                status = "breakdown"
                break
            zeta = div(add(mul(mu1, mu2, p), neg(mul(mu3, mu4, p)), p), tau, p)
            eta = div(add(mul(mu5, mu3, p), neg(mul(mu4, mu2, p)), p), tau, p)
            u = axpy(eta, axpy(beta, u, s, p), scal(zeta, q, p), p)
        z = axpy(alpha, u, vadd(scal(zeta, r, p), scal(eta, z, p), p), p, negate=True)
        x = vadd(axpy(alpha, pv, x, p), z, p)
        r = axpy(zeta, v, axpy(eta, y, t, p, negate=True), p, negate=True)
        nrm = norm2(r, p)
        norms.append(nrm)
        it = i
        if trace:
            hist.append(dict(rho=rho, alpha=alpha, zeta=zeta, eta=eta, beta=beta, nrm=nrm))
        rho_prev, alpha_prev = rho, alpha
        if le(nrm, thr):
            status = "converged"
            break
        if zeta[1] == 0:
            status = "breakdown"
            break
    return dict(x=x, iters=it, status=status, norms=norms, thr=thr, hist=hist)
