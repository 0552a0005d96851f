"""Independent references used to pin the oracle (tests only).

None of these reuse oracle code:
  * MPFR (libmpfr.so.6 through ctypes): mpfr_mul / mpfr_add with MPFR_RNDN,
    the library routine the paper's BNCpack is built on.
  * mpmath.libmp: mpf_mul / mpf_add with rnd='n' (pure-Python big-float).
  * Fraction: exact rational value followed by ONE correct rounding, computed
    by binade search with rational comparisons (no bit_length / shifting).
"""
from __future__ import annotations

import ctypes
import ctypes.util
from fractions import Fraction

ZERO = (0, 0, 0)


# ---------------------------------------------------------------- Fraction
def to_frac(v, p):
    s, M, E = v
    if M == 0:
        return Fraction(0)
    val = Fraction(M) * (Fraction(2) ** (E - p))
    return -val if s else val


def frac_round(v: Fraction, p: int):
    """Correct RNE rounding of a rational to p bits -> triple (s, M, E)."""
    if v == 0:
        return ZERO
    s = 1 if v < 0 else 0
    a = -v if s else v
    # binade: 2^(E-1) <= a < 2^E, found by comparisons only
    E = 0
    while a >= Fraction(2) ** E:
        E += 1
    while a < Fraction(2) ** (E - 1):
        E -= 1
    scaled = a * Fraction(2) ** (p - E)          # in [2^(p-1), 2^p)
    q = scaled.numerator // scaled.denominator
    rem = scaled - q
    half = Fraction(1, 2)
    if rem > half or (rem == half and q % 2 == 1):
        q += 1
    if q == 2 ** p:
        q = 2 ** (p - 1)
        E += 1
    return (s, q, E)


# ---------------------------------------------------------------- mpmath
def mpmath_ops():
    import mpmath.libmp as lm

    def to_mpf(v, p):
        s, M, E = v
        if M == 0:
            return lm.fzero
        return lm.from_man_exp(-M if s else M, E - p)

    def from_mpf(t, p):
        if t == lm.fzero:
            return ZERO
        sign, man, exp, bc = t
        man = int(man)
        b = man.bit_length()
        return (int(sign), man << (p - b), exp + b)

    def mul(a, b, p):
        return from_mpf(lm.mpf_mul(to_mpf(a, p), to_mpf(b, p), p, 'n'), p)

    def add(a, b, p):
        return from_mpf(lm.mpf_add(to_mpf(a, p), to_mpf(b, p), p, 'n'), p)

    return mul, add


# ---------------------------------------------------------------- MPFR
class _MPFR(ctypes.Structure):
    _fields_ = [("prec", ctypes.c_long), ("sign", ctypes.c_int),
                ("exp", ctypes.c_long), ("d", ctypes.POINTER(ctypes.c_uint64))]


class MPFR:
    """Minimal ctypes wrapper around libmpfr (no headers needed)."""

    def __init__(self):
        name = ctypes.util.find_library("mpfr") or "libmpfr.so.6"
        self.lib = ctypes.CDLL(name)
        lib = self.lib
        lib.mpfr_get_emin_min.restype = ctypes.c_long
        lib.mpfr_get_emax_max.restype = ctypes.c_long
        lib.mpfr_set_emin.argtypes = [ctypes.c_long]
        lib.mpfr_set_emax.argtypes = [ctypes.c_long]
        lib.mpfr_set_emin(lib.mpfr_get_emin_min())
        lib.mpfr_set_emax(lib.mpfr_get_emax_max())
        lib.mpfr_zero_p.restype = ctypes.c_int

    def _new(self, p):
        x = _MPFR()
        self.lib.mpfr_init2(ctypes.byref(x), ctypes.c_long(p))
        return x

    def _set(self, x, v, p):
        s, M, E = v
        if M == 0:
            self.lib.mpfr_set_zero(ctypes.byref(x), 1)
            return
        txt = ("-" if s else "") + format(M, "x") + "p" + str(E - p)
        rc = self.lib.mpfr_set_str(ctypes.byref(x), txt.encode(), 16, 0)
        assert rc == 0, txt

    def _get(self, x, p):
        if self.lib.mpfr_zero_p(ctypes.byref(x)):
            return ZERO
        nl = (p + 63) // 64
        M = 0
        for i in range(nl):
            M |= int(x.d[i]) << (64 * i)
        M >>= (64 * nl - p)
        return (1 if x.sign < 0 else 0, M, int(x.exp))

    def op(self, name, a, b, p):
        xa, xb, xr = self._new(p), self._new(p), self._new(p)
        try:
            self._set(xa, a, p)
            self._set(xb, b, p)
            getattr(self.lib, name)(ctypes.byref(xr), ctypes.byref(xa), ctypes.byref(xb), 0)  # RNDN
            r = self._get(xr, p)
        finally:
            for x in (xa, xb, xr):
                self.lib.mpfr_clear(ctypes.byref(x))
        # MPFR keeps signed zeros (e.g. (-3)*(+0) = -0); the build's zero is +0
        return ZERO if r[1] == 0 else r

    def mul(self, a, b, p):
        return self.op("mpfr_mul", a, b, p)

    def add(self, a, b, p):
        return self.op("mpfr_add", a, b, p)


def try_mpfr():
    try:
        return MPFR()
    except OSError:
        return None
