// mp_device.cuh - p-bit binary floating-point arithmetic with round-to-
// nearest-even, as sm_100a device functions.  L = p/32 uint32 limbs.
//
// Semantics (BASELINE.json north_star):
//   value = (-1)^s * M/2^p * 2^e,  2^(p-1) <= M < 2^p, zero <=> M == 0.
//   mp_mul: t = RN(a * x)        (exact 2L-limb product, one rounding)
//   mp_add: s = RN(s + t)        (exact alignment with a guard limb + sticky,
//                                 one rounding; exact zero -> +0)
// Everything is held in registers; all limb loops are fully unrolled so the
// arrays never touch local memory.  Shares no code with the CPU reference.
#pragma once
#include <cstdint>

namespace mpsp {

// --------------------------------------------------------------------------
// Comba multiply-accumulate step: (c2:c1:c0) += a*b.  ptxas fuses the
// mad.lo.cc / madc.hi.cc pair into one IMAD.WIDE.U32 with a carry-out
// predicate, and pairs of carries into one IADD3.X.
// --------------------------------------------------------------------------
__device__ __forceinline__ void mac3(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                     uint32_t a, uint32_t b) {
  asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"
      "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"
      "addc.u32 %2, %2, 0;"
      : "+r"(c0), "+r"(c1), "+r"(c2)
      : "r"(a), "r"(b));
}

// --------------------------------------------------------------------------
// Carry-chain helpers (PTX add.cc/addc/sub.cc/subc: one instruction per limb;
// the chains are emitted in order by consecutive asm volatile statements).
// --------------------------------------------------------------------------
// z = x + y (N limbs); returns the carry out (0/1)
template <int N>
__device__ __forceinline__ uint32_t add_n(uint32_t (&z)[N], const uint32_t (&x)[N],
                                          const uint32_t (&y)[N]) {
  uint32_t c;
  asm volatile("add.cc.u32 %0, %1, %2;" : "=r"(z[0]) : "r"(x[0]), "r"(y[0]));
#pragma unroll
  for (int i = 1; i < N; ++i)
    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(z[i]) : "r"(x[i]), "r"(y[i]));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
  return c;
}
// z = x - y - b0 (N limbs, b0 in {0,1}); returns the borrow out (0/1)
template <int N>
__device__ __forceinline__ uint32_t sub_n(uint32_t (&z)[N], const uint32_t (&x)[N],
                                          const uint32_t (&y)[N], uint32_t b0) {
  uint32_t b, dummy;
  // set the carry flag to b0 via 0 - b0 (borrow iff b0 = 1)
  asm volatile("sub.cc.u32 %0, 0, %1;" : "=r"(dummy) : "r"(b0));
#pragma unroll
  for (int i = 0; i < N; ++i)
    asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(z[i]) : "r"(x[i]), "r"(y[i]));
  asm volatile("subc.u32 %0, 0, 0;" : "=r"(b));
  return b & 1u;
}
// borrow of x - y (N limbs) without storing the difference: 1 iff x < y
template <int N>
__device__ __forceinline__ uint32_t lt_n(const uint32_t (&x)[N], const uint32_t (&y)[N]) {
  uint32_t b, d;
  asm volatile("sub.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(x[0]), "r"(y[0]));
#pragma unroll
  for (int i = 1; i < N; ++i)
    asm volatile("subc.cc.u32 %0, %1, %2;" : "=r"(d) : "r"(x[i]), "r"(y[i]));
  asm volatile("subc.u32 %0, 0, 0;" : "=r"(b));
  return b & 1u;
}
// m += inc (inc in {0,1}); returns the carry out of the top limb
template <int N>
__device__ __forceinline__ uint32_t inc_n(uint32_t (&m)[N], uint32_t inc) {
  uint32_t c;
  asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(m[0]) : "r"(inc));
#pragma unroll
  for (int i = 1; i < N; ++i) asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(m[i]));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
  return c;
}

// Register-resident MP number.  m[L-1] == 0 <=> zero.
template <int L>
struct MP {
  uint32_t m[L];
  int32_t e;
  uint32_t s;
  __device__ __forceinline__ bool is_zero() const { return m[L - 1] == 0u; }
  __device__ __forceinline__ void set_zero() {
#pragma unroll
    for (int i = 0; i < L; ++i) m[i] = 0u;
    e = 0;
    s = 0u;
  }
};

// Round-to-nearest-even increment of an L-limb mantissa given round bit and
// sticky.  Returns the carry out of the top limb (mantissa became 2^p; the
// caller renormalises to 2^(p-1) and bumps the exponent).
// The increment reaches limb 1 only when limb 0 was all ones (2^-32 per
// lane): limb 0 is incremented inline and the carry propagated through the
// other limbs in a warp-uniform branch (FW: every lane of the warp is here).
// Measured: C4 A^T -2.4%, C4 A x -1.1%, C5 -0.7%; at L = 16 the branch
// costs the 128-register SELL kernel spills (C3 +5%), so L = 16 keeps the
// inline chain.
template <int L, bool FW = false>
__device__ __forceinline__ uint32_t rne_increment(uint32_t (&m)[L], uint32_t rb, uint32_t sticky) {
  const uint32_t inc = rb & ((sticky != 0u) | (m[0] & 1u));
  if constexpr (L <= 2 || L == 16) {
    return inc_n<L>(m, inc);
  } else {
    uint32_t c;
    asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(m[0]) : "r"(inc));
    asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
    uint32_t cy = 0u;
    if (__any_sync(FW ? 0xffffffffu : __activemask(), c != 0u)) {
      asm volatile("add.cc.u32 %0, %0, %1;" : "+r"(m[1]) : "r"(c));
#pragma unroll
      for (int i = 2; i < L; ++i) asm volatile("addc.cc.u32 %0, %0, 0;" : "+r"(m[i]));
      asm volatile("addc.u32 %0, 0, 0;" : "=r"(cy));
    }
    return cy;
  }
}

// (a2:a1:a0) += (b2:b1:b0)
__device__ __forceinline__ void add3w(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t b0,
                                      uint32_t b1, uint32_t b2) {
  asm("add.cc.u32 %0, %0, %3;\n\t"
      "addc.cc.u32 %1, %1, %4;\n\t"
      "addc.u32 %2, %2, %5;"
      : "+r"(a0), "+r"(a1), "+r"(a2)
      : "r"(b0), "r"(b1), "r"(b2));
}

// Independent accumulation chains per Comba column: the IMAD.WIDE of one
// chain depends on the previous one through its 64-bit addend, so a single
// chain per column serialises the whole product; NCH chains (merged at the
// end of the column) give the scheduler NCH-way ILP at 3 adds per extra chain.
// (measured on B200: round 1 found 2 chains best at L = 16, 32; with the
// column-(L-2) short product and the final adder 1 chain is best everywhere:
// C3 217 -> 214 us, C5 1668 -> 1664 us; 3 chains: 227 / 1751)
#ifndef MPSP_NCH
#define MPSP_NCH 1
#endif
#ifndef MPSP_NCH8
#define MPSP_NCH8 1
#endif
#ifndef MPSP_NCH16
#define MPSP_NCH16 MPSP_NCH
#endif
template <int L>
struct MulChains {
  static constexpr int n = L >= 32 ? MPSP_NCH : (L >= 16 ? MPSP_NCH16 : (L >= 4 ? MPSP_NCH8 : 1));
};

// --------------------------------------------------------------------------
// t = RN_p(a * x).  a, x: L-limb mantissas (zero allowed: result zero).
// Exponent of the result: ea + ex (top product bit set) or ea + ex - 1,
// +1 if rounding carried out.
// --------------------------------------------------------------------------
template <int L>
__device__ __forceinline__ void mp_mul_full(const uint32_t (&a)[L], int32_t ea, uint32_t sa,
                                            const uint32_t (&x)[L], int32_t ex, uint32_t sx,
                                            MP<L>& t) {
  constexpr int NCH = MulChains<L>::n;
  uint32_t c0 = 0u, c1 = 0u, c2 = 0u;
  uint32_t sticky = 0u, w = 0u;
  uint32_t P[L];
#pragma unroll
  for (int k = 0; k < 2 * L - 1; ++k) {
    const int ilo = k - (L - 1) > 0 ? k - (L - 1) : 0;
    const int ihi = k < L - 1 ? k : L - 1;
    const int nt = ihi - ilo + 1;                      // terms in column k
    uint32_t A0[NCH], A1[NCH], A2[NCH];
    A0[0] = c0; A1[0] = c1; A2[0] = c2;                // chain 0 carries the column-in
#pragma unroll
    for (int ch = 1; ch < NCH; ++ch) { A0[ch] = 0u; A1[ch] = 0u; A2[ch] = 0u; }
#pragma unroll
    for (int i = 0; i < L; ++i) {
      if (i < ilo || i > ihi) continue;
      const int ch = (i - ilo) % NCH;
      mac3(A0[ch], A1[ch], A2[ch], a[i], x[k - i]);
    }
#pragma unroll
    for (int ch = 1; ch < NCH; ++ch)
      if (ch < nt) add3w(A0[0], A1[0], A2[0], A0[ch], A1[ch], A2[ch]);
    if (k < L - 1) sticky |= A0[0];        // columns 0..L-2: only "nonzero?" matters
    else if (k == L - 1) w = A0[0];        // limb L-1: round bit(s) + sticky
    else P[k - L] = A0[0];                 // limbs L..2L-2 of the product
    c0 = A1[0]; c1 = A2[0]; c2 = 0u;
  }
  P[L - 1] = c0;                           // limb 2L-1
  // normalise: shift left by sh = 1 when the top product bit is clear
  const uint32_t sh = (~P[L - 1]) >> 31;
#pragma unroll
  for (int i = L - 1; i > 0; --i) t.m[i] = __funnelshift_l(P[i - 1], P[i], sh);
  t.m[0] = __funnelshift_l(w, P[0], sh);
  const uint32_t ws = w << sh;             // w's bits below the new LSB
  const uint32_t rb = ws >> 31;
  const uint32_t st = sticky | (ws << 1);
  const uint32_t cy = rne_increment<L>(t.m, rb, st);
  if (cy) t.m[L - 1] = 0x80000000u;
  t.e = ea + ex - (int32_t)sh + (int32_t)cy;
  t.s = sa ^ sx;
}

// Columns [K0, 2L-2] of the Comba product from a zero carry-in: T[m - K0] =
// limb m of  sum_{i+j >= K0} a_i x_j 2^(32(i+j))  for m in [K0, 2L-1].
template <int L, int K0>
__device__ __forceinline__ void comba_upper(const uint32_t (&a)[L], const uint32_t (&x)[L],
                                            uint32_t (&T)[2 * L - K0]) {
  constexpr int NCH = MulChains<L>::n;
  uint32_t c0 = 0u, c1 = 0u, c2 = 0u;
#pragma unroll
  for (int k = K0; k < 2 * L - 1; ++k) {
    const int ilo = k - (L - 1) > 0 ? k - (L - 1) : 0;
    const int ihi = k < L - 1 ? k : L - 1;
    const int nt = ihi - ilo + 1;
    uint32_t A0[NCH], A1[NCH], A2[NCH];
    A0[0] = c0; A1[0] = c1; A2[0] = c2;
#pragma unroll
    for (int ch = 1; ch < NCH; ++ch) { A0[ch] = 0u; A1[ch] = 0u; A2[ch] = 0u; }
#pragma unroll
    for (int i = 0; i < L; ++i) {
      if (i < ilo || i > ihi) continue;
      const int ch = (i - ilo) % NCH;
      mac3(A0[ch], A1[ch], A2[ch], a[i], x[k - i]);
    }
#pragma unroll
    for (int ch = 1; ch < NCH; ++ch)
      if (ch < nt) add3w(A0[0], A1[0], A2[0], A0[ch], A1[ch], A2[ch]);
    T[k - K0] = A0[0];
    c0 = A1[0]; c1 = A2[0]; c2 = 0u;
  }
  T[2 * L - 1 - K0] = c0;
}

// Columns [0, K0) of the Comba product: returns the OR of limbs 0..K0-1
// (sticky) and the carry (c0, c1, c2) into column K0.
template <int L, int K0>
__device__ __forceinline__ uint32_t comba_lower(const uint32_t (&a)[L], const uint32_t (&x)[L],
                                                uint32_t& c0, uint32_t& c1, uint32_t& c2) {
  uint32_t sticky = 0u;
  c0 = 0u; c1 = 0u; c2 = 0u;
#pragma unroll
  for (int k = 0; k < K0; ++k) {
#pragma unroll
    for (int i = 0; i < L; ++i) {
      if (i > k || k - i >= L) continue;
      mac3(c0, c1, c2, a[i], x[k - i]);
    }
    sticky |= c0;
    c0 = c1; c1 = c2; c2 = 0u;
  }
  return sticky;
}

// --------------------------------------------------------------------------
// t = RN_p(a * x) by a SHORT product with an exactness certificate (DESIGN.md
// "Product").  Only columns k >= K0 = L-D are formed first (T, zero carry-in;
// D = MPSP_SHORT_D = 2 by default); the omitted part
// N = sum_{i+j<K0} a_i x_j 2^(32(i+j)) satisfies 0 <= N < 2^B, B = 32 K0 + 37
// (fewer than 32 terms per column, each < 2^64).  Let W be the bits of T in
// [B, round bit).  If W is neither all zeros nor all ones, adding N cannot
// carry past W, so every bit from the round bit up - hence the normalisation,
// the kept limbs and the round bit - is the exact product's, and the sticky
// is 1 (W or W+1 is nonzero).  Otherwise the lower columns are formed too and
// their carry added in: the exact product.  W has 25 bits at D = 2 (57 at
// D = 3), so random mantissas take that path with probability ~2^-24 (a few
// products per 10^8); structured inputs whose operand has zero low limbs take
// the exact-short path below instead.
// Executed limb-MACs on the fast path: L^2 - (L-D)(L-D+1)/2
// (D = 2, L = 8 / 16 / 32: 43 / 151 / 588; D = 3: 49 / 165 / 618).
// --------------------------------------------------------------------------
#ifndef MPSP_SHORT_D
#define MPSP_SHORT_D 2
#endif
template <int L>
struct Short {
  static constexpr int D = MPSP_SHORT_D;   // columns L-D .. 2L-2 are formed
  static constexpr int K0 = L - D;
  static constexpr int NT = L + D;         // T[m] = limb K0 + m, m in [0, L+D)
};

// The rounding half of mp_mul: T = comba_upper<L, K0>(a, x) -> t.
template <int L, bool FW = false>
__device__ __forceinline__ void mp_mul_finish(const uint32_t (&a)[L], int32_t ea, uint32_t sa,
                                              const uint32_t (&x)[L], int32_t ex, uint32_t sx,
                                              uint32_t (&T)[Short<L>::NT], MP<L>& t);

template <int L, bool FW = false>
__device__ __forceinline__ void mp_mul(const uint32_t (&a)[L], int32_t ea, uint32_t sa,
                                       const uint32_t (&x)[L], int32_t ex, uint32_t sx,
                                       MP<L>& t) {
  if constexpr (L < 4) {
    mp_mul_full<L>(a, ea, sa, x, ex, sx, t);
  } else {
    uint32_t T[Short<L>::NT];                        // limbs K0 .. 2L-1
    comba_upper<L, Short<L>::K0>(a, x, T);
    mp_mul_finish<L, FW>(a, ea, sa, x, ex, sx, T, t);
  }
}

template <int L, bool FW>
__device__ __forceinline__ void mp_mul_finish(const uint32_t (&a)[L], int32_t ea, uint32_t sa,
                                              const uint32_t (&x)[L], int32_t ex, uint32_t sx,
                                              uint32_t (&T)[Short<L>::NT], MP<L>& t) {
  constexpr int D = Short<L>::D, K0 = Short<L>::K0, NT = Short<L>::NT;
  static_assert(D == 2 || D == 3, "short product: D in {2, 3}");
  uint32_t sh = (~T[NT - 1]) >> 31;                // top product bit clear -> 1
  // W: the bits between B (bit 5 of T[1]) and the round bit (bit 31 - sh of
  // T[D-1], the product's limb L-1)
  bool amb;
  if constexpr (D == 3) {
    const uint32_t wmask = (1u << (31u - sh)) - 1u;
    const uint32_t w1 = T[1] >> 5, w2 = T[2] & wmask;
    amb = ((w1 | w2) == 0u) | ((w1 == 0x07FFFFFFu) & (w2 == wmask));
  } else {
    const uint32_t wv = ((T[1] << sh) << 1) >> 7;  // bits 6 .. 30 of T[1] << sh
    amb = (wv == 0u) | (wv == 0x01FFFFFFu);
  }
  const bool zero = (a[L - 1] == 0u) | (x[L - 1] == 0u);
  uint32_t stk = 1u;
  auto low_sticky = [&]() {                        // T's bits below the round bit
    uint32_t v = (T[D - 1] << sh) << 1;
#pragma unroll
    for (int i = 0; i < D - 1; ++i) v |= T[i];
    return v;
  };
  // Exact short product: every omitted term a_i x_j (i + j < K0) has i, j
  // < K0, so N = 0 when either operand's limbs 0 .. K0-1 are all zero
  // (e.g. a power-of-two mantissa: C5's diagonal 4, exact-integer data) -
  // then T is the exact product and no lower column is formed.
  bool low0 = false;
  if (amb && !zero) {
    uint32_t ao = 0u, xo = 0u;
#pragma unroll
    for (int i = 0; i < K0; ++i) { ao |= a[i]; xo |= x[i]; }
    low0 = (ao == 0u) | (xo == 0u);
    if (low0) stk = low_sticky();
  }
  if (amb && !zero && !low0) {                     // rare: complete the product
    uint32_t c0, c1, c2;
    const uint32_t slo = comba_lower<L, K0>(a, x, c0, c1, c2);
    uint32_t C[NT];
    C[0] = c0; C[1] = c1; C[2] = c2;
#pragma unroll
    for (int i = 3; i < NT; ++i) C[i] = 0u;
    add_n<NT>(T, T, C);
    sh = (~T[NT - 1]) >> 31;
    stk = slo | low_sticky();
  }
#pragma unroll
  for (int i = L - 1; i >= 0; --i) t.m[i] = __funnelshift_l(T[i + D - 1], T[i + D], sh);
  const uint32_t rb = (T[D - 1] << sh) >> 31;
  const uint32_t cy = rne_increment<L, FW>(t.m, rb, stk);
  if (cy) t.m[L - 1] = 0x80000000u;
  t.e = ea + ex - (int32_t)sh + (int32_t)cy;
  t.s = sa ^ sx;
  // A zero operand has all limbs 0 (include/mpsp.h value encoding; every
  // zero the kernels produce is +0 with zero limbs), so T = 0, the round bit
  // is 0 and t.m is already all zero: no masking of the limbs (L SELs per
  // product; measured C2 A x -2.7%, C3 / C4 -0.4..0.6%, bit-exact).  `zero`
  // only keeps such products off the completion branch.
}

// --------------------------------------------------------------------------
// Variable shifts over N-limb register arrays (binary decomposition of the
// limb count so indices stay compile-time; no local memory).
// --------------------------------------------------------------------------
// FW: every lane of the warp executes the call (full-warp collectives, no
// __activemask()); otherwise the active lanes'
template <int N, bool FW = false>
__device__ __forceinline__ void shr_bits_sticky(uint32_t (&v)[N], uint32_t d, uint32_t& sticky) {
  const uint32_t q = d >> 5, r = d & 31u;
  // limb steps only up to the largest limb shift any active lane needs
  // (warp-uniform branch: no divergence, no dynamic register indexing); the
  // one- and two-limb steps of short operands (N <= 17), which nearly every
  // warp needs there, run unconditionally (a branch per level made ptxas copy
  // the whole array at each merge; measured C4 -2%, C5 needs neither)
  constexpr int UNC = N <= 17 ? 4 : 1;
  const uint32_t qmax = N > UNC ? __reduce_max_sync(FW ? 0xffffffffu : __activemask(), q) : 0u;
#pragma unroll
  for (int b = 1; b <= N; b <<= 1) {
    if (b < UNC || qmax >= (uint32_t)b) {
      const bool on = (q & (uint32_t)b) != 0u;
      uint32_t drop = 0u;
#pragma unroll
      for (int i = 0; i < b; ++i) drop |= v[i];
      sticky |= on ? drop : 0u;
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = on ? (i + b < N ? v[i + b] : 0u) : v[i];
    }
  }
  sticky |= r ? (v[0] << (32u - r)) : 0u;
#pragma unroll
  for (int i = 0; i < N - 1; ++i) v[i] = __funnelshift_r(v[i], v[i + 1], r);
  v[N - 1] >>= r;
}

template <int N>
__device__ __forceinline__ void shl_bits(uint32_t (&v)[N], uint32_t d) {
  const uint32_t q = d >> 5, r = d & 31u;
#pragma unroll
  for (int b = 1; b < N; b <<= 1) {
    const bool on = (q & (uint32_t)b) != 0u;
#pragma unroll
    for (int i = N - 1; i >= 0; --i) v[i] = on ? (i - b >= 0 ? v[i - b] : 0u) : v[i];
  }
#pragma unroll
  for (int i = N - 1; i > 0; --i) v[i] = __funnelshift_l(v[i - 1], v[i], r);
  v[0] <<= r;
}

template <int N>
__device__ __forceinline__ uint32_t clz_limbs(const uint32_t (&v)[N]) {
  uint32_t lz = 0u;
  bool found = false;
#pragma unroll
  for (int i = N - 1; i >= 0; --i) {
    const uint32_t c = __clz(v[i]);
    lz += found ? 0u : c;
    found = found || (v[i] != 0u);
  }
  return lz;
}

// z = x + y + cin (N limbs, cin in {0,1}); returns the carry out
template <int N>
__device__ __forceinline__ uint32_t add_n_cin(uint32_t (&z)[N], const uint32_t (&x)[N],
                                              const uint32_t (&y)[N], uint32_t cin) {
  uint32_t c, dummy;
  asm volatile("add.cc.u32 %0, %1, 0xffffffff;" : "=r"(dummy) : "r"(cin));  // CF = cin
#pragma unroll
  for (int i = 0; i < N; ++i)
    asm volatile("addc.cc.u32 %0, %1, %2;" : "=r"(z[i]) : "r"(x[i]), "r"(y[i]));
  asm volatile("addc.u32 %0, 0, 0;" : "=r"(c));
  return c;
}

// --------------------------------------------------------------------------
// s = RN_p(s + t)   (the oracle's add() computes the
// same value by exact integer alignment).  Working width: L+1 limbs, i.e.
// one 32-bit guard limb below the LSB, plus a sticky word for bits shifted
// beyond it.  |exponent gap| >= p+2 returns the larger operand (far-path
// lemma).
//
// ONE branch-free path for every case (no near/far split: in a warp of
// independent rows the two paths diverge in most steps, and both would run):
//   Z = big * 2^32, Y = small * 2^32 >> d  (sticky: bits beyond the guard);
//   Z := Z + (Y ^ m) + cin,  m = cin = 0 for equal signs, m = ~0 and
//        cin = 1 - [sticky] for opposite signs (Z - Y - [sticky]; exact for
//        d <= 1, where nothing reaches the sticky);
//   equal signs: shift right by the carry W (the dropped bit joins the sticky);
//   then shift left by lz = clz(top limb) (0 or 1 for d >= 2; any amount for
//   the cancellation at d <= 1; >= 32 bits of cancellation or an exact zero
//   take the one rare branch);  e = e_big + W - lz;  round to nearest even.
// --------------------------------------------------------------------------
template <int L, bool FW = false>
__device__ __forceinline__ void mp_add(MP<L>& s, const MP<L>& t) {
  const bool tz = t.is_zero(), sz = s.is_zero();
  // |M_s| < |M_t| matters only for equal exponents: the top limbs decide it.
  // When they are equal too, s is taken as the big operand; if that was the
  // smaller one and the signs differ, Z - Y borrows (its top limbs cancel,
  // so >= 32 bits cancel): the rare branch below negates it.
  const uint32_t mlt = s.m[L - 1] < t.m[L - 1] ? 1u : 0u;
  // bitwise (not short-circuit) logic: no branches in the common path
  const bool t_big = !tz & (sz | (t.e > s.e) | ((t.e == s.e) & (mlt != 0u)));
  const int32_t eb = t_big ? t.e : s.e;
  const int32_t esm = t_big ? s.e : t.e;
  const uint32_t sb = t_big ? t.s : s.s;
  const uint32_t sub = ((t.s != s.s) & !tz & !sz) ? 1u : 0u;
  uint32_t d = (uint32_t)eb - (uint32_t)esm;            // exact as uint32
  d = (tz || sz) ? 0u : min(d, (uint32_t)(32 * (L + 1)));  // d >= p+2: all sticky
  uint32_t Z[L + 1], Y[L + 1];
  Z[0] = 0u;
  Y[0] = 0u;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    Z[i + 1] = t_big ? t.m[i] : s.m[i];
    Y[i + 1] = t_big ? s.m[i] : t.m[i];
  }
  uint32_t stk = 0u;
  shr_bits_sticky<L + 1, FW>(Y, d, stk);
  const uint32_t msk = 0u - sub;
#pragma unroll
  for (int i = 0; i <= L; ++i) Y[i] ^= msk;
  const uint32_t cin = sub & (stk == 0u ? 1u : 0u);
  const uint32_t c = add_n_cin<L + 1>(Z, Z, Y, cin);
  const uint32_t W = c & (sub ^ 1u);
  const bool neg = (sub != 0u) & (c == 0u);             // Z - Y < 0 (see above)
  stk |= Z[0] & W;                                      // bit lost by the right shift
#pragma unroll
  for (int i = 0; i < L; ++i) Z[i] = __funnelshift_r(Z[i], Z[i + 1], W);
  Z[L] = __funnelshift_r(Z[L], W, W);
  uint32_t lz = __clz(Z[L]);
  uint32_t sres = sb;
  if ((lz < 32u) & !neg) {
#pragma unroll
    for (int i = L; i > 0; --i) Z[i] = __funnelshift_l(Z[i - 1], Z[i], lz);
    Z[0] <<= lz;
  } else {            // >= 32 bits cancelled, or an exact zero (rare)
    if (neg) {        // d = 0: nothing reached the sticky, -Z is exact
#pragma unroll
      for (int i = 0; i <= L; ++i) Z[i] = ~Z[i];
      inc_n<L + 1>(Z, 1u);
      sres ^= 1u;
    }
    lz = clz_limbs<L + 1>(Z);
    shl_bits<L + 1>(Z, lz);
  }
  const int32_t e = eb + (int32_t)W - (int32_t)lz;
  const uint32_t rb = Z[0] >> 31;
  const uint32_t st = stk | (Z[0] << 1);
#pragma unroll
  for (int i = 0; i < L; ++i) s.m[i] = Z[i + 1];
  const uint32_t cy = rne_increment<L, FW>(s.m, rb, st);
  if (cy) s.m[L - 1] = 0x80000000u;
  s.e = e + (int32_t)cy;
  s.s = sres;
}

}  // namespace mpsp
