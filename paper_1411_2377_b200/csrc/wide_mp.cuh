// wide_mp.cuh - p-bit arithmetic with the limbs of every value spread over a
// warp's 32 lanes (lane j holds limbs jK .. jK+K-1, K = L/32; exponent and
// sign warp-uniform), for p > 1024 (L = 64, 128, 256).  Used by the SpMV
// kernel spmv_wide.cu and the solver kernels krylov_wide.cu.  Every function
// is called by all 32 lanes of a warp together.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernel_common.cuh"

namespace mpsp {
namespace wide {

constexpr unsigned FULL = 0xffffffffu;

template <int K>
struct WMP {
  uint32_t m[K];   // limbs lane*K .. lane*K+K-1
  int32_t e;       // warp-uniform
  uint32_t s;      // warp-uniform
};

template <int K>
__device__ __forceinline__ bool all_ones(const uint32_t (&v)[K]) {
  uint32_t a = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < K; ++i) a &= v[i];
  return a == 0xffffffffu;
}

// Carry into this lane of a cross-lane ripple: g = the lane produced a carry
// out of its top limb, p = its limbs are all ones (a carry in passes through;
// g and p never both hold).  With A = P|G, B = G, the carries of the 32-bit
// addition A + B are exactly the lane carries:  C = (A + B) ^ A ^ B.
// *cout = carry out of lane 31.
__device__ __forceinline__ uint32_t ripple(bool g, bool p, int lane, uint32_t* cout) {
  const uint32_t G = __ballot_sync(FULL, g), P = __ballot_sync(FULL, p && !g);
  const uint64_t A = (uint64_t)(P | G);
  const uint64_t S = A + G;
  const uint32_t C = (uint32_t)S ^ (uint32_t)A ^ G;
  if (cout) *cout = (uint32_t)(S >> 32);
  return (C >> lane) & 1u;
}

// (acc64 : c2) += a*b with the low two words held as ONE 64-bit register
// pair: IMAD.WIDE.U32 accumulates in place (three separate 32-bit words made
// ptxas copy them into a fresh aligned pair before every multiply-add).
__device__ __forceinline__ void mac64(uint64_t& acc, uint32_t& c2, uint32_t a, uint32_t b) {
  asm("{\n\t.reg .u32 lo, hi;\n\t"
      "mov.b64 {lo, hi}, %0;\n\t"
      "mad.lo.cc.u32 lo, %2, %3, lo;\n\t"
      "madc.hi.cc.u32 hi, %2, %3, hi;\n\t"
      "addc.u32 %1, %1, 0;\n\t"
      "mov.b64 %0, {lo, hi};\n\t}"
      : "+l"(acc), "+r"(c2)
      : "r"(a), "r"(b));
}

template <int K>
__device__ __forceinline__ bool wzero(const WMP<K>& v) {
  return __shfl_sync(FULL, v.m[K - 1], 31) == 0u;
}

template <int K>
__device__ __forceinline__ void wset_zero(WMP<K>& v) {
#pragma unroll
  for (int i = 0; i < K; ++i) v.m[i] = 0u;
  v.e = 0;
  v.s = 0u;
}

// RNE increment of a distributed L-limb mantissa; returns the carry out of
// the top (mantissa became 2^p; the caller renormalises).
template <int K>
__device__ __forceinline__ uint32_t wround(uint32_t (&m)[K], uint32_t inc, int lane) {
  uint32_t c = 0u;
  if (lane == 0) c = inc_n<K>(m, inc);
  uint32_t cout;
  const uint32_t cin = ripple(c != 0u, all_ones<K>(m), lane, &cout);
  if (lane != 0) inc_n<K>(m, cin);
  return cout;
}

// Comba column sums of a x (operands in sA, sX) into cs0/cs1/cs2 = cs,
// cs + 2L, cs + 4L (three words per column, 2L columns).  Lane j owns columns
// c = j + 32u and c + L (u < K): their term counts add up to L, so the MACs
// are balanced; in the 32-step diagonal chunk (u == v) lanes switch from c to
// c + L at different steps and both accumulators take a MAC (one with a zero
// operand).  SHORT: only the columns >= L-3 (others written as 0): the hi
// columns as above, the three top lo columns from per-lane partial sums over
// i = j (mod 32) reduced across the warp - the lo MACs (u > v) are skipped.
// sA: a in the ZERO-GAPPED layout, chunk v (limbs 32v .. 32v+31) at words
// [64v, 64v + 32) and 32 zero words after it, so the diagonal chunk's skewed
// reads past the chunk load zeros (no per-MAC select).  The 32 steps of a
// chunk are unrolled 16x at K = 2, 4 and 8x at K = 8 (measured, C2 at p =
// 2048 / 4096 / 8192: 4x 1301 / 2917 / 8655 us, 8x 1234 / 2802 / 8509, 16x
// 1185 / 2763 / 8910, 32x 1762 at p = 2048; before the zero-gapped layout
// and these unrolls 1456 / 3174 / 8714).
template <int K, bool SHORT>
__device__ __forceinline__ void wcolumns(const uint32_t* sA, const uint32_t* sX, uint32_t* cs,
                                         int lane) {
  constexpr int L = 32 * K;
  uint64_t lo[K], hi[K];
  uint32_t lo2[K], hi2[K];
#pragma unroll
  for (int u = 0; u < K; ++u) { lo[u] = hi[u] = 0u; lo2[u] = hi2[u] = 0u; }
#pragma unroll
  for (int v = 0; v < K; ++v) {                    // i in [32v, 32v + 32)
#pragma unroll (K >= 8 ? 8 : 16)
    for (int ii = 0; ii < 32; ++ii) {
      const int i = 32 * v + ii;
      const uint32_t ai = sA[64 * v + ii];
#pragma unroll
      for (int u = 0; u < K; ++u) {
        const int c = lane + 32 * u;
        if (u > v) {                               // i <= c: column c
          if (!SHORT) mac64(lo[u], lo2[u], ai, sX[c - i]);
        } else if (u < v) {                        // i > c: column c + L
          mac64(hi[u], hi2[u], ai, sX[c + L - i]);
        } else if (SHORT) {                        // diagonal chunk, hi part only
          // skewed: lane j takes i2 = 32v + j + 1 + ii, so x[c + L - i2] =
          // x[L - 1 - ii] is one broadcast word; i2 past the chunk (ii >=
          // 31 - j) contributes a zero operand
          const uint32_t a2 = sA[64 * v + lane + 1 + ii];   // a zero past the chunk
          const uint32_t x2 = sX[L - 1 - ii];
          mac64(hi[u], hi2[u], a2, x2);
        } else {                                   // diagonal chunk: both
          const bool l = ii <= lane;
          const uint32_t xv = sX[l ? c - i : c + L - i];
          mac64(lo[u], lo2[u], ai, l ? xv : 0u);
          mac64(hi[u], hi2[u], ai, l ? 0u : xv);
        }
      }
    }
  }
  uint64_t top[2] = {0u, 0u};                      // SHORT: columns L-2, L-1
  uint32_t top2[2] = {0u, 0u};
  if (SHORT) {
#pragma unroll
    for (int m = 0; m < K; ++m) {
      const int i = lane + 32 * m;
      const uint32_t ai = sA[64 * m + lane];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int xi = L - 2 + r - i;
        const uint32_t xv = sX[xi >= 0 ? xi : 0];
        mac64(top[r], top2[r], ai, xi >= 0 ? xv : 0u);
      }
    }
    // warp sums of the two columns' per-lane partials (top2:top < K 2^64)
    // by redux.sync on 16-bit pieces: each piece's 32-lane sum is < 2^21, so
    // the u32 reductions are exact (5 REDUX per column instead of a 5-level
    // butterfly of three shuffles and a 96-bit add per level)
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const uint64_t v = top[r];
      const uint32_t s0 = __reduce_add_sync(FULL, (uint32_t)v & 0xffffu);
      const uint32_t s1 = __reduce_add_sync(FULL, (uint32_t)v >> 16);
      const uint32_t s2 = __reduce_add_sync(FULL, (uint32_t)(v >> 32) & 0xffffu);
      const uint32_t s3 = __reduce_add_sync(FULL, (uint32_t)(v >> 48));
      const uint32_t t2 = __reduce_add_sync(FULL, top2[r]);
      const uint64_t A = (uint64_t)s0 + ((uint64_t)s1 << 16);    // < 2^38
      const uint64_t B = (uint64_t)s2 + ((uint64_t)s3 << 16);    // < 2^38
      const uint64_t lo64 = A + (B << 32);
      top[r] = lo64;
      top2[r] = (uint32_t)(B >> 32) + t2 + (lo64 < A ? 1u : 0u);
    }
  }
  uint32_t* cs0 = cs;
  uint32_t* cs1 = cs + 2 * L;
  uint32_t* cs2 = cs + 4 * L;
  __syncwarp();                                    // sA (in cs2's words) fully read
#pragma unroll
  for (int u = 0; u < K; ++u) {
    const int c = lane + 32 * u;
    uint64_t lv = lo[u];
    uint32_t l2 = lo2[u];
    if (SHORT) {
      lv = 0u;
      l2 = 0u;
      if (u == K - 1 && lane >= 30) {
        lv = lane == 30 ? top[0] : top[1];
        l2 = lane == 30 ? top2[0] : top2[1];
      }
    }
    cs0[c] = (uint32_t)lv; cs1[c] = (uint32_t)(lv >> 32); cs2[c] = l2;
    cs0[c + L] = (uint32_t)hi[u]; cs1[c + L] = (uint32_t)(hi[u] >> 32); cs2[c + L] = hi2[u];
  }
}

// The column sums in cs -> the product's limbs, written to cs[0 .. 2L) (lane
// j sums limbs [2Kj, 2Kj+2K) lane-locally; the carry words are passed up one
// lane and the one-bit ripple resolved by ripple()).
template <int K>
__device__ __forceinline__ void wcarry(uint32_t* cs, int lane) {
  constexpr int L = 32 * K;
  const uint32_t* cs0 = cs;
  const uint32_t* cs1 = cs + 2 * L;
  const uint32_t* cs2 = cs + 4 * L;
  uint32_t Pl[2 * K];
  uint64_t carry = 0u;
#pragma unroll
  for (int q = 0; q < 2 * K; ++q) {
    const int k = 2 * K * lane + q;
    const uint64_t sum = (uint64_t)cs0[k] + (k >= 1 ? cs1[k - 1] : 0u) + (k >= 2 ? cs2[k - 2] : 0u) + carry;
    Pl[q] = (uint32_t)sum;
    carry = sum >> 32;
  }
  {
    const uint32_t cw = __shfl_up_sync(FULL, (uint32_t)carry, 1);
    uint32_t c0 = 0u;
    if (lane > 0) {
      uint32_t Cv[2 * K];
      Cv[0] = cw;
#pragma unroll
      for (int q = 1; q < 2 * K; ++q) Cv[q] = 0u;
      c0 = add_n<2 * K>(Pl, Pl, Cv);
    }
    const uint32_t cin = ripple(c0 != 0u, all_ones<2 * K>(Pl), lane, nullptr);
    inc_n<2 * K>(Pl, cin);
  }
  __syncwarp();                                    // everyone is done reading cs
#pragma unroll
  for (int q = 0; q < 2 * K; ++q) cs[2 * K * lane + q] = Pl[q];
  __syncwarp();
}

// t = RN(a * x).  sA, sX: L words each, cs: 6L words (per-warp shared memory).
// SHORT PRODUCT with an exactness certificate (the wide form of mp_mul's):
// only the columns >= K0 = L-2 are formed; the omitted part is
// N < K0 2^(32(L-1)) (1 + eps) < 2^B, B = 32(L-1) + 8 (K0 < 256), so if the
// 22-23 bits between B and the round bit are neither all 0 nor all 1, the
// rounded product is the exact one's with sticky 1; otherwise (~2^-21 per
// random product) the full product.
template <int K>
__device__ __forceinline__ void wmul(const uint32_t (&a)[K], int32_t ea, uint32_t sa,
                                     const uint32_t (&x)[K], int32_t ex, uint32_t sx,
                                     uint32_t* sA, uint32_t* sX, uint32_t* cs, int lane,
                                     WMP<K>& t) {
  constexpr int L = 32 * K;
  const bool az = __shfl_sync(FULL, a[K - 1], 31) == 0u;
  const bool xz = __shfl_sync(FULL, x[K - 1], 31) == 0u;
  if (az || xz) {                                  // warp-uniform
    wset_zero<K>(t);
    return;
  }
  // a goes to cs + 4L in the zero-gapped layout of wcolumns (2L words; the
  // column sums overwrite it at the end of wcolumns); sA is not used
  uint32_t* sAg = cs + 4 * L;
  __syncwarp();                                    // a caller's reads of cs are done
  auto put_a = [&]() {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int m = lane * K + i;
      sAg[64 * (m >> 5) + (m & 31)] = a[i];
      sAg[64 * (m >> 5) + 32 + (m & 31)] = 0u;
    }
  };
  put_a();
#pragma unroll
  for (int i = 0; i < K; ++i) sX[lane * K + i] = x[i];
  __syncwarp();
  wcolumns<K, true>(sAg, sX, cs, lane);
  __syncwarp();
  wcarry<K>(cs, lane);
  const uint32_t* Ps = cs;                         // P (short: limbs >= L-1 valid), 2L words
  uint32_t sh = (~Ps[2 * L - 1]) >> 31;            // top bit clear -> 1
  {
    const uint32_t wmask = (1u << (31u - sh)) - 1u;   // Ps[L-1] below the round bit
    const uint32_t w = (Ps[L - 1] & wmask) >> 8;       // the window, 23 - sh bits
    const bool amb = (w == 0u) | (w == (wmask >> 8));
    if (amb) {                                     // warp-uniform (same smem words): full product
      __syncwarp();
      put_a();                                     // (the column sums overwrote it)
      __syncwarp();
      wcolumns<K, false>(sAg, sX, cs, lane);
      __syncwarp();
      wcarry<K>(cs, lane);
      sh = (~Ps[2 * L - 1]) >> 31;
    }
    const uint32_t wl = Ps[L - 1] << sh;           // the limb below the kept ones
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int m = lane * K + i;
      t.m[i] = __funnelshift_l(Ps[L + m - 1], Ps[L + m], sh);
    }
    bool sticky = true;                            // certified: the window is nonzero
    if (amb) {
      uint32_t orr = 0u;
      for (int k = lane; k < L - 1; k += 32) orr |= Ps[k];
      sticky = (__ballot_sync(FULL, orr != 0u) != 0u) || ((wl << 1) != 0u);
    }
    const uint32_t rb = wl >> 31;
    const uint32_t lsb = __shfl_sync(FULL, t.m[0], 0) & 1u;
    const uint32_t inc = rb & ((sticky ? 1u : 0u) | lsb);
    __syncwarp();                                  // Ps reads done before cs is reused
    const uint32_t cy = wround<K>(t.m, inc, lane);
    if (cy && lane == 31) t.m[K - 1] = 0x80000000u;
    t.e = ea + ex - (int32_t)sh + (int32_t)cy;
  }
  t.s = sa ^ sx;
}

// s = RN(s + t).  ys: 2L+2 words of per-warp shared memory.
template <int K>
__device__ __forceinline__ void wadd(WMP<K>& s, const WMP<K>& t, uint32_t* ys, int lane) {
  constexpr int L = 32 * K;
  if (wzero<K>(t)) return;
  if (wzero<K>(s)) {
    s = t;
    return;
  }
  // |t| > |s| ?
  bool tb;
  if (t.e != s.e) {
    tb = t.e > s.e;
  } else {
    int cmp = 0;                                   // this lane's limbs: t vs s
#pragma unroll
    for (int i = K - 1; i >= 0; --i)
      if (cmp == 0 && t.m[i] != s.m[i]) cmp = t.m[i] > s.m[i] ? 1 : -1;
    const unsigned ne = __ballot_sync(FULL, cmp != 0);
    tb = ne ? (__shfl_sync(FULL, cmp, 31 - __clz(ne)) > 0) : false;
  }
  uint32_t Z[K], Y[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    Z[i] = tb ? t.m[i] : s.m[i];
    Y[i] = tb ? s.m[i] : t.m[i];
  }
  const int32_t eb = tb ? t.e : s.e, esm = tb ? s.e : t.e;
  const uint32_t sb = tb ? t.s : s.s;
  const uint32_t sub = t.s != s.s ? 1u : 0u;
  const int64_t d = (int64_t)eb - (int64_t)esm;
  if (d >= 32 * L + 2) {                           // far path: RN(big +- small) = big
#pragma unroll
    for (int i = 0; i < K; ++i) s.m[i] = Z[i];
    s.e = eb;
    s.s = sb;
    return;
  }
  // Y (with a guard limb at index 0) shifted right by d: ys[1 + m] = small limb m
  const uint32_t q = (uint32_t)d >> 5, r = (uint32_t)d & 31u;
  uint32_t y[K], yg = 0u, stk0 = 0u;
  if (q == 0u) {                                   // d < 32 (warp-uniform): a lane shuffle,
    const uint32_t nx = __shfl_down_sync(FULL, Y[0], 1);   // nothing below the guard
#pragma unroll
    for (int i = 0; i < K; ++i) y[i] = __funnelshift_r(Y[i], i + 1 < K ? Y[i + 1] : (lane < 31 ? nx : 0u), r);
    if (lane == 0) yg = __funnelshift_r(0u, Y[0], r);
  } else {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      ys[1 + lane * K + i] = Y[i];
      ys[L + 1 + lane * K + i] = 0u;
    }
    if (lane == 0) { ys[0] = 0u; ys[2 * L + 1] = 0u; }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int k = lane * K + 1 + i;                // aligned position k (1..L)
      y[i] = __funnelshift_r(ys[k + q], ys[k + q + 1], r);
    }
    if (lane == 0) yg = __funnelshift_r(ys[q], ys[q + 1], r);
    // bits below the guard limb: ys[0 .. q) and ys[q]'s low r bits, i.e. the
    // small operand's limbs 0 .. q-2 and limb q-1's low r bits - read from
    // the registers of the lanes that hold them
    uint32_t orr = 0u;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const uint32_t m1 = (uint32_t)(lane * K + i) + 1u;   // ys position of limb lane*K+i
      orr |= m1 < q ? Y[i] : (m1 == q ? (Y[i] & ((1u << r) - 1u)) : 0u);
    }
    stk0 = __ballot_sync(FULL, orr != 0u) != 0u ? 1u : 0u;
    __syncwarp();                                    // ys reads done
  }
  // Z + (Y ^ m) + cin over [guard | L limbs]; m = ~0, cin = 1 - stk for a subtraction
  const uint32_t msk = 0u - sub;
  uint32_t zg = 0u, c = 0u;
  if (lane == 0) {
    const uint64_t g = (uint64_t)(yg ^ msk) + (sub & (stk0 ^ 1u));
    zg = (uint32_t)g;
    c = (uint32_t)(g >> 32);
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const uint64_t v = (uint64_t)Z[i] + (y[i] ^ msk) + c;
    Z[i] = (uint32_t)v;
    c = (uint32_t)(v >> 32);
  }
  uint32_t ctop;
  const uint32_t cin = ripple(c != 0u, all_ones<K>(Z), lane, &ctop);
  inc_n<K>(Z, cin);
  const uint32_t W = ctop & (sub ^ 1u);
  uint32_t stk = stk0;
  int32_t lz = 0;
  const uint32_t below = __shfl_up_sync(FULL, Z[K - 1], 1);   // lane j-1's top limb
  const uint32_t above = __shfl_down_sync(FULL, Z[0], 1);     // lane j+1's bottom limb
  if (W) {                                         // carry: shift right 1, top bit = 1
    if (lane == 0) { stk |= zg & 1u; zg = __funnelshift_r(zg, Z[0], 1); }
#pragma unroll
    for (int i = 0; i < K - 1; ++i) Z[i] = __funnelshift_r(Z[i], Z[i + 1], 1);
    Z[K - 1] = __funnelshift_r(Z[K - 1], lane == 31 ? 1u : above, 1);
    stk = __shfl_sync(FULL, stk, 0);
  } else {
    const uint32_t top = __shfl_sync(FULL, Z[K - 1], 31);
    lz = (int32_t)__clz(top);
    if (lz < 32) {
      const uint32_t lo = lane == 0 ? zg : below;
#pragma unroll
      for (int i = K - 1; i > 0; --i) Z[i] = __funnelshift_l(Z[i - 1], Z[i], (uint32_t)lz);
      Z[0] = __funnelshift_l(lo, Z[0], (uint32_t)lz);
      if (lane == 0) zg <<= lz;
    } else {                                       // >= 32 bits cancelled (rare)
#pragma unroll
      for (int i = 0; i < K; ++i) ys[1 + lane * K + i] = Z[i];
      if (lane == 0) ys[0] = zg;
      __syncwarp();
      int hi = -1;                                 // highest nonzero word of [guard | Z]
      for (int k = lane; k <= L; k += 32)
        if (ys[k] != 0u) hi = k;
      const int top_w = __reduce_max_sync(FULL, hi + 1) - 1;
      if (top_w < 0) {                             // exact zero -> +0
        __syncwarp();
        wset_zero<K>(s);
        return;
      }
      const uint32_t wsh = (uint32_t)(L - top_w);  // whole words to shift left
      const uint32_t bsh = __clz(ys[top_w]);
      lz = (int32_t)(32 * wsh + bsh);
      // new word k (0..L) = bits of old words k - wsh - 1, k - wsh shifted by bsh
      uint32_t nz[K], ng = 0u;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const int k = lane * K + 1 + i;
        const int s0 = k - (int)wsh;
        const uint32_t hw = s0 >= 0 ? ys[s0] : 0u, lw = s0 >= 1 ? ys[s0 - 1] : 0u;
        nz[i] = __funnelshift_l(lw, hw, bsh);
      }
      if (lane == 0) {
        const int s0 = -(int)wsh;
        const uint32_t hw = s0 >= 0 ? ys[s0] : 0u;
        ng = hw << bsh;
      }
      __syncwarp();
#pragma unroll
      for (int i = 0; i < K; ++i) Z[i] = nz[i];
      zg = ng;
    }
  }
  const int32_t e = eb + (int32_t)W - lz;
  const uint32_t g0 = __shfl_sync(FULL, zg, 0);
  const uint32_t rb = g0 >> 31;
  const uint32_t st = stk | (g0 << 1);
  const uint32_t lsb = __shfl_sync(FULL, Z[0], 0) & 1u;
  const uint32_t inc = rb & ((st != 0u ? 1u : 0u) | lsb);
  const uint32_t cy = wround<K>(Z, inc, lane);
  if (cy && lane == 31) Z[K - 1] = 0x80000000u;
#pragma unroll
  for (int i = 0; i < K; ++i) s.m[i] = Z[i];
  s.e = e + (int32_t)cy;
  s.s = sb;
}

template <int K>
__device__ __forceinline__ void load_k(const uint32_t* __restrict__ p, uint32_t (&v)[K]) {
  if constexpr (K % 4 == 0) {
#pragma unroll
    for (int c = 0; c < K / 4; ++c) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(p) + c);
      v[4 * c] = w.x; v[4 * c + 1] = w.y; v[4 * c + 2] = w.z; v[4 * c + 3] = w.w;
    }
  } else if constexpr (K % 2 == 0) {
#pragma unroll
    for (int c = 0; c < K / 2; ++c) {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(p) + c);
      v[2 * c] = w.x; v[2 * c + 1] = w.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] = __ldg(p + i);
  }
}

}  // namespace wide
}  // namespace mpsp
