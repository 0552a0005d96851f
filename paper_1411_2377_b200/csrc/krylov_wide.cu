// krylov_wide.cu - the BiCG / GPBiCG building blocks at p > 1024 (L = 64,
// 128, 256; the paper runs its solvers at 2048 bits
// and more), on warp-distributed values
// (wide_mp.cuh).  Same operations and readings as krylov.cu:
//   dot   : s = RN(s + RN(u_k v_k)), k ascending, from +0.  Products in
//           parallel (a warp per element); the ordered chain of adds split
//           into segments evaluated speculatively in parallel and validated
//           in order by one warp (see wseg_*).
//   axpy  : z_k = RN(y_k + RN(+-alpha x_k)), a warp per element.
//   scalar: the solver's scalar steps (krylov.cu bicg_scalar ops 0-8) in one
//           warp: RN division by restoring long division (p+4 quotient bits,
//           sticky, one rounding), RN square root digit by digit, exact
//           comparison - the big integers spread over the lanes (W words per
//           lane), carries and borrows resolved by the ballot ripple.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "wide_mp.cuh"

namespace mpsp {
namespace wide {

// ------------------------------------------------------------ big integers
// lane j holds words jW .. jW+W-1 (little endian over the warp)

template <int W>
__device__ __forceinline__ bool wi_lt(const uint32_t (&a)[W], const uint32_t (&b)[W]) {
  int cmp = 0;
#pragma unroll
  for (int i = W - 1; i >= 0; --i)
    if (cmp == 0 && a[i] != b[i]) cmp = a[i] > b[i] ? 1 : -1;
  const unsigned ne = __ballot_sync(FULL, cmp != 0);
  return ne ? (__shfl_sync(FULL, cmp, 31 - __clz(ne)) < 0) : false;
}

// a += b (carry out of the top dropped)
template <int W>
__device__ __forceinline__ void wi_add(uint32_t (&a)[W], const uint32_t (&b)[W], int lane) {
  uint32_t c = 0u;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const uint64_t v = (uint64_t)a[i] + b[i] + c;
    a[i] = (uint32_t)v;
    c = (uint32_t)(v >> 32);
  }
  inc_n<W>(a, ripple(c != 0u, all_ones<W>(a), lane, nullptr));
}

// a -= b (a >= b): a + ~b + 1
template <int W>
__device__ __forceinline__ void wi_sub(uint32_t (&a)[W], const uint32_t (&b)[W], int lane) {
  uint32_t c = lane == 0 ? 1u : 0u;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const uint64_t v = (uint64_t)a[i] + (~b[i]) + c;
    a[i] = (uint32_t)v;
    c = (uint32_t)(v >> 32);
  }
  inc_n<W>(a, ripple(c != 0u, all_ones<W>(a), lane, nullptr));
}

// a += 2^pos
template <int W>
__device__ __forceinline__ void wi_add_bit(uint32_t (&a)[W], int pos, int lane) {
  uint32_t b[W];
#pragma unroll
  for (int i = 0; i < W; ++i) b[i] = (lane * W + i == (pos >> 5)) ? (1u << (pos & 31)) : 0u;
  wi_add<W>(a, b, lane);
}

template <int W>
__device__ __forceinline__ void wi_shl1(uint32_t (&a)[W], int lane) {
  const uint32_t below = __shfl_up_sync(FULL, a[W - 1], 1);
  const uint32_t lo = lane ? below : 0u;
#pragma unroll
  for (int i = W - 1; i > 0; --i) a[i] = __funnelshift_l(a[i - 1], a[i], 1);
  a[0] = __funnelshift_l(lo, a[0], 1);
}

template <int W>
__device__ __forceinline__ void wi_shr1(uint32_t (&a)[W], int lane) {
  const uint32_t above = __shfl_down_sync(FULL, a[0], 1);
  const uint32_t hi = lane < 31 ? above : 0u;
#pragma unroll
  for (int i = 0; i < W - 1; ++i) a[i] = __funnelshift_r(a[i], a[i + 1], 1);
  a[W - 1] = __funnelshift_r(a[W - 1], hi, 1);
}

template <int W>
__device__ __forceinline__ bool wi_nonzero(const uint32_t (&a)[W]) {
  uint32_t o = 0u;
#pragma unroll
  for (int i = 0; i < W; ++i) o |= a[i];
  return __ballot_sync(FULL, o != 0u) != 0u;
}

// bit length (0 for zero)
template <int W>
__device__ __forceinline__ int wi_bitlen(const uint32_t (&a)[W], int lane) {
  int b = 0;
#pragma unroll
  for (int i = 0; i < W; ++i)
    if (a[i]) b = 32 * (lane * W + i) + 32 - __clz(a[i]);
  return (int)__reduce_max_sync(FULL, (unsigned)b);
}

// a <<= s (any s >= 0; bits beyond 32*32W dropped) through shared memory
// sm: at least 32W + 1 words
template <int W>
__device__ __forceinline__ void wi_shl(uint32_t (&a)[W], int s, uint32_t* sm, int lane) {
  __syncwarp();
#pragma unroll
  for (int i = 0; i < W; ++i) sm[1 + lane * W + i] = a[i];
  if (lane == 0) sm[0] = 0u;
  __syncwarp();
  const int q = s >> 5;
  const uint32_t r = (uint32_t)s & 31u;
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const int k = lane * W + i - q;                // source word (sm index k + 1)
    const uint32_t hw = k >= 0 ? sm[1 + k] : 0u, lw = k >= 1 ? sm[k] : 0u;
    a[i] = __funnelshift_l(lw, hw, r);
  }
  __syncwarp();
}

// element layout (K limbs per lane) <-> big integer layout (W words per lane)
template <int K, int W>
__device__ __forceinline__ void to_wi(const uint32_t (&m)[K], uint32_t (&a)[W], uint32_t* sm,
                                      int lane) {
  constexpr int L = 32 * K;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < K; ++i) sm[lane * K + i] = m[i];
  __syncwarp();
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const int k = lane * W + i;
    a[i] = k < L ? sm[k] : 0u;
  }
  __syncwarp();
}

// o = RN_p(N 2^f), N > 0 (the p-bit rounding of krylov.cu round_int)
template <int K, int W>
__device__ void wi_round(const uint32_t (&N)[W], int32_t f, uint32_t* sm, int lane, WMP<K>& o) {
  constexpr int L = 32 * K, P = 32 * L;
  const int b = wi_bitlen<W>(N, lane);
  __syncwarp();
#pragma unroll
  for (int i = 0; i < W; ++i) sm[lane * W + i] = N[i];
  if (lane == 0) { sm[32 * W] = 0u; sm[32 * W + 1] = 0u; }
  __syncwarp();
  uint32_t cy = 0u;
  if (b > P) {
    const int sh = b - P;                          // bits dropped below the LSB
    const int q = sh >> 5;
    const uint32_t r = (uint32_t)sh & 31u;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int m = lane * K + i;
      o.m[i] = __funnelshift_r(sm[q + m], sm[q + m + 1], r);
    }
    const int rbpos = sh - 1;
    const uint32_t rb = (sm[rbpos >> 5] >> (rbpos & 31)) & 1u;
    uint32_t orr = 0u;                             // bits [0, sh-1)
    for (int k = lane; k < (rbpos >> 5); k += 32) orr |= sm[k];
    if (lane == 0) orr |= sm[rbpos >> 5] & ((1u << (rbpos & 31)) - 1u);
    const bool sticky = __ballot_sync(FULL, orr != 0u) != 0u;
    const uint32_t lsb = __shfl_sync(FULL, o.m[0], 0) & 1u;
    __syncwarp();
    cy = wround<K>(o.m, rb & ((sticky ? 1u : 0u) | lsb), lane);
    if (cy && lane == 31) o.m[K - 1] = 0x80000000u;
  } else {
    const int s = P - b;                           // exact left shift
    const int q = s >> 5;
    const uint32_t r = (uint32_t)s & 31u;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int k = lane * K + i - q;
      const uint32_t hw = k >= 0 ? sm[k] : 0u, lw = k >= 1 ? sm[k - 1] : 0u;
      o.m[i] = __funnelshift_l(lw, hw, r);
    }
    __syncwarp();
  }
  o.e = f + b + (int32_t)cy;
}

// q = RN(a / b), b != 0 (krylov.cu mp_div: restoring division, K = p+3)
template <int K>
__device__ void wdiv(const WMP<K>& a, const WMP<K>& b, WMP<K>& q, uint32_t* sm, int lane) {
  constexpr int L = 32 * K, W = K + 1, KD = 32 * L + 3;
  if (wzero<K>(a) || wzero<K>(b)) { wset_zero<K>(q); return; }
  uint32_t R[W], D[W], Q[W];
  to_wi<K, W>(a.m, R, sm, lane);
  to_wi<K, W>(b.m, D, sm, lane);
#pragma unroll
  for (int i = 0; i < W; ++i) Q[i] = 0u;
  for (int i = 0; i <= KD; ++i) {
    wi_shl1<W>(Q, lane);
    if (!wi_lt<W>(R, D)) {
      wi_sub<W>(R, D, lane);
      if (lane == 0) Q[0] |= 1u;
    }
    wi_shl1<W>(R, lane);
  }
  const bool nz = wi_nonzero<W>(R);
  wi_shl1<W>(Q, lane);
  if (lane == 0 && nz) Q[0] |= 1u;
  wi_round<K, W>(Q, a.e - b.e - KD - 1, sm, lane, q);
  q.s = a.s ^ b.s;
}

// r = RN(sqrt(a)), a >= 0 (krylov.cu mp_sqrt: digit by digit, K = p/2 + 3)
template <int K>
__device__ void wsqrt(const WMP<K>& a, WMP<K>& r, uint32_t* sm, int lane) {
  constexpr int L = 32 * K, W = 2 * K + 1, KS = 16 * L + 3;
  if (wzero<K>(a)) { wset_zero<K>(r); return; }
  int32_t e = a.e - 32 * L;
  uint32_t X[W], Rt[W], T[W];
  to_wi<K, W>(a.m, X, sm, lane);
#pragma unroll
  for (int i = 0; i < W; ++i) Rt[i] = 0u;
  if (e & 1) { wi_shl1<W>(X, lane); e -= 1; }
  wi_shl<W>(X, 2 * KS, sm, lane);
  int pos = (wi_bitlen<W>(X, lane) - 1) & ~1;      // highest power of 4 <= X
  for (; pos >= 0; pos -= 2) {
#pragma unroll
    for (int i = 0; i < W; ++i) T[i] = Rt[i];
    wi_add_bit<W>(T, pos, lane);                     // T = res + bit
    wi_shr1<W>(Rt, lane);
    if (!wi_lt<W>(X, T)) {
      wi_sub<W>(X, T, lane);
      wi_add_bit<W>(Rt, pos, lane);
    }
  }
  const bool nz = wi_nonzero<W>(X);
  wi_shl1<W>(Rt, lane);
  if (lane == 0 && nz) Rt[0] |= 1u;
  wi_round<K, W>(Rt, e / 2 - KS - 1, sm, lane, r);
  r.s = 0u;
}

// exact comparison: -1, 0, 1 (warp-uniform)
template <int K>
__device__ int wcmp(const WMP<K>& a, const WMP<K>& b) {
  const bool az = wzero<K>(a), bz = wzero<K>(b);
  const int ga = az ? 0 : (a.s ? -1 : 1);
  const int gb = bz ? 0 : (b.s ? -1 : 1);
  if (ga != gb) return ga < gb ? -1 : 1;
  if (ga == 0) return 0;
  int c = (a.e > b.e) - (a.e < b.e);
  if (c == 0) {
    c = wi_lt<K>(b.m, a.m) ? 1 : (wi_lt<K>(a.m, b.m) ? -1 : 0);
  }
  return ga > 0 ? c : -c;
}

// ----------------------------------------------------------- load / store
template <int K>
__device__ __forceinline__ void wload(const VecIn& v, int64_t k, int lane, WMP<K>& a) {
  constexpr int L = 32 * K;
  load_k<K>(v.limbs + k * L + lane * K, a.m);
  a.e = __ldg(v.exps + k);
  a.s = __ldg(v.signs + k);
  if (wzero<K>(a)) { a.e = 0; a.s = 0u; }
}

template <int K>
__device__ __forceinline__ void wstore(const YView& y, int64_t k, int lane, const WMP<K>& a) {
  constexpr int L = 32 * K;
  const bool z = wzero<K>(a);
#pragma unroll
  for (int i = 0; i < K; ++i) y.limbs[k * L + lane * K + i] = a.m[i];
  if (lane == 0) {
    y.exps[k] = z ? 0 : a.e;
    y.signs[k] = z ? (uint8_t)0 : (uint8_t)a.s;
  }
}

// ------------------------------------------------------------------ kernels
constexpr int KW = 4;                                // warps per block

// t_k = RN(u_k v_k) into the scratch vector P (ABI element layout)
template <int K>
__global__ void __launch_bounds__(32 * KW) wdot_products(int64_t n, VecIn u, VecIn v, YView P,
                                                         double* fp, const int* stop) {
  constexpr int L = 32 * K;
  if (stop && *stop) return;
  extern __shared__ uint32_t wsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* sA = wsm + warp * 8 * L;
  for (int64_t k = (int64_t)blockIdx.x * KW + warp; k < n; k += (int64_t)gridDim.x * KW) {
    WMP<K> a, b, t;
    wload<K>(u, k, lane, a);
    wload<K>(v, k, lane, b);
    wmul<K>(a.m, a.e, a.s, b.m, b.e, b.s, sA, sA + L, sA + 2 * L, lane, t);
    wstore<K>(P, k, lane, t);
    if (fp && lane == 31) {                        // fp64 estimate from the top two limbs
      const unsigned long long top = ((unsigned long long)t.m[K - 1] << 32) | t.m[K - 2];
      const double dv = t.m[K - 1] ? ldexp(__ull2double_rn(top), t.e - 64) : 0.0;
      fp[k] = t.s ? -dv : dv;
    }
    __syncwarp();
  }
}

// ------------------------------------------- segmented speculative dot chain
// (krylov.cu's segmented dot, on warp-distributed values)
//  S1: the products t_k and fp64 estimates (wdot_products);
//  S2: fp64 sum per segment of WSEG products;
//  S3 (a warp per segment s >= 1): the accumulator's binade E_g and sign at
//      the segment start GUESSED from the fp64 prefix; each step's grid
//      increment Q_k = +-RN_int(|t_k| / 2^(E_g - p)) is added EXACTLY to a
//      two's complement big integer R (W words per lane), the minimum and
//      maximum of the partial sums R_k recorded; a tie on the grid or a
//      product reaching the binade (t.e >= E_g) invalidates the segment;
//  S4 (one warp): the chain walks the segments in order; when the exact state
//      s = S 2^(E - p) has E = E_g, the guessed sign, and S + min >= 2^(p-1)+1,
//      S + max <= 2^p - 1, every step of the segment is S += Q_k on the grid
//      (RN(S u + t_k) = (S + Q_k) u: no tie, no binade change), so S += R;
//      any other segment is walked step by step with wadd from the stored
//      products.  The result is the ordered chain's, bit for bit.
#ifndef MPSP_WSEG
#define MPSP_WSEG 64
#endif
#ifndef MPSP_WSUB
#define MPSP_WSUB 16
#endif
constexpr int WSEG = MPSP_WSEG;
// Lower levels: a segment that fails validation is retried as WSEG / WSUB
// sub-segments with their own speculation records (guessed from the fp64
// prefix at each sub-segment start), a failing sub-segment as WSUB / WSUB2
// third-level segments, and only those that fail are walked element by
// element (BiCG at p = 2048: 17% of the 64-element segments failed, and
// their walks dominated the solve).  Measured, BiCG / GPBiCG per iteration
// at p = 2048 (n = 84,617): one level 28.9 / 91.8 ms; (64, 16) 20.5 / 63.2;
// (64, 16, 4) 19.9 / 60.0; (64, 16, 8) 19.2 / 58.0; (64, 16, 2) 30.1 / 75.6;
// (64, 8) 22.3 / 60.5; (128, 16) 20.0 / 63.4; (128, 32) 22.9 / 74.1.
constexpr int WSUB = MPSP_WSUB;
#ifndef MPSP_WSUB2
#define MPSP_WSUB2 8
#endif
constexpr int WSUB2 = MPSP_WSUB2;                 // third level (0: none)
static_assert(WSEG % WSUB == 0, "sub-segments tile a segment");
static_assert(WSUB2 == 0 || WSUB % WSUB2 == 0, "third-level segments tile a sub-segment");

template <int K>
struct WSeg {
  static constexpr int W = K + 1;                  // big-integer words per lane
  double* fp;          // [n]
  double* segsum;      // [nseg]
  int32_t* valid;      // [nseg]
  int32_t* eg;         // [nseg]
  uint32_t* sg;        // [nseg]
  uint32_t* ds;        // [nseg][32 W]
  uint32_t* mn;        // [nseg][32 W]
  uint32_t* mx;        // [nseg][32 W]
};

template <int K>
__global__ void __launch_bounds__(128) wseg_sums(int64_t n, int64_t nseg, int seglen, WSeg<K> G,
                                                 const int* stop) {
  if (stop && *stop) return;
  const int64_t seg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (seg >= nseg) return;
  double acc = 0.0;
  for (int j = lane; j < seglen; j += 32) {
    const int64_t k = seg * seglen + j;
    if (k < n) acc += G.fp[k];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
  if (lane == 0) G.segsum[seg] = acc;
}

// signed a < b for two's complement big integers
template <int W>
__device__ __forceinline__ bool wi_slt(const uint32_t (&a)[W], const uint32_t (&b)[W], int lane) {
  uint32_t x[W], y[W];
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const uint32_t f = (lane == 31 && i == W - 1) ? 0x80000000u : 0u;
    x[i] = a[i] ^ f;
    y[i] = b[i] ^ f;
  }
  return wi_lt<W>(x, y);
}

template <int W>
__device__ __forceinline__ void wi_load(const uint32_t* g, uint32_t (&a)[W], int lane) {
#pragma unroll
  for (int i = 0; i < W; ++i) a[i] = g[lane * W + i];
}
template <int W>
__device__ __forceinline__ void wi_store(uint32_t* g, const uint32_t (&a)[W], int lane) {
#pragma unroll
  for (int i = 0; i < W; ++i) g[lane * W + i] = a[i];
}

template <int K>
__global__ void __launch_bounds__(32 * KW) wseg_speculate(int64_t n, int64_t nseg, int seglen, VecIn P,
                                                          WSeg<K> G, const int* stop) {
  constexpr int L = 32 * K, W = K + 1, PB = 32 * L;
  if (stop && *stop) return;
  extern __shared__ uint32_t wsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t seg = (int64_t)blockIdx.x * KW + warp;
  if (seg >= nseg || seg == 0) return;
  uint32_t* sm = wsm + warp * 8 * L;               // 2L + 34 words used
  const double pre = G.segsum[seg];               // fp64 prefix (launch_dot_prefix)
  int e2 = 0;
  frexp(fabs(pre), &e2);
  bool valid = pre != 0.0 && isfinite(pre);
  const int32_t Eg = e2;
  const uint32_t sgg = pre < 0.0 ? 1u : 0u;
  uint32_t R[W], mn[W], mx[W];
#pragma unroll
  for (int i = 0; i < W; ++i) { R[i] = 0u; mn[i] = 0u; mx[i] = 0u; }
  for (int j = 0; j < seglen && valid; ++j) {
    const int64_t k = seg * seglen + j;
    if (k >= n) break;
    WMP<K> t;
    wload<K>(P, k, lane, t);
    if (wzero<K>(t)) continue;
    const int64_t d = (int64_t)Eg - (int64_t)t.e;   // |t| / u = M_t / 2^d
    if (d < 1) { valid = false; break; }            // reaches the binade
    if (d > PB + 2) continue;                       // |t| < u/4: Q = 0
    // Y = floor(M_t / 2^d), rb = bit d-1, sticky = bits below it
    __syncwarp();
#pragma unroll
    for (int i = 0; i < K; ++i) { sm[lane * K + i] = t.m[i]; sm[L + 1 + lane * K + i] = 0u; }
    if (lane == 0) { sm[L] = 0u; sm[2 * L + 1] = 0u; sm[2 * L + 2] = 0u; }
    __syncwarp();
    const int q = (int)(d >> 5);
    const uint32_t r = (uint32_t)d & 31u;
    uint32_t Q[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const int m = lane * W + i + q;               // source word of Y word lane*W+i
      const uint32_t lo_ = m <= 2 * L + 1 ? sm[m] : 0u;
      const uint32_t hi_ = m + 1 <= 2 * L + 1 ? sm[m + 1] : 0u;
      Q[i] = (m < 2 * L + 2) ? __funnelshift_r(lo_, hi_, r) : 0u;
    }
    const int64_t rp = d - 1;                       // round bit position in M_t
    const uint32_t rb = (sm[rp >> 5] >> (rp & 31)) & 1u;
    uint32_t orr = 0u;
    for (int w = lane; w < (int)(rp >> 5); w += 32) orr |= sm[w];
    if (lane == 0) orr |= sm[rp >> 5] & ((1u << (rp & 31)) - 1u);
    const bool sticky = __ballot_sync(FULL, orr != 0u) != 0u;
    __syncwarp();
    if (rb && !sticky) { valid = false; break; }    // grid tie: needs the parity of S
    if (rb) {
      uint32_t one[W];
#pragma unroll
      for (int i = 0; i < W; ++i) one[i] = (lane == 0 && i == 0) ? 1u : 0u;
      wi_add<W>(Q, one, lane);
    }
    if (t.s == sgg) wi_add<W>(R, Q, lane); else wi_sub<W>(R, Q, lane);
    if (wi_slt<W>(R, mn, lane)) {
#pragma unroll
      for (int i = 0; i < W; ++i) mn[i] = R[i];
    }
    if (wi_slt<W>(mx, R, lane)) {
#pragma unroll
      for (int i = 0; i < W; ++i) mx[i] = R[i];
    }
  }
  if (lane == 0) {
    G.valid[seg] = valid ? 1 : 0;
    G.eg[seg] = Eg;
    G.sg[seg] = sgg;
  }
  wi_store<W>(G.ds + seg * 32 * W, R, lane);
  wi_store<W>(G.mn + seg * 32 * W, mn, lane);
  wi_store<W>(G.mx + seg * 32 * W, mx, lane);
}

// diagnostics: segments walked element by element / committed (added to
// mpsp_debug_dot_stats' counters)
__device__ unsigned long long g_wdot_stats[2];

template <int K>
__global__ void __launch_bounds__(32) wseg_chain(int64_t n, int64_t nseg, VecIn P, WSeg<K> G,
                                                 WSeg<K> Gs, WSeg<K> Gt, YView out, const int* stop) {
  constexpr int L = 32 * K, W = K + 1;
  if (stop && *stop) return;
  extern __shared__ uint32_t wsm[];
  const int lane = threadIdx.x & 31;
  uint32_t LO[W], HI[W];                            // 2^(p-1) + 1, 2^p - 1
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const int w = lane * W + i;
    LO[i] = w == 0 ? 1u : (w == L - 1 ? 0x80000000u : 0u);
    HI[i] = w < L ? 0xffffffffu : 0u;
  }
  WMP<K> s;
  wset_zero<K>(s);
  // commit segment j of the records R if its guess and bounds hold for the
  // exact state s (then every step was S += Q_k on the grid: S += ds)
  // one segment's speculation record, loaded with every load issued up
  // front (one memory latency on the lone chain warp's path instead of four)
  struct Rec {
    int v;
    int32_t eg;
    uint32_t sg;
    uint32_t Mn[W], Mx[W], D[W];
  };
  auto load_rec = [&](const WSeg<K>& R, int64_t j, Rec& r) {
    r.v = R.valid[j];
    r.eg = R.eg[j];
    r.sg = R.sg[j];
    wi_load<W>(R.mn + j * 32 * W, r.Mn, lane);
    wi_load<W>(R.mx + j * 32 * W, r.Mx, lane);
    wi_load<W>(R.ds + j * 32 * W, r.D, lane);
  };
  auto commit_rec = [&](const Rec& r, int64_t j) -> bool {
    const int vj = r.v;
    const int32_t egj = r.eg;
    const uint32_t sgj = r.sg;
    const uint32_t(&Mn)[W] = r.Mn;
    const uint32_t(&Mx)[W] = r.Mx;
    uint32_t D[W];
#pragma unroll
    for (int i = 0; i < W; ++i) D[i] = r.D[i];
    bool ok = j > 0 && vj && !wzero<K>(s) && egj == s.e && sgj == s.s;
    if (lane == 0) atomicAdd(&g_wdot_stats[ok ? 1 : 0], 1ull);
    if (!ok) return false;
    uint32_t S[W];
    to_wi<K, W>(s.m, S, wsm, lane);
    uint32_t A[W], B[W];
#pragma unroll
    for (int i = 0; i < W; ++i) A[i] = S[i];
    wi_add<W>(A, Mn, lane);
#pragma unroll
    for (int i = 0; i < W; ++i) B[i] = S[i];
    wi_add<W>(B, Mx, lane);
    if (wi_slt<W>(A, LO, lane) || wi_slt<W>(HI, B, lane)) return false;   // warp-uniform
    wi_add<W>(S, D, lane);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < W; ++i) wsm[lane * W + i] = S[i];
    __syncwarp();
#pragma unroll
    for (int i = 0; i < K; ++i) s.m[i] = wsm[lane * K + i];
    __syncwarp();
    return true;
  };
  auto try_commit = [&](const WSeg<K>& R, int64_t j) -> bool {
    Rec r;
    load_rec(R, j, r);
    return commit_rec(r, j);
  };
  auto walk = [&](int64_t k0, int64_t k1) {
    WMP<K> t;
    for (int64_t k = k0; k < k1; ++k) {
      wload<K>(P, k, lane, t);
      wadd<K>(s, t, wsm, lane);
      __syncwarp();
    }
  };
  constexpr int NSUB = WSEG / WSUB;
  Rec cur, nxt;
  if (nseg > 0) load_rec(G, 0, cur);
  for (int64_t seg = 0; seg < nseg; ++seg) {
    if (seg + 1 < nseg) load_rec(G, seg + 1, nxt);  // in flight during this segment
    const bool done = commit_rec(cur, seg);
    cur = nxt;
    if (done) continue;
    for (int u = 0; u < NSUB; ++u) {               // the segment's sub-segments
      const int64_t j = seg * NSUB + u;
      const int64_t k0 = j * WSUB;
      if (k0 >= n) break;
      if (try_commit(Gs, j)) continue;
      if constexpr (WSUB2 > 0) {
        constexpr int NSUB2 = WSUB / (WSUB2 > 0 ? WSUB2 : 1);
        for (int v = 0; v < NSUB2; ++v) {          // and theirs
          const int64_t jj = j * NSUB2 + v;
          const int64_t kk = jj * WSUB2;
          if (kk >= n) break;
          if (!try_commit(Gt, jj)) walk(kk, min(n, kk + WSUB2));
        }
      } else {
        walk(k0, min(n, k0 + WSUB));
      }
    }
  }
  wstore<K>(out, 0, lane, s);
}

// z_k = RN(y_k + RN(+-alpha x_k))
template <int K>
__global__ void __launch_bounds__(32 * KW) waxpy(int64_t n, VecIn alpha, int negate, VecIn x, VecIn y,
                                                 YView z, const int* stop) {
  constexpr int L = 32 * K;
  if (stop && *stop) return;
  extern __shared__ uint32_t wsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* sA = wsm + warp * 8 * L;
  WMP<K> al;
  wload<K>(alpha, 0, lane, al);
  for (int64_t k = (int64_t)blockIdx.x * KW + warp; k < n; k += (int64_t)gridDim.x * KW) {
    WMP<K> xv, s, t;
    wload<K>(x, k, lane, xv);
    wload<K>(y, k, lane, s);
    wmul<K>(al.m, al.e, al.s ^ (uint32_t)negate, xv.m, xv.e, xv.s, sA, sA + L, sA + 2 * L, lane, t);
    wadd<K>(s, t, sA + 2 * L, lane);
    wstore<K>(z, k, lane, s);
    __syncwarp();
  }
}

enum { S_RHO = KS_RHO, S_RHOP = KS_RHOP, S_SIGMA = KS_SIGMA, S_ALPHA = KS_ALPHA, S_BETA = KS_BETA,
       S_RR = KS_RR, S_NRM = KS_NRM, S_THR = KS_THR, S_C1 = KS_C1, S_C2 = KS_C2, S_ONE = KS_ONE,
       S_T20 = KS_T20, S_T50 = KS_T50, S_ALPHAP = KS_ALPHAP, S_ZETA = KS_ZETA, S_ETA = KS_ETA,
       S_MU1 = KS_MU1, S_MU2 = KS_MU2, S_MU3 = KS_MU3, S_MU4 = KS_MU4, S_MU5 = KS_MU5,
       S_TAU = KS_TAU };
enum { F_STOP = KF_STOP, F_BREAK = KF_BREAK, F_CONV = KF_CONV, F_BRK2 = KF_BRK2 };

// the scalar steps of krylov.cu bicg_scalar (same op numbers), one warp
template <int K>
__global__ void __launch_bounds__(32) wscalar(YView S, int* fl, int op) {
  constexpr int L = 32 * K;
  if (fl[F_STOP]) return;
  extern __shared__ uint32_t wsm[];
  const int lane = threadIdx.x & 31;
  uint32_t* sA = wsm;
  uint32_t* sX = wsm + L;
  uint32_t* cs = wsm + 2 * L;                        // 6L words: wmul / wadd / big-int scratch
  const VecIn Sv{S.limbs, S.exps, S.signs};
  auto ld = [&](int i, WMP<K>& a) { wload<K>(Sv, i, lane, a); };
  auto st = [&](int i, const WMP<K>& a) { wstore<K>(S, i, lane, a); __syncwarp(); };
  auto mul = [&](const WMP<K>& a, const WMP<K>& b, WMP<K>& o) {
    wmul<K>(a.m, a.e, a.s, b.m, b.e, b.s, sA, sX, cs, lane, o);
    __syncwarp();
  };
  auto add = [&](WMP<K>& s, const WMP<K>& t) { wadd<K>(s, t, cs, lane); __syncwarp(); };
  auto det = [&](const WMP<K>& a, const WMP<K>& b, const WMP<K>& c, const WMP<K>& d, WMP<K>& o) {
    WMP<K> t;
    mul(a, b, o);
    mul(c, d, t);
    t.s ^= 1u;
    add(o, t);
  };
  auto div = [&](const WMP<K>& a, const WMP<K>& b, WMP<K>& o) { wdiv<K>(a, b, o, cs, lane); __syncwarp(); };
  auto sqr = [&](const WMP<K>& a, WMP<K>& o) { wsqrt<K>(a, o, cs, lane); __syncwarp(); };
  auto flag = [&](int f) { if (lane == 0) fl[f] = 1; };
  WMP<K> a, b, c;
  switch (op) {
    case 0: {
      WMP<K> c1, t;
      ld(S_ONE, a);
      ld(S_T20, b);
      div(a, b, c1);
      st(S_C1, c1);
      ld(S_T50, b);
      div(a, b, c);
      st(S_C2, c);
      ld(S_RR, a);
      sqr(a, b);                                     // nrm0
      mul(c1, b, t);
      add(t, c);
      st(S_THR, t);
      break;
    }
    case 1:
      ld(S_RHO, a);
      if (wzero<K>(a)) { flag(F_BREAK); flag(F_STOP); }
      break;
    case 2:
      ld(S_RHO, a);
      ld(S_RHOP, b);
      div(a, b, c);
      st(S_BETA, c);
      break;
    case 3:
      ld(S_RHO, a);
      ld(S_SIGMA, b);
      if (wzero<K>(b)) { flag(F_BREAK); flag(F_STOP); break; }
      div(a, b, c);
      st(S_ALPHA, c);
      break;
    case 4:
      ld(S_RR, a);
      sqr(a, b);
      st(S_NRM, b);
      ld(S_THR, c);
      if (wcmp<K>(b, c) <= 0) { flag(F_CONV); flag(F_STOP); }
      ld(S_RHO, a);
      st(S_RHOP, a);
      break;
    case 5:
      ld(S_MU2, a);
      ld(S_MU5, b);
      if (wzero<K>(b)) wset_zero<K>(c); else div(a, b, c);
      st(S_ZETA, c);
      wset_zero<K>(c);
      st(S_ETA, c);
      break;
    case 6: {
      WMP<K> d, e;
      ld(S_RHO, a);
      ld(S_RHOP, b);
      div(a, b, c);
      ld(S_ALPHAP, a);
      ld(S_ZETA, b);
      div(a, b, d);
      mul(c, d, e);
      st(S_BETA, e);
      break;
    }
    case 7: {
      WMP<K> m1, m2, m3, m4, m5, tau, num;
      ld(S_MU1, m1);
      ld(S_MU2, m2);
      ld(S_MU3, m3);
      ld(S_MU4, m4);
      ld(S_MU5, m5);
      det(m5, m1, m4, m4, tau);
      st(S_TAU, tau);
      if (wzero<K>(tau)) { flag(F_BREAK); flag(F_STOP); break; }
      det(m1, m2, m3, m4, num);
      div(num, tau, c);
      st(S_ZETA, c);
      det(m5, m3, m4, m2, num);
      div(num, tau, c);
      st(S_ETA, c);
      break;
    }
    case 8:
      ld(S_RR, a);
      sqr(a, b);
      st(S_NRM, b);
      ld(S_THR, c);
      if (wcmp<K>(b, c) <= 0) {
        flag(F_CONV); flag(F_STOP);
      } else {
        ld(S_ZETA, a);
        if (wzero<K>(a)) { flag(F_BRK2); flag(F_STOP); }
      }
      ld(S_RHO, a);
      st(S_RHOP, a);
      ld(S_ALPHA, a);
      st(S_ALPHAP, a);
      break;
  }
}

template <int K>
struct WideOps {
  static constexpr int L = 32 * K;
  static constexpr size_t SM = (size_t)8 * L * 4;   // per-warp shared memory (bytes)
  template <class Kern>
  static int attr(Kern k, size_t bytes) {
    return (int)cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  }
  static size_t rec_bytes(size_t nseg) {          // one level's speculation records
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    constexpr int W = K + 1;
    return al(nseg * 8) + 3 * al(nseg * 4) + 3 * al(nseg * 32 * W * 4);
  }
  static size_t bytes(int64_t n) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t nseg = (size_t)((n + WSEG - 1) / WSEG), nsub = (size_t)((n + WSUB - 1) / WSUB);
    const size_t nsub2 = WSUB2 > 0 ? (size_t)((n + WSUB2 - 1) / WSUB2) : 1;
    return al((size_t)n * L * 4) + al((size_t)n * 4) + al((size_t)n) + al((size_t)n * 8) +
           rec_bytes(nseg) + rec_bytes(nsub) + rec_bytes(nsub2);
  }
  // carve one level's records out of p
  static WSeg<K> records(char*& p, double* fp, size_t nseg) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    constexpr int W = K + 1;
    WSeg<K> G;
    G.fp = fp;
    G.segsum = (double*)p; p += al(nseg * 8);
    G.valid = (int32_t*)p; p += al(nseg * 4);
    G.eg = (int32_t*)p; p += al(nseg * 4);
    G.sg = (uint32_t*)p; p += al(nseg * 4);
    G.ds = (uint32_t*)p; p += al(nseg * 32 * W * 4);
    G.mn = (uint32_t*)p; p += al(nseg * 32 * W * 4);
    G.mx = (uint32_t*)p; p += al(nseg * 32 * W * 4);
    return G;
  }
  static int dot(int64_t n, VecIn u, VecIn v, YView out, const int* stop, cudaStream_t st, void* work) {
    if (!work && n > 0) return (int)cudaErrorInvalidValue;
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const int64_t nseg = (n + WSEG - 1) / WSEG, nsub = (n + WSUB - 1) / WSUB;
    const int64_t nsub2 = WSUB2 > 0 ? (n + WSUB2 - 1) / WSUB2 : 1;
    char* p = (char*)work;
    YView P{(uint32_t*)p, (int32_t*)(p + al((size_t)n * L * 4)),
            (uint8_t*)(p + al((size_t)n * L * 4) + al((size_t)n * 4))};
    p += al((size_t)n * L * 4) + al((size_t)n * 4) + al((size_t)n);
    double* fp = (double*)p;
    p += al((size_t)n * 8);
    const WSeg<K> G = records(p, fp, (size_t)nseg);
    const WSeg<K> Gs = records(p, fp, (size_t)nsub);
    const WSeg<K> Gt = records(p, fp, (size_t)nsub2);
    const VecIn Pin{P.limbs, P.exps, P.signs};
    int e;
    if (n > 0) {
      if ((e = attr(wdot_products<K>, KW * SM))) return e;
      const int64_t blocks = std::min<int64_t>((n + KW - 1) / KW, 148 * 16);
      wdot_products<K><<<(unsigned)blocks, 32 * KW, KW * SM, st>>>(n, u, v, P, fp, stop);
      if ((e = attr(wseg_speculate<K>, KW * SM))) return e;
      for (int lev = 0; lev < (WSUB2 > 0 ? 3 : 2); ++lev) {   // the segment levels
        const WSeg<K>& R = lev == 0 ? G : (lev == 1 ? Gs : Gt);
        const int64_t ns = lev == 0 ? nseg : (lev == 1 ? nsub : nsub2);
        const int len = lev == 0 ? WSEG : (lev == 1 ? WSUB : WSUB2);
        wseg_sums<K><<<(unsigned)((ns * 32 + 127) / 128), 128, 0, st>>>(n, ns, len, R, stop);
        if ((e = launch_dot_prefix(R.segsum, ns, stop, st))) return e;
        wseg_speculate<K><<<(unsigned)((ns + KW - 1) / KW), 32 * KW, KW * SM, st>>>(n, ns, len, Pin, R,
                                                                                stop);
      }
      launch_counter_add(WSUB2 > 0 ? 7 : 5);
    }
    if ((e = attr(wseg_chain<K>, SM))) return e;
    wseg_chain<K><<<1, 32, SM, st>>>(n, nseg, Pin, G, Gs, Gt, out, stop);
    launch_counter_add(1);
    return (int)cudaGetLastError();
  }
  static int axpy(int64_t n, VecIn a, int neg, VecIn x, VecIn y, YView z, const int* stop, cudaStream_t st) {
    if (n <= 0) return 0;
    int e;
    if ((e = attr(waxpy<K>, KW * SM))) return e;
    const int64_t blocks = std::min<int64_t>((n + KW - 1) / KW, 148 * 16);
    waxpy<K><<<(unsigned)blocks, 32 * KW, KW * SM, st>>>(n, a, neg, x, y, z, stop);
    launch_counter_add(1);
    return (int)cudaGetLastError();
  }
  static int scalar(YView S, int* fl, int op, cudaStream_t st) {
    int e;
    if ((e = attr(wscalar<K>, SM))) return e;
    wscalar<K><<<1, 32, SM, st>>>(S, fl, op);
    launch_counter_add(1);
    return (int)cudaGetLastError();
  }
};

}  // namespace wide

int krylov_wide_dot(int L, int64_t n, const VecIn& u, const VecIn& v, const YView& out, const int* stop,
                    void* stream, void* work) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 64: return wide::WideOps<2>::dot(n, u, v, out, stop, st, work);
    case 128: return wide::WideOps<4>::dot(n, u, v, out, stop, st, work);
    case 256: return wide::WideOps<8>::dot(n, u, v, out, stop, st, work);
    default: return (int)cudaErrorInvalidValue;
  }
}

size_t krylov_wide_dot_work_bytes(int L, int64_t n) {
  switch (L) {
    case 64: return wide::WideOps<2>::bytes(n);
    case 128: return wide::WideOps<4>::bytes(n);
    case 256: return wide::WideOps<8>::bytes(n);
    default: return 0;
  }
}

int krylov_wide_axpy(int L, int64_t n, const VecIn& al, int neg, const VecIn& x, const VecIn& y,
                     const YView& z, const int* stop, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 64: return wide::WideOps<2>::axpy(n, al, neg, x, y, z, stop, st);
    case 128: return wide::WideOps<4>::axpy(n, al, neg, x, y, z, stop, st);
    case 256: return wide::WideOps<8>::axpy(n, al, neg, x, y, z, stop, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

int krylov_wide_scalar(int L, const YView& S, int* fl, int op, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 64: return wide::WideOps<2>::scalar(S, fl, op, st);
    case 128: return wide::WideOps<4>::scalar(S, fl, op, st);
    case 256: return wide::WideOps<8>::scalar(S, fl, op, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

// [walked, committed] segments of the p > 1024 dot chain since the last
// call (then reset); mpsp_debug_dot_stats adds them to the narrow chain's
int krylov_wide_dot_stats(unsigned long long out[2]) {
  cudaError_t e = cudaMemcpyFromSymbol(out, wide::g_wdot_stats, sizeof(unsigned long long) * 2);
  if (e == cudaSuccess) {
    const unsigned long long z[2] = {0ull, 0ull};
    e = cudaMemcpyToSymbol(wide::g_wdot_stats, z, sizeof z);
  }
  return (int)e;
}

}  // namespace mpsp
