// krylov.cu - multiple-precision BiCG and GPBiCG on the GPU (SURVEY.md 8(f)
// ranks 1-2): PAPER.md:249-369 (Fig. 4) with K = I, the SpMVs by this
// library's kernels, and PAPER.md:375-380 (convergence test
// ||r|| <= 1e-20 ||r_0|| + 1e-50).  Every operation is one p-bit RN
// operation in the order the figure writes it (readings c26-c35);
// p > 1024 runs the same steps on warp-distributed values (krylov_wide.cu).
//   dot      (u, v) = ordered chain s = RN(s + RN(u_k v_k)), k ascending
//            (segments evaluated speculatively in parallel and validated in
//            order by one warp; the exact speculative block sum of
//            wchain.cuh for the segments that do not validate)
//   axpy     z_k = RN(y_k + RN(+-alpha x_k))            (thread per element)
//   scalars  RN(a / b), RN(sqrt(a)), exact compare      (one thread:
//            integer long division / square root + one rounding)
// The host loop keeps every value on the device; one 3-int flag read per
// iteration decides breakdown / convergence (kernels after a stop flag do
// nothing, so x keeps the last complete iterate, as in the oracle).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstring>
#include <vector>

#include "../../include/mpsp.h"
#include "kernel_common.cuh"
#include "wchain.cuh"

namespace mpsp {

template <int L>
__device__ __forceinline__ void load_mp(const VecIn& v, int64_t k, MP<L>& a) {
  const uint32_t* base = v.limbs + k * L;
  using C = Chunk<L>;
  constexpr int NC = L / C::CW;
  const typename C::T* p = reinterpret_cast<const typename C::T*>(base);
#pragma unroll
  for (int c = 0; c < NC; ++c) unpack_chunk(__ldg(p + c), &a.m[c * C::CW]);
  a.e = __ldg(v.exps + k);
  a.s = __ldg(v.signs + k);
}

// ---------------------------------------------------------------- kernels
template <int L>
__global__ void __launch_bounds__(32) vec_dot(int64_t n, VecIn u, VecIn v, YView out,
                                              const int* stop) {
  if (stop && *stop) return;
  const int lane = threadIdx.x & 31;
  WChain<L> ch;
  ch.init();
  for (int64_t b = 0; b < n; b += 32) {
    const int64_t k = b + lane;
    MP<L> t;
    if (k < n) {
      MP<L> a, c;
      load_mp<L>(u, k, a);
      load_mp<L>(v, k, c);
      mp_mul<L>(a.m, a.e, a.s, c.m, c.e, c.s, t);
    } else {
      t.set_zero();
    }
    ch.consume(t, lane);
  }
  MP<L> s;
  ch.exact(s);
  if (lane == 0) store_y<L>(out, 0, s);
}

// ---------------------------------------------------------------------------
// Fast exact dot: the chain split into segments of DSEG steps, evaluated
// speculatively in parallel and validated in order.
//  D1 (warp per segment): products t_k into a scratch array, and an fp64
//     estimate of the segment's sum;
//  D2 (warp per segment s >= 1): the accumulator's binade E_g and sign at the
//     segment start are GUESSED from the fp64 prefix sum; every step's grid
//     increment Q_k against (E_g, sign) is formed (align_q), summed exactly
//     (dS), and the relative high-part prefix bounds of the segment's partial
//     sums (minv, maxv) recorded; a tie or a step reaching the binade makes
//     the segment invalid;
//  D3 (one warp): the chain itself (WChain) walks the segments in order: a
//     segment whose guess matches the exact state (E, sign) and whose bounds
//     hold for the exact Shi / err is committed by adding dS (32 segments
//     validated per warp step, by scans of the segments' h sums and step
//     counts); any other segment is evaluated step by step from the stored
//     products.  Validation uses exactly the conditions WChain::consume
//     checks block by block, so the result is the ordered chain's, bit for bit.
// ---------------------------------------------------------------------------
#ifndef MPSP_DSEG_NB
#define MPSP_DSEG_NB 4
#endif
constexpr int DSEG_NB = MPSP_DSEG_NB;            // blocks of 32 steps per segment
constexpr int DSEG = 32 * DSEG_NB;

struct DotWork {                                  // device scratch (sizes: dot_work_bytes)
  uint32_t* prod;                                 // [nblk][L+2][32] products
  double* segsum;                                 // [nseg]
  int32_t* valid;                                 // [nseg]
  int32_t* eg;                                    // [nseg]
  uint32_t* sg;                                   // [nseg]
  long long* minv;                                // [nseg]
  long long* maxv;                                // [nseg]
  long long* htot;                                // [nseg]
  uint32_t* ds;                                    // [nseg][L+2] exact segment sums
};

template <int L>
__device__ __forceinline__ double mp_to_f64(const MP<L>& t) {
  if (t.is_zero()) return 0.0;
  const unsigned long long top = ((unsigned long long)t.m[L - 1] << 32) | (L > 1 ? t.m[L > 1 ? L - 2 : 0] : 0u);
  const double d = ldexp(__ull2double_rn(top), t.e - 64);
  return t.s ? -d : d;
}

template <int L>
__global__ void __launch_bounds__(128) dot_products(int64_t n, VecIn u, VecIn v, DotWork W,
                                                    int64_t nseg, const int* stop) {
  if (stop && *stop) return;
  const int64_t seg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (seg >= nseg) return;
  double acc = 0.0;
  for (int b = 0; b < DSEG_NB; ++b) {
    const int64_t blk = seg * DSEG_NB + b;
    const int64_t k = blk * 32 + lane;
    MP<L> t;
    if (k < n) {
      MP<L> a, c;
      load_mp<L>(u, k, a);
      load_mp<L>(v, k, c);
      mp_mul<L>(a.m, a.e, a.s, c.m, c.e, c.s, t);
    } else {
      t.set_zero();
    }
    uint32_t* P = W.prod + blk * (L + 2) * 32;
#pragma unroll
    for (int i = 0; i < L; ++i) P[i * 32 + lane] = t.m[i];
    P[L * 32 + lane] = (uint32_t)t.e;
    P[(L + 1) * 32 + lane] = t.s;
    acc += mp_to_f64<L>(t);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) W.segsum[seg] = acc;
}

template <int L>
__device__ __forceinline__ void load_prod(const DotWork& W, int64_t blk, int lane, MP<L>& t) {
  const uint32_t* P = W.prod + blk * (L + 2) * 32;
#pragma unroll
  for (int i = 0; i < L; ++i) t.m[i] = P[i * 32 + lane];
  t.e = (int32_t)P[L * 32 + lane];
  t.s = P[(L + 1) * 32 + lane];
}

// Exclusive prefix of the segments' fp64 sums, in place (one block of 1024
// threads, O(nseg)): the guess of each segment's starting binade.  Only
// estimates - a wrong guess just makes a segment fail validation.
__global__ void __launch_bounds__(1024) dot_prefix(double* segsum, int64_t nseg, const int* stop) {
  if (stop && *stop) return;
  __shared__ double part[1024];
  const int t = threadIdx.x;
  const int64_t per = (nseg + 1023) / 1024;
  const int64_t a = (int64_t)t * per, b = min(nseg, a + per);
  double acc = 0.0;
  for (int64_t k = a; k < b; ++k) acc += segsum[k];
  part[t] = acc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {            // inclusive Hillis-Steele scan
    const double v = t >= o ? part[t - o] : 0.0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  double run = t > 0 ? part[t - 1] : 0.0;
  for (int64_t k = a; k < b; ++k) {
    const double v = segsum[k];
    segsum[k] = run;
    run += v;
  }
}

int launch_dot_prefix(double* segsum, int64_t nseg, const int* stop, void* stream) {
  if (nseg <= 0) return 0;
  dot_prefix<<<1, 1024, 0, (cudaStream_t)stream>>>(segsum, nseg, stop);
  launch_counter_add(1);
  return (int)cudaGetLastError();
}

template <int L>
__global__ void __launch_bounds__(128) dot_speculate(DotWork W, int64_t nseg, const int* stop) {
  if (stop && *stop) return;
  constexpr int N = L + 2;
  constexpr unsigned FULL = 0xffffffffu;
  const int64_t seg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (seg >= nseg || seg == 0) return;
  const double pre = W.segsum[seg];                // fp64 prefix (dot_prefix)
  int e2 = 0;
  const double f = frexp(fabs(pre), &e2);
  bool valid = (pre != 0.0) && isfinite(pre) && f > 0.0;
  const int32_t Eg = e2;
  const uint32_t sgg = pre < 0.0 ? 1u : 0u;
  uint32_t R[N];
#pragma unroll
  for (int i = 0; i < N; ++i) R[i] = 0u;
  long long base = 0, mn = LLONG_MAX, mx = LLONG_MIN;
  for (int b = 0; b < DSEG_NB && valid; ++b) {
    MP<L> t;
    load_prod<L>(W, seg * DSEG_NB + b, lane, t);
    const bool act = !t.is_zero();
    uint32_t Q[N];
    int32_t h;
    bool prex;
    align_q<L>(t, act, Eg, sgg, Q, h, prex);
    if (__ballot_sync(FULL, act && prex)) valid = false;
    long long Pi = act ? h : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long x = __shfl_up_sync(FULL, Pi, o);
      if (lane >= o) Pi += x;
    }
    const long long before = base + Pi - (act ? h : 0);
    long long cmn = act ? before + h : LLONG_MAX;
    long long cmx = act ? before + h + b * 32 + lane : LLONG_MIN;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cmn = min(cmn, (long long)__shfl_xor_sync(FULL, cmn, o));
      cmx = max(cmx, (long long)__shfl_xor_sync(FULL, cmx, o));
    }
    mn = min(mn, cmn);
    mx = max(mx, cmx);
    add_n<N>(R, R, Q);
    base += __shfl_sync(FULL, Pi, 31);
  }
  warp_sum_limbs<N>(R);
  if (lane == 0) {
    W.valid[seg] = valid ? 1 : 0;
    W.eg[seg] = Eg;
    W.sg[seg] = sgg;
    W.minv[seg] = mn;
    W.maxv[seg] = mx;
    W.htot[seg] = base;
  }
  if (lane == 0) {                                 // all N limbs (N = L+2 may exceed 32)
#pragma unroll
    for (int i = 0; i < N; ++i) W.ds[seg * N + i] = R[i];
  }
}

// diagnostics: segments evaluated step by step / validated (mpsp_debug_dot_stats)
__device__ unsigned long long g_dot_stats[2];

template <int L>
__global__ void __launch_bounds__(32) dot_chain(int64_t n, DotWork W, int64_t nseg, YView out,
                                                const int* stop) {
  if (stop && *stop) return;
  constexpr int N = L + 2;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr long long LO = 1ll << (HB - 1), HI = 1ll << HB;
  const int lane = threadIdx.x & 31;
  WChain<L> ch;
  ch.init();
  // (block b+1's products are loaded while block b is consumed: the lone
  // chain warp would otherwise wait a full memory latency per block; the
  // first block of a segment to walk is loaded by the caller, before the
  // commits of the segments ahead of it)
  auto sequential = [&](int64_t seg, MP<L>& first) {
    if (lane == 0) atomicAdd(&g_dot_stats[0], 1ull);
    const int64_t b0 = seg * DSEG_NB;
    MP<L> t, tn = first;
    for (int b = 0; b < DSEG_NB; ++b) {
      const int64_t blk = b0 + b;
      if (blk * 32 >= n) break;
      t = tn;
      if (b + 1 < DSEG_NB && (blk + 1) * 32 < n) load_prod<L>(W, blk + 1, lane, tn);
      ch.consume(t, lane);
    }
  };
  auto first_of = [&](int64_t seg, MP<L>& t) {
    if (seg * DSEG_NB * 32 < n) load_prod<L>(W, seg * DSEG_NB, lane, t);
    else t.set_zero();
  };
  // The window of 32 segments [base, base+32): lane j holds segment base+j's
  // speculation record.  After committing f segments and walking segment
  // base+f, the records of base+f+1 .. base+31 move down by f+1 lanes and
  // only the tail is loaded - issued before the walk, so its latency hides
  // behind it.
  int64_t base = 0;
  int wv = 0;
  int32_t weg = 0;
  uint32_t wsg = 0u;
  long long wmn = 0, wmx = 0, wht = 0;
  auto load_rec = [&](int64_t jj) {
    const bool in = jj < nseg;
    wv = in ? W.valid[jj] : 0;
    weg = in ? W.eg[jj] : 0;
    wsg = in ? W.sg[jj] : 0u;
    wmn = in ? W.minv[jj] : 0;
    wmx = in ? W.maxv[jj] : 0;
    wht = in ? W.htot[jj] : 0;
  };
  {
    MP<L> t0;
    first_of(0, t0);
    sequential(0, t0);                          // segment 0 starts from +0
    base = 1;
    load_rec(base + lane);
  }
  while (base < nseg) {
    if (ch.szero) {                             // the chain is exactly zero: walk
      MP<L> t0;
      first_of(base, t0);
      sequential(base, t0);
      const int sh = 1;
      const int64_t jn = base + lane + sh;
      // shift the window down by one lane, load the new tail
      const int v2 = __shfl_down_sync(FULL, wv, sh);
      const int32_t e2 = __shfl_down_sync(FULL, weg, sh);
      const uint32_t s2 = __shfl_down_sync(FULL, wsg, sh);
      const long long m1 = __shfl_down_sync(FULL, wmn, sh), m2 = __shfl_down_sync(FULL, wmx, sh);
      const long long h2 = __shfl_down_sync(FULL, wht, sh);
      if (lane < 32 - sh) { wv = v2; weg = e2; wsg = s2; wmn = m1; wmx = m2; wht = h2; }
      else load_rec(jn);
      base += sh;
      continue;
    }
    const int64_t j = base + lane;
    const bool in = j < nseg;
    const long long ht = in ? wht : 0;
    const long long cn = DSEG;
    long long hi = ht, ci = cn;                     // inclusive scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long x = __shfl_up_sync(FULL, hi, o);
      const long long y = __shfl_up_sync(FULL, ci, o);
      if (lane >= o) { hi += x; ci += y; }
    }
    const long long hpre = hi - ht, cpre = ci - cn;
    bool ok = in && wv && weg == ch.E && wsg == ch.sg;
    ok = ok && ((long long)ch.Shi + hpre + wmn - 1 >= LO) &&
         ((long long)ch.Shi + hpre + (long long)ch.err + cpre + wmx + 1 <= HI);
    const unsigned failM = __ballot_sync(FULL, !ok);
    const int f = failM ? __ffs(failM) - 1 : 32;
    const bool walk = f < 32 && base + f < nseg;
    MP<L> t0;
    if (walk) first_of(base + f, t0);              // in flight during the commits
    if (f > 0) {
      if (lane == 0) atomicAdd(&g_dot_stats[1], (unsigned long long)f);
      if (lane < f) {
        uint32_t D[N];
#pragma unroll
        for (int i = 0; i < N; ++i) D[i] = W.ds[j * N + i];
        add_n<N>(ch.R, ch.R, D);
      }
      ch.Shi = (int32_t)((long long)ch.Shi + __shfl_sync(FULL, hi, f - 1));
      ch.err = (int32_t)min((long long)ch.err + __shfl_sync(FULL, ci, f - 1), 1ll << 28);
    }
    // next window: base + f + 1 (after the walk of base + f) or base + 32
    const int sh = walk ? f + 1 : 32;
    {
      const int src = min(lane + sh, 31);
      const int v2 = __shfl_sync(FULL, wv, src);
      const int32_t e2 = __shfl_sync(FULL, weg, src);
      const uint32_t s2 = __shfl_sync(FULL, wsg, src);
      const long long m1 = __shfl_sync(FULL, wmn, src), m2 = __shfl_sync(FULL, wmx, src);
      const long long h2 = __shfl_sync(FULL, wht, src);
      if (lane + sh < 32) { wv = v2; weg = e2; wsg = s2; wmn = m1; wmx = m2; wht = h2; }
      else load_rec(base + lane + sh);              // issued before the walk
    }
    if (walk) sequential(base + f, t0);
    base += sh;
  }
  MP<L> r;
  ch.exact(r);
  if (lane == 0) store_y<L>(out, 0, r);
}

template <int L>
__global__ void __launch_bounds__(128) vec_axpy(int64_t n, VecIn alpha, int negate, VecIn x, VecIn y,
                                                YView z, const int* stop) {
  if (stop && *stop) return;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  MP<L> al, xv, s, t;
  load_mp<L>(alpha, 0, al);
  load_mp<L>(x, k, xv);
  load_mp<L>(y, k, s);
  mp_mul<L>(al.m, al.e, al.s ^ (uint32_t)negate, xv.m, xv.e, xv.s, t);
  mp_add<L>(s, t);
  store_y<L>(z, k, s);
}

// round the positive integer N (NW limbs, value N * 2^f) to p = 32L bits, RNE
template <int L, int NW>
__device__ void round_int(uint32_t (&N)[NW], int32_t f, MP<L>& o) {
  const uint32_t lz = clz_limbs<NW>(N);
  const int32_t b = 32 * NW - (int32_t)lz;           // bit length (N > 0)
  uint32_t stk = 0u;
  if (b > 32 * L) {
    shr_bits_sticky<NW>(N, (uint32_t)(b - 32 * L - 1), stk);   // keep p+1 bits: round bit at 0
    const uint32_t rb = N[0] & 1u;
    shr_bits_sticky<NW>(N, 1u, stk);
#pragma unroll
    for (int i = 0; i < L; ++i) o.m[i] = N[i];
    const uint32_t cy = rne_increment<L>(o.m, rb, stk);
    if (cy) o.m[L - 1] = 0x80000000u;
    o.e = f + b + (int32_t)cy;
  } else {
    shl_bits<NW>(N, (uint32_t)(32 * L - b));
#pragma unroll
    for (int i = 0; i < L; ++i) o.m[i] = N[i];
    o.e = f + b;
  }
}

template <int N>
__device__ __forceinline__ void shl1(uint32_t (&v)[N]) {
#pragma unroll
  for (int i = N - 1; i > 0; --i) v[i] = __funnelshift_l(v[i - 1], v[i], 1);
  v[0] <<= 1;
}
template <int N>
__device__ __forceinline__ void shr1(uint32_t (&v)[N]) {
#pragma unroll
  for (int i = 0; i < N - 1; ++i) v[i] = __funnelshift_r(v[i], v[i + 1], 1);
  v[N - 1] >>= 1;
}

// RN_p(a / b), b != 0 (a zero -> +0): quotient floor(Ma 2^K / Mb), K = p+3,
// by restoring binary long division, a sticky bit, one rounding
template <int L>
__device__ void mp_div(const MP<L>& a, const MP<L>& b, MP<L>& q) {
  if (a.is_zero() || b.is_zero()) { q.set_zero(); return; }
  constexpr int K = 32 * L + 3;
  uint32_t R[L + 1], D[L + 1], Q[L + 1];
#pragma unroll
  for (int i = 0; i < L; ++i) { R[i] = a.m[i]; D[i] = b.m[i]; Q[i] = 0u; }
  R[L] = 0u; D[L] = 0u; Q[L] = 0u;
  for (int i = 0; i <= K; ++i) {
    shl1<L + 1>(Q);
    if (!lt_n<L + 1>(R, D)) {
      sub_n<L + 1>(R, R, D, 0u);
      Q[0] |= 1u;
    }
    shl1<L + 1>(R);
  }
  uint32_t nz = 0u;
#pragma unroll
  for (int i = 0; i <= L; ++i) nz |= R[i];
  shl1<L + 1>(Q);                                      // N = 2Q + sticky
  Q[0] |= nz ? 1u : 0u;
  round_int<L, L + 1>(Q, a.e - b.e - K - 1, q);
  q.s = a.s ^ b.s;
}

// RN_p(sqrt(a)), a >= 0: floor(sqrt(M 2^(2K))) by the digit-by-digit method,
// K = p/2 + 3, a sticky bit, one rounding
template <int L>
__device__ void mp_sqrt(const MP<L>& a, MP<L>& r) {
  if (a.is_zero()) { r.set_zero(); return; }
  constexpr int NX = 2 * L + 1;
  constexpr int K = 16 * L + 3;
  int32_t e = a.e - 32 * L;
  uint32_t X[NX], Rt[NX], B[NX], T[NX];
#pragma unroll
  for (int i = 0; i < NX; ++i) { X[i] = i < L ? a.m[i] : 0u; Rt[i] = 0u; }
  if (e & 1) { shl1<NX>(X); e -= 1; }
  shl_bits<NX>(X, 2u * K);
  const uint32_t lz = clz_limbs<NX>(X);
  int pos = (32 * NX - 1 - (int)lz) & ~1;              // highest power of 4 <= X
  for (; pos >= 0; pos -= 2) {
#pragma unroll
    for (int i = 0; i < NX; ++i) B[i] = (i == (pos >> 5)) ? (1u << (pos & 31)) : 0u;
    add_n<NX>(T, Rt, B);                                 // T = res + bit
    shr1<NX>(Rt);
    if (!lt_n<NX>(X, T)) {
      sub_n<NX>(X, X, T, 0u);
      add_n<NX>(Rt, Rt, B);
    }
  }
  uint32_t nz = 0u;
#pragma unroll
  for (int i = 0; i < NX; ++i) nz |= X[i];
  uint32_t N2[L + 1];
#pragma unroll
  for (int i = 0; i <= L; ++i) N2[i] = Rt[i];
  shl1<L + 1>(N2);
  N2[0] |= nz ? 1u : 0u;
  round_int<L, L + 1>(N2, e / 2 - K - 1, r);
  r.s = 0u;
}

// exact comparison: -1, 0, 1
template <int L>
__device__ int mp_cmp(const MP<L>& a, const MP<L>& b) {
  const int ga = a.is_zero() ? 0 : (a.s ? -1 : 1);
  const int gb = b.is_zero() ? 0 : (b.s ? -1 : 1);
  if (ga != gb) return ga < gb ? -1 : 1;
  if (ga == 0) return 0;
  int c = (a.e > b.e) - (a.e < b.e);
  if (c == 0) c = lt_n<L>(b.m, a.m) ? 1 : (lt_n<L>(a.m, b.m) ? -1 : 0);
  return ga > 0 ? c : -c;
}

// BiCG scalars (device, ABI format [NSC] elements) and flags
enum { S_RHO = KS_RHO, S_RHOP = KS_RHOP, S_SIGMA = KS_SIGMA, S_ALPHA = KS_ALPHA, S_BETA = KS_BETA,
       S_RR = KS_RR, S_NRM = KS_NRM, S_THR = KS_THR, S_C1 = KS_C1, S_C2 = KS_C2, S_ONE = KS_ONE,
       S_T20 = KS_T20, S_T50 = KS_T50, S_ALPHAP = KS_ALPHAP, S_ZETA = KS_ZETA, S_ETA = KS_ETA,
       S_MU1 = KS_MU1, S_MU2 = KS_MU2, S_MU3 = KS_MU3, S_MU4 = KS_MU4, S_MU5 = KS_MU5,
       S_TAU = KS_TAU };
enum { F_STOP = KF_STOP, F_BREAK = KF_BREAK, F_CONV = KF_CONV, F_BRK2 = KF_BRK2 };

template <int L>
__device__ __forceinline__ void sc_mul(const MP<L>& a, const MP<L>& b, MP<L>& o) {
  mp_mul<L>(a.m, a.e, a.s, b.m, b.e, b.s, o);
}
// o = RN(RN(a b) - RN(c d))
template <int L>
__device__ __forceinline__ void sc_det(const MP<L>& a, const MP<L>& b, const MP<L>& c,
                                       const MP<L>& d, MP<L>& o) {
  MP<L> t;
  sc_mul<L>(a, b, o);
  sc_mul<L>(c, d, t);
  t.s ^= 1u;
  mp_add<L>(o, t);
}

template <int L>
__device__ __forceinline__ void sc_load(const YView& S, int i, MP<L>& a) {
  VecIn v{S.limbs, S.exps, S.signs};
  load_mp<L>(v, i, a);
  if (a.is_zero()) { a.e = 0; a.s = 0u; }
}

// op: 0 init (c1 = 1/10^20, c2 = 1/10^50, nrm0 = sqrt(rr), thr = c1 nrm0 + c2)
//     1 rho check (rho == 0 -> breakdown)    2 beta = rho / rho_prev
//     3 alpha = rho / sigma (sigma == 0 -> breakdown)
//     4 nrm = sqrt(rr), converged iff nrm <= thr; rho_prev = rho
//   GPBiCG (readings c32-c35 of DESIGN.md):
//     5 zeta = mu5 == 0 ? 0 : mu2 / mu5, eta = 0              (first iteration)
//     6 beta = RN(RN(rho / rho_prev) * RN(alpha_prev / zeta))
//     7 tau = RN(RN(mu5 mu1) - RN(mu4 mu4)) (0 -> breakdown),
//       zeta = RN(RN(RN(mu1 mu2) - RN(mu3 mu4)) / tau), eta = RN(RN(RN(mu5 mu3) - RN(mu4 mu2)) / tau)
//     8 nrm = sqrt(rr), converged iff nrm <= thr, else zeta = 0 -> breakdown;
//       rho_prev = rho, alpha_prev = alpha
template <int L>
__global__ void bicg_scalar(YView S, int* fl, int op) {
  if (fl[F_STOP]) return;
  MP<L> a, b, c;
  switch (op) {
    case 0: {
      sc_load<L>(S, S_ONE, a);
      sc_load<L>(S, S_T20, b);
      mp_div<L>(a, b, c);
      store_y<L>(S, S_C1, c);
      sc_load<L>(S, S_T50, b);
      mp_div<L>(a, b, c);
      store_y<L>(S, S_C2, c);
        MP<L> c1;
      sc_load<L>(S, S_C1, c1);
      sc_load<L>(S, S_RR, a);
      mp_sqrt<L>(a, b);                         // nrm0
      MP<L> t;
      mp_mul<L>(c1.m, c1.e, c1.s, b.m, b.e, b.s, t);
      sc_load<L>(S, S_C2, c);
      mp_add<L>(t, c);
      store_y<L>(S, S_THR, t);
      break;
    }
    case 1:
      sc_load<L>(S, S_RHO, a);
      if (a.is_zero()) { fl[F_BREAK] = 1; fl[F_STOP] = 1; }
      break;
    case 2:
      sc_load<L>(S, S_RHO, a);
      sc_load<L>(S, S_RHOP, b);
      mp_div<L>(a, b, c);
      store_y<L>(S, S_BETA, c);
      break;
    case 3:
      sc_load<L>(S, S_RHO, a);
      sc_load<L>(S, S_SIGMA, b);
      if (b.is_zero()) { fl[F_BREAK] = 1; fl[F_STOP] = 1; break; }
      mp_div<L>(a, b, c);
      store_y<L>(S, S_ALPHA, c);
      break;
    case 4: {
      sc_load<L>(S, S_RR, a);
      mp_sqrt<L>(a, b);
      store_y<L>(S, S_NRM, b);
      sc_load<L>(S, S_THR, c);
      if (mp_cmp<L>(b, c) <= 0) { fl[F_CONV] = 1; fl[F_STOP] = 1; }
      sc_load<L>(S, S_RHO, a);
      store_y<L>(S, S_RHOP, a);
      break;
    }
    case 5: {
      sc_load<L>(S, S_MU2, a);
      sc_load<L>(S, S_MU5, b);
      if (b.is_zero()) c.set_zero(); else mp_div<L>(a, b, c);
      store_y<L>(S, S_ZETA, c);
      c.set_zero();
      store_y<L>(S, S_ETA, c);
      break;
    }
    case 6: {
      MP<L> d, e;
      sc_load<L>(S, S_RHO, a);
      sc_load<L>(S, S_RHOP, b);
      mp_div<L>(a, b, c);
      sc_load<L>(S, S_ALPHAP, a);
      sc_load<L>(S, S_ZETA, b);
      mp_div<L>(a, b, d);
      sc_mul<L>(c, d, e);
      store_y<L>(S, S_BETA, e);
      break;
    }
    case 7: {
      MP<L> m1, m2, m3, m4, m5, tau, num;
      sc_load<L>(S, S_MU1, m1);
      sc_load<L>(S, S_MU2, m2);
      sc_load<L>(S, S_MU3, m3);
      sc_load<L>(S, S_MU4, m4);
      sc_load<L>(S, S_MU5, m5);
      sc_det<L>(m5, m1, m4, m4, tau);
      store_y<L>(S, S_TAU, tau);
      if (tau.is_zero()) { fl[F_BREAK] = 1; fl[F_STOP] = 1; break; }
      sc_det<L>(m1, m2, m3, m4, num);
      mp_div<L>(num, tau, c);
      store_y<L>(S, S_ZETA, c);
      sc_det<L>(m5, m3, m4, m2, num);
      mp_div<L>(num, tau, c);
      store_y<L>(S, S_ETA, c);
      break;
    }
    case 8: {
      sc_load<L>(S, S_RR, a);
      mp_sqrt<L>(a, b);
      store_y<L>(S, S_NRM, b);
      sc_load<L>(S, S_THR, c);
      if (mp_cmp<L>(b, c) <= 0) {
        fl[F_CONV] = 1; fl[F_STOP] = 1;
      } else {
        sc_load<L>(S, S_ZETA, a);
        if (a.is_zero()) { fl[F_BRK2] = 1; fl[F_STOP] = 1; }
      }
      sc_load<L>(S, S_RHO, a);
      store_y<L>(S, S_RHOP, a);
      sc_load<L>(S, S_ALPHA, a);
      store_y<L>(S, S_ALPHAP, a);
      break;
    }
  }
}

// ---------------------------------------------------------------- launchers
template <int L>
struct KrylovOps {
  static int dot(int64_t n, VecIn u, VecIn v, YView out, const int* stop, cudaStream_t st,
                 void* work) {
    const int64_t nseg = (n + DSEG - 1) / DSEG;
    if (!work || nseg <= 1) {                      // short vectors: one warp
      vec_dot<L><<<1, 32, 0, st>>>(n, u, v, out, stop);
      launch_counter_add(1);
      return (int)cudaGetLastError();
    }
    DotWork W = carve(work, nseg);
    const unsigned nb = (unsigned)((nseg * 32 + 127) / 128);
    dot_products<L><<<nb, 128, 0, st>>>(n, u, v, W, nseg, stop);
    dot_prefix<<<1, 1024, 0, st>>>(W.segsum, nseg, stop);
    dot_speculate<L><<<nb, 128, 0, st>>>(W, nseg, stop);
    dot_chain<L><<<1, 32, 0, st>>>(n, W, nseg, out, stop);
    launch_counter_add(4);
    return (int)cudaGetLastError();
  }
  static size_t bytes(int64_t n) {
    const int64_t nseg = (n + DSEG - 1) / DSEG;
    return carve_bytes(nseg);
  }
  static size_t carve_bytes(int64_t nseg) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t nblk = (size_t)nseg * DSEG_NB;
    return al(nblk * (L + 2) * 32 * 4) + al(nseg * 8) + 3 * al(nseg * 4) + 3 * al(nseg * 8) +
           al((size_t)nseg * (L + 2) * 4);
  }
  static DotWork carve(void* work, int64_t nseg) {
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    char* p = (char*)work;
    const size_t nblk = (size_t)nseg * DSEG_NB;
    DotWork W;
    W.prod = (uint32_t*)p; p += al(nblk * (L + 2) * 32 * 4);
    W.segsum = (double*)p; p += al(nseg * 8);
    W.valid = (int32_t*)p; p += al(nseg * 4);
    W.eg = (int32_t*)p; p += al(nseg * 4);
    W.sg = (uint32_t*)p; p += al(nseg * 4);
    W.minv = (long long*)p; p += al(nseg * 8);
    W.maxv = (long long*)p; p += al(nseg * 8);
    W.htot = (long long*)p; p += al(nseg * 8);
    W.ds = (uint32_t*)p;
    return W;
  }
  static int axpy(int64_t n, VecIn al, int neg, VecIn x, VecIn y, YView z, const int* stop,
                  cudaStream_t st) {
    if (n <= 0) return 0;
    vec_axpy<L><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, al, neg, x, y, z, stop);
    launch_counter_add(1);
    return (int)cudaGetLastError();
  }
  static int scalar(YView S, int* fl, int op, cudaStream_t st) {
    bicg_scalar<L><<<1, 1, 0, st>>>(S, fl, op);
    launch_counter_add(1);
    return (int)cudaGetLastError();
  }
};

int krylov_dot(int L, int64_t n, const VecIn& u, const VecIn& v, const YView& out, const int* stop,
               void* stream, void* work) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 1: return KrylovOps<1>::dot(n, u, v, out, stop, st, work);
    case 2: return KrylovOps<2>::dot(n, u, v, out, stop, st, work);
    case 4: return KrylovOps<4>::dot(n, u, v, out, stop, st, work);
    case 8: return KrylovOps<8>::dot(n, u, v, out, stop, st, work);
    case 16: return KrylovOps<16>::dot(n, u, v, out, stop, st, work);
    case 32: return KrylovOps<32>::dot(n, u, v, out, stop, st, work);
    default: return L > 32 ? krylov_wide_dot(L, n, u, v, out, stop, stream, work)
                           : (int)cudaErrorInvalidValue;
  }
}

int krylov_dot_stats(unsigned long long out[2]) {
  cudaError_t e = cudaMemcpyFromSymbol(out, g_dot_stats, sizeof(unsigned long long) * 2);
  if (e == cudaSuccess) {
    unsigned long long z[2] = {0ull, 0ull};
    e = cudaMemcpyToSymbol(g_dot_stats, z, sizeof z);
  }
  return (int)e;
}

size_t krylov_dot_work_bytes(int L, int64_t n) {
  switch (L) {
    case 1: return KrylovOps<1>::bytes(n);
    case 2: return KrylovOps<2>::bytes(n);
    case 4: return KrylovOps<4>::bytes(n);
    case 8: return KrylovOps<8>::bytes(n);
    case 16: return KrylovOps<16>::bytes(n);
    case 32: return KrylovOps<32>::bytes(n);
    default: return L > 32 ? krylov_wide_dot_work_bytes(L, n) : 0;
  }
}

int krylov_axpy(int L, int64_t n, const VecIn& al, int neg, const VecIn& x, const VecIn& y,
                const YView& z, const int* stop, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 1: return KrylovOps<1>::axpy(n, al, neg, x, y, z, stop, st);
    case 2: return KrylovOps<2>::axpy(n, al, neg, x, y, z, stop, st);
    case 4: return KrylovOps<4>::axpy(n, al, neg, x, y, z, stop, st);
    case 8: return KrylovOps<8>::axpy(n, al, neg, x, y, z, stop, st);
    case 16: return KrylovOps<16>::axpy(n, al, neg, x, y, z, stop, st);
    case 32: return KrylovOps<32>::axpy(n, al, neg, x, y, z, stop, st);
    default: return L > 32 ? krylov_wide_axpy(L, n, al, neg, x, y, z, stop, stream)
                           : (int)cudaErrorInvalidValue;
  }
}

int krylov_scalar(int L, const YView& S, int* fl, int op, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 4: return KrylovOps<4>::scalar(S, fl, op, st);
    case 8: return KrylovOps<8>::scalar(S, fl, op, st);
    case 16: return KrylovOps<16>::scalar(S, fl, op, st);
    case 32: return KrylovOps<32>::scalar(S, fl, op, st);
    default: return L > 32 ? krylov_wide_scalar(L, S, fl, op, stream) : (int)cudaErrorInvalidValue;
  }
}

}  // namespace mpsp
