// krylov.cu - multiple-precision BiCG on the GPU:
// PAPER.md:249-297 (Fig. 4, BiCG) with K = I, the two SpMVs (A p, A^T p~)
// by this library's kernels, and PAPER.md:375-380 (convergence test
// ||r|| <= 1e-20 ||r_0|| + 1e-50).  Every operation is one p-bit RN
// operation in the order the figure writes it (readings c26-c31):
//   dot      (u, v) = ordered chain s = RN(s + RN(u_k v_k)), k ascending
//            (one warp, the exact speculative block sum of wchain.cuh)
//   axpy     z_k = RN(y_k + RN(+-alpha x_k))            (thread per element)
//   scalars  RN(a / b), RN(sqrt(a)), exact compare      (one thread:
//            integer long division / square root + one rounding)
// The host loop keeps every value on the device; one 3-int flag read per
// iteration decides breakdown / convergence (kernels after a stop flag do
// nothing, so x keeps the last complete iterate, as in the oracle).
#include <cuda_runtime.h>

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
       S_T20 = KS_T20, S_T50 = KS_T50 };
enum { F_STOP = KF_STOP, F_BREAK = KF_BREAK, F_CONV = KF_CONV };

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
  }
}

// ---------------------------------------------------------------- launchers
template <int L>
struct KrylovOps {
  static int dot(int64_t n, VecIn u, VecIn v, YView out, const int* stop, cudaStream_t st) {
    vec_dot<L><<<1, 32, 0, st>>>(n, u, v, out, stop);
    launch_counter_add(1);
    return (int)cudaGetLastError();
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
               void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 1: return KrylovOps<1>::dot(n, u, v, out, stop, st);
    case 2: return KrylovOps<2>::dot(n, u, v, out, stop, st);
    case 4: return KrylovOps<4>::dot(n, u, v, out, stop, st);
    case 8: return KrylovOps<8>::dot(n, u, v, out, stop, st);
    case 16: return KrylovOps<16>::dot(n, u, v, out, stop, st);
    case 32: return KrylovOps<32>::dot(n, u, v, out, stop, st);
    default: return (int)cudaErrorInvalidValue;
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
    default: return (int)cudaErrorInvalidValue;
  }
}

int krylov_scalar(int L, const YView& S, int* fl, int op, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 4: return KrylovOps<4>::scalar(S, fl, op, st);
    case 8: return KrylovOps<8>::scalar(S, fl, op, st);
    case 16: return KrylovOps<16>::scalar(S, fl, op, st);
    case 32: return KrylovOps<32>::scalar(S, fl, op, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace mpsp
