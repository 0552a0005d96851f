// wchain.cuh - the exact speculative block sum of an ordered rounded chain
// s = RN(s + t_k) held by one warp (used by the warp-row SpMV kernels and by
// the BiCG dot product).  See spmv_wrow.cu for the argument and DESIGN.md.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "mp_device.cuh"

namespace mpsp {

// Tuning counters (-DMPSP_WSTATS builds only; per translation unit):
// [0] passes, [1] fast commits, [2] failing steps, [3] up, [4] down,
// [5] dominant, [6] exact adder, [7] zero-accumulator absorptions
#ifdef MPSP_WSTATS
static __device__ unsigned long long g_wstats[8];
#define WSTAT(i) do { if ((threadIdx.x & 31) == 0) atomicAdd(&g_wstats[i], 1ull); } while (0)
#else
#define WSTAT(i) do { } while (0)
#endif

// High-part scale H = 2^(p-HB) grid units: S/H in [2^(HB-1), 2^HB).  HB = 26
// keeps the 32-lane scan of |h| <= 2^25 (plus Shi and the error count) in
// int32; one unit of H is >= one grid unit u for every p >= 32.
constexpr int HB = 26;

template <int L>
__device__ __forceinline__ int32_t hi_of_mant(const uint32_t (&m)[L]) {
  return (int32_t)(m[L - 1] >> (32 - HB));
}

// floor(Q / H) for an (L+2)-limb two's complement Q with |Q| <= 2^(p-1) + 1
template <int L>
__device__ __forceinline__ int32_t hi_of_q(const uint32_t (&Q)[L + 2]) {
  return (int32_t)__funnelshift_r(Q[L - 1], Q[L], 32 - HB);
}

// a - b saturated to the int32 range (exponent differences: |a|, |b| < 2^31)
__device__ __forceinline__ int32_t sub_sat(int32_t a, int32_t b) {
  int32_t d;
  asm("sub.sat.s32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

template <int N>
__device__ __forceinline__ void warp_sum_limbs(uint32_t (&S)[N]) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint32_t T[N];
#pragma unroll
    for (int i = 0; i < N; ++i) T[i] = __shfl_xor_sync(0xffffffffu, S[i], o);
    add_n<N>(S, S, T);
  }
}

// Grid alignment of one product against the accumulator tag (E, sg): Q =
// +-RN_int(|t|/u) in (L+2)-limb two's complement, its high part, and whether
// the step must take the exact path (|t| reaches the binade, or a grid tie).
template <int L>
__device__ __forceinline__ void align_q(const MP<L>& t, bool act, int32_t E, uint32_t sg,
                                        uint32_t (&Q)[L + 2], int32_t& h, bool& pre) {
  constexpr int N = L + 2;
  const int64_t d64 = (int64_t)E - (int64_t)t.e;
  const bool badd = act && d64 < 1;
  const bool use = act && !badd;
  const uint32_t dd = use ? (uint32_t)min(d64, (int64_t)(32 * L + 32)) : 0u;
  uint32_t Y[L + 1];
  Y[0] = 0u;
#pragma unroll
  for (int i = 0; i < L; ++i) Y[i + 1] = t.m[i];
  uint32_t stk = 0u;
  shr_bits_sticky<L + 1>(Y, dd, stk);
  const uint32_t rb = Y[0] >> 31;
  const bool sticky = (stk | (Y[0] << 1)) != 0u;
  const bool tie = use && rb && !sticky;
  const uint32_t inc = (rb && sticky) ? 1u : 0u;
  pre = badd || tie;
  const uint32_t neg = (use && t.s != sg) ? 1u : 0u;
  const uint32_t nm = 0u - neg;
#pragma unroll
  for (int i = 0; i < L; ++i) Q[i] = (use ? Y[i + 1] : 0u) ^ nm;
  Q[L] = nm;
  Q[L + 1] = nm;
  inc_n<N>(Q, use ? (neg ? 1u - inc : inc) : 0u);
  h = hi_of_q<L>(Q);
}

// The chain state of one row held by one warp, and the exact block sum.
template <int L>
struct WChain {
  static constexpr int N = L + 2;
  uint32_t R[N];          // this lane's share of S (two's complement)
  bool szero;             // accumulator is exactly zero (warp-uniform)
  int32_t E;              // accumulator exponent (warp-uniform)
  uint32_t sg;            // accumulator sign
  int32_t Shi, err;       // S/H in [Shi, Shi + err)

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < N; ++i) R[i] = 0u;
    szero = true;
    E = 0;
    sg = 0u;
    Shi = 0;
    err = 0;
  }

  __device__ __forceinline__ void reset_to(const MP<L>& s, int lane) {
    szero = s.is_zero();
#pragma unroll
    for (int i = 0; i < N; ++i) R[i] = (lane == 0 && i < L) ? s.m[i] : 0u;
    E = s.e;
    sg = s.s;
    Shi = szero ? 0 : hi_of_mant<L>(s.m);
    err = 1;
  }

  // exact S (all lanes)
  __device__ __forceinline__ void exact(MP<L>& s) const {
    uint32_t S[N];
#pragma unroll
    for (int i = 0; i < N; ++i) S[i] = R[i];
    warp_sum_limbs<N>(S);
#pragma unroll
    for (int i = 0; i < L; ++i) s.m[i] = szero ? 0u : S[i];
    s.e = E;
    s.s = sg;
  }

  // s := the chain over this warp's 32 products t (lane k holds step k).
  // Clobbers t: the steps a pass has disposed of (lanes <= f) are zeroed
  // before the next pass, so "act" is just t != 0 and the aligned product
  // needs no lane mask (padding lanes hold zero limbs already).
  __device__ __forceinline__ void consume(MP<L>& t, int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int32_t LO = 1 << (HB - 1), HI = 1 << HB;
    const unsigned below = (1u << lane) - 1u;
    int start = 0;
    auto retire = [&](int f) {          // steps 0..f are done
      if (lane <= f) {
#pragma unroll
        for (int i = 0; i < L; ++i) t.m[i] = 0u;
      }
    };
    while (start < 32) {
      const bool tz = t.is_zero();
      if (szero) {
        // s = +0: the first nonzero product is absorbed exactly
        const unsigned nzm = __ballot_sync(FULL, !tz && lane >= start);
        if (nzm == 0u) break;
        const int f = __ffs(nzm) - 1;
        MP<L> tf;
#pragma unroll
        for (int i = 0; i < L; ++i) tf.m[i] = __shfl_sync(FULL, t.m[i], f);
        tf.e = __shfl_sync(FULL, t.e, f);
        tf.s = __shfl_sync(FULL, t.s, f);
        reset_to(tf, lane);
        WSTAT(7);
        retire(f);
        start = f + 1;
        continue;
      }
      const bool act = !tz;
      WSTAT(0);
      const int32_t d32 = sub_sat(E, t.e);            // E - t.e, saturated to int32
      const bool badd = act && d32 < 1;              // |t| >= 2^(E-1): leaves the binade
      const bool use = act && !badd;
      const uint32_t dd = use ? (uint32_t)min(d32, 32 * L + 32) : 0u;
      // Y = |t| / u  as integer limbs Y[1..L] and guard limb Y[0]
      uint32_t Y[L + 1];
      Y[0] = 0u;
#pragma unroll
      for (int i = 0; i < L; ++i) Y[i + 1] = t.m[i];
      uint32_t stk = 0u;
      shr_bits_sticky<L + 1, true>(Y, dd, stk);      // the whole warp is here
      const uint32_t rb = Y[0] >> 31;
      const bool sticky = (stk | (Y[0] << 1)) != 0u;
      const bool tie = use && rb && !sticky;
      uint32_t inc = (rb && sticky) ? 1u : 0u;
      const uint32_t lsbY = Y[1] & 1u;
      const unsigned tieM = __ballot_sync(FULL, tie);
      if (tieM) {                                     // warp-uniform, rare
        // parity of S_{k-1}: that of S (XOR of the lanes' R low bits), reset
        // to 0 by the last tie before k, XORed with the non-tie Q_j low bits
        const uint32_t par = (uint32_t)__popc(__ballot_sync(FULL, R[0] & 1u)) & 1u;
        const unsigned bM = __ballot_sync(FULL, use && !tie && ((lsbY ^ inc) & 1u));
        if (tie) {
          const unsigned tb = tieM & below;
          const int lt = tb ? 31 - __clz(tb) : -1;
          const unsigned seg = below & (lt >= 0 ? ~((2u << lt) - 1u) : FULL);
          const uint32_t pS = ((lt >= 0 ? 0u : par) ^ (uint32_t)__popc(bM & seg)) & 1u;
          inc = pS ^ lsbY;                            // make S_k even
        }
      }
      // Q = +-(Y + inc) in N-limb two's complement = P + cin with P = Y ^ nm
      // (one's complement for the minus sign) and cin = inc or 1 - inc: the
      // carry-in is added by the commit's own carry chain.  The high part h
      // is taken from P, so Q/H lies in [h, h + 2): the bounds below count
      // two units of error per step.
      const uint32_t neg = (use && t.s != sg) ? 1u : 0u;
      // (Y of a lane that leaves the binade - badd - is not masked: such a
      // lane fails, so neither its Q nor its h reach a committed step or a
      // bound of one, and step_f reads hf only for a lane that is "use")
      const uint32_t nm = 0u - neg;
      const uint32_t cin = use ? (neg ? 1u - inc : inc) : 0u;
      uint32_t Q[N];
#pragma unroll
      for (int i = 0; i < L; ++i) Q[i] = Y[i + 1] ^ nm;
      Q[L] = nm;
      Q[L + 1] = nm;
      const int32_t h = hi_of_q<L>(Q);
      int32_t Pi = h;                                 // inclusive scan of h
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(FULL, Pi, o);
        if (lane >= o) Pi += v;
      }
      const int32_t LB = Shi + (Pi - h);              // S_{k-1}/H >= LB
      const int32_t ek = err + 2 * lane;              // S_{k-1}/H < LB + ek
      const bool ok = !act || (!badd && LB + h - 1 >= LO && LB + ek + h + 2 <= HI);
      const unsigned failM = __ballot_sync(FULL, !ok);
      if (failM == 0u) {
        add_n_cin<N>(R, R, Q, cin);
        Shi += __shfl_sync(FULL, Pi, 31);
        err = min(err + 64, 1 << 28);                 // saturates: checks then fail
        WSTAT(1);
        break;
      }
      // ---- the first failing step f
      const int f = __ffs(failM) - 1;
      WSTAT(2);
      if (lane < f) add_n_cin<N>(R, R, Q, cin);      // steps before f are valid
      step_f(t, f, __shfl_sync(FULL, LB, f), __shfl_sync(FULL, h, f), err + 2 * f, lane);
      retire(f);
      start = f + 1;
    }
  }

  // The first failing step f of a block: lane f holds its product t; LBf, hf,
  // ekf are its high-part bounds (S_{f-1}/H in [LBf, LBf + ekf), Q_f/H in
  // [hf, hf + 2)).  One-binade transitions (tests/test_kernel_algorithms.py
  // models them): if step f's exact sum V = S + tau provably crosses 2^p
  // (equal signs) or provably lands in [2^(p-2), 2^(p-1)) (opposite signs),
  // it is rounded directly on the new grid 2u / u/2 from the low bits of
  // W = S (+ floor tau) - read off the lanes' R by ballots - and tau's
  // fraction bits; R is halved / doubled lane by lane.  A dominant product
  // (|t| >= 2^(E-1)) whose sum's binade E + k is certified is rounded on the
  // grid 2^k u from one redux over the lanes' R.  Everything else takes the
  // exact adder.  All lanes call it (warp-uniform control flow).
  __device__ __forceinline__ void step_f(const MP<L>& t, int f, int32_t LBf, int32_t hf,
                                         int32_t ekf, int lane) {
    constexpr unsigned FULL = 0xffffffffu;
    constexpr int32_t LO = 1 << (HB - 1), HI = 1 << HB;
    const bool act = !t.is_zero();
    const int64_t d64 = (int64_t)E - (int64_t)t.e;
    const bool badd = act && d64 < 1;                // |t| >= 2^(E-1)
    const bool use = act && !badd;
    const uint32_t dd0 = use ? (uint32_t)min(d64, (int64_t)(32 * L + 32)) : 0u;
    uint32_t Y[L + 1];
    Y[0] = 0u;
#pragma unroll
    for (int i = 0; i < L; ++i) Y[i + 1] = t.m[i];
    uint32_t stk = 0u;
    shr_bits_sticky<L + 1, true>(Y, dd0, stk);
    {
      const uint32_t fy = Y[0];                     // tau's 32 fraction bits
      const bool fnz = (fy != 0u) || (stk != 0u);   // fraction != 0
      const bool up_f = use && t.s == sg && LBf + hf - 1 >= HI;
      const bool dn_f = use && t.s != sg && LBf + ekf + hf + 3 <= LO && LBf + hf - 1 >= LO / 2;
      // dominant product (|t| >= 2^(E-1), t.e - E = dd in [0, 27]): the binade
      // E + k of V = S u + t certified from the high-part bounds and t's top
      // 32 bits (units 2^(E-HB)); t/u = M_t 2^dd is an integer
      const int dd = (int)min(max(-d64, (int64_t)0), (int64_t)27);
      const uint32_t mt = t.m[L - 1];
      const int64_t tl = dd >= 6 ? ((int64_t)mt << (dd - 6)) : (int64_t)(mt >> (6 - dd));
      const int64_t th = tl + (dd >= 6 ? ((int64_t)1 << (dd - 6)) : (int64_t)1);
      const bool same = t.s == sg;
      const int64_t vlo = same ? (int64_t)LBf + tl : tl - (int64_t)LBf - ekf;
      const int64_t vhi = same ? (int64_t)LBf + ekf + th : th - (int64_t)LBf + 1;
      const int kd = vlo > 0 ? (64 - __clzll(vlo)) - HB : 0;
      const bool dom_f = badd && -d64 <= 27 && kd >= 1 && kd <= 26 &&
                         vhi <= ((int64_t)1 << (HB + kd)) - 1;
#ifdef MPSP_TRANS_MASK
      const int mode = __shfl_sync(FULL, up_f ? 1 : (dn_f ? 2 : (dom_f ? 4 : 0)), f) & MPSP_TRANS_MASK;
#else
      const int mode = __shfl_sync(FULL, up_f ? 1 : (dn_f ? 2 : (dom_f ? 4 : 0)), f);
#endif
      if (mode == 4) {
        WSTAT(5);
        const int k = __shfl_sync(FULL, kd, f);
        const int64_t vlof = __shfl_sync(FULL, vlo, f), vhif = __shfl_sync(FULL, vhi, f);
        const uint32_t sgf = __shfl_sync(FULL, t.s, f);
        if (sgf != sg) {                            // S := -S: W = |t|/u - S > 0
#pragma unroll
          for (int i = 0; i < N; ++i) R[i] = ~R[i];
          inc_n<N>(R, 1u);
        }
        if (lane == f) {                            // W = R-sum + M_t << dd
          uint32_t Yv[N];
          Yv[0] = t.m[0] << dd;
#pragma unroll
          for (int i = 1; i < L; ++i) Yv[i] = __funnelshift_l(t.m[i - 1], t.m[i], dd);
          Yv[L] = dd ? (t.m[L - 1] >> (32 - dd)) : 0u;
          Yv[L + 1] = 0u;
          add_n<N>(R, R, Yv);
        }
        // RN_int(W / 2^k): W mod 2^k from the lanes' low k bits (k <= 26:
        // their sum fits 31 bits), floor(W / 2^k) = sum of the lanes'
        // arithmetic shifts + the carry of that sum
        const uint32_t lows = __reduce_add_sync(FULL, R[0] & ((1u << k) - 1u));
        const uint32_t c = lows >> k;
        const uint32_t rb = (lows >> (k - 1)) & 1u;
        const uint32_t stk2 = (lows & ((1u << (k - 1)) - 1u)) != 0u ? 1u : 0u;
        const uint32_t par = ((uint32_t)__popc(__ballot_sync(FULL, (R[0] >> k) & 1u)) + c) & 1u;
        const uint32_t incr = rb & (stk2 | par);
#pragma unroll
        for (int i = 0; i < N - 1; ++i) R[i] = __funnelshift_r(R[i], R[i + 1], k);
        R[N - 1] = (uint32_t)((int32_t)R[N - 1] >> k);
        if (lane == 0) {
          uint32_t Cv[N];
          Cv[0] = c + incr;
#pragma unroll
          for (int i = 1; i < N; ++i) Cv[i] = 0u;
          add_n<N>(R, R, Cv);
        }
        sg = sgf;
        E += k;
        Shi = (int32_t)((vlof >> k) - 1);
        err = (int32_t)((vhif >> k) - (vlof >> k) + 3);
        return;
      }
      if (mode == 1) {                              // V in [2^p, 1.5 2^p): grid 2u
        WSTAT(3);
        if (lane == f) {
          uint32_t Yv[N];
#pragma unroll
          for (int i = 0; i < L; ++i) Yv[i] = Y[i + 1];
          Yv[L] = 0u;
          Yv[L + 1] = 0u;
          add_n<N>(R, R, Yv);                       // W = S + floor(tau)
        }
        const uint32_t c0 = (uint32_t)__popc(__ballot_sync(FULL, R[0] & 1u));
        const uint32_t c1 = (uint32_t)__popc(__ballot_sync(FULL, (R[0] >> 1) & 1u));
        const uint32_t w0 = c0 & 1u, w1 = ((c0 >> 1) + c1) & 1u;
        const uint32_t frac = __shfl_sync(FULL, fnz ? 1u : 0u, f);
        const uint32_t incr = w0 & (frac | w1);     // RNE of W/2 + (w0 + frac)/2
#pragma unroll
        for (int i = 0; i < N - 1; ++i) R[i] = __funnelshift_r(R[i], R[i + 1], 1);
        R[N - 1] = (uint32_t)((int32_t)R[N - 1] >> 1);
        if (lane == 0) {
          uint32_t Cv[N];
          Cv[0] = (c0 >> 1) + incr;
#pragma unroll
          for (int i = 1; i < N; ++i) Cv[i] = 0u;
          add_n<N>(R, R, Cv);                       // sum of halves + lost carries
        }
        E += 1;
        Shi = (LBf + hf - 1) >> 1;
        err = ((ekf + 4) >> 1) + 2;
        return;
      }
      if (mode == 2) {                              // V in [2^(p-2), 2^(p-1)): grid u/2
        WSTAT(4);
#pragma unroll
        for (int i = N - 1; i > 0; --i) R[i] = __funnelshift_l(R[i - 1], R[i], 1);
        R[0] <<= 1;
        const uint32_t b1 = fy >> 31, b2 = (fy >> 30) & 1u;
        const bool low = ((fy << 1) != 0u) || (stk != 0u);
        const bool tie2 = b2 && ((fy << 2) == 0u) && (stk == 0u);
        if (lane == f) {                            // R -= 2 floor(tau) + b1 (+1 if low)
          uint32_t Yv[N];                           // (floor(tau) << 1) | b1
#pragma unroll
          for (int i = 0; i < N; ++i) {
            const uint32_t lo_ = (i >= 1 && i - 1 < L) ? Y[i] : 0u;      // limb i-1
            const uint32_t cur = (i < L) ? Y[i + 1] : 0u;                // limb i
            Yv[i] = __funnelshift_l(lo_, cur, 1);
          }
          Yv[0] |= b1;
          sub_n<N>(R, R, Yv, low ? 1u : 0u);
        }
        const uint32_t low_f = __shfl_sync(FULL, low ? 1u : 0u, f);
        const uint32_t b1f = __shfl_sync(FULL, b1, f), b2f = __shfl_sync(FULL, b2, f);
        const uint32_t tie2f = __shfl_sync(FULL, tie2 ? 1u : 0u, f);
        if (lane == 0 && low_f) {
          const uint32_t upb = (b2f == 0u) | (tie2f & (b1f ^ 1u));
          inc_n<N>(R, upb);
        }
        E -= 1;
        Shi = 2 * (LBf + hf - 1) - 2;
        err = 2 * (ekf + 3) + 4;
        return;
      }
    }
    WSTAT(6);
    MP<L> s, tf;
    exact(s);
#pragma unroll
    for (int i = 0; i < L; ++i) tf.m[i] = __shfl_sync(FULL, t.m[i], f);
    tf.e = __shfl_sync(FULL, t.e, f);
    tf.s = __shfl_sync(FULL, t.s, f);
    mp_add<L, true>(s, tf);
    reset_to(s, lane);
  }
};

}  // namespace mpsp
