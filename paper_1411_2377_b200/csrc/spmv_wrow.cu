// spmv_wrow.cu - one warp per long row: products in parallel across the
// lanes, and the ordered rounded add chain evaluated 32 steps at a time by an
// EXACT speculative block sum (hard part 2: the chain
// s = RN(s + t_k) of a 5000-long C4 row is a serial critical path).
//
// Why a block of steps can be summed in parallel.  Let s have exponent E, so
// s = S*u with u = 2^(E-p) and S an integer in [2^(p-1), 2^p).  If the exact
// value V = s + t_k lies in the same binade and its rounding stays below 2^E,
// RN_p(s + t_k) = (S + RN_int(t_k/u)) * u: the rounding grid is u, and s is on
// it.  So while the partial sums stay in one binade, the chain is the integer
// sum  S_k = S_{k-1} + Q_k  with Q_k = +-RN_int(|t_k|/u)  - associative, i.e.
// computable in any order.  RN_int's only dependence on the running sum is the
// tie case (|t_k|/u = m + 1/2 exactly: round to the EVEN S_k), which needs the
// parity of S_{k-1}; parities are prefix XORs of the Q_k's low bits and a tie
// resets the parity to 0, so every lane gets its own in O(1) from two ballots.
//
// Per block of 32 entries (one per lane): each lane forms t_k = RN(a_k x_col)
// (Comba, IMAD.WIDE), aligns it to the grid u, and rounds it (Q_k).  A warp
// scan of int32 high parts h_k = floor(Q_k/H) (H = 2^(p-26) grid units)
// gives conservative bounds on every partial sum; if all are provably inside
// [2^(p-1), 2^p - 1] the block commits: each lane adds Q_k to its private
// (L+2)-limb partial sum R_lane (S = sum over lanes of R, exact mod
// 2^(32(L+2)), reduced only when needed).  Otherwise, at the first failing
// step f, the steps before f commit; a step that provably moves the sum one
// binade up or down, or whose product dominates the sum, is rounded on the
// certified new grid from ballots / one redux over the lanes' R (WChain's
// transitions); any other failing step reduces S exactly (warp butterfly),
// runs the general adder mp_add (all lanes redundantly), and the block
// resumes at f+1 in the new binade.  Nothing is approximated: the bounds
// only decide fast vs exact (wchain.cuh; CPU model in
// tests/test_kernel_algorithms.py).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdlib>

#include "kernel_common.cuh"
#include "wchain.cuh"

namespace mpsp {

// Read at every mpsp_csr_create: rows longer than this go to spmv_wrow
// (tests lower it to route rows of any length through this kernel).
int long_row_threshold() {
  const char* v = std::getenv("MPSP_LONG_T");
  return v ? std::atoi(v) : 192;
}

// Rows at least this long (and above the warp-row threshold) go to the
// producer/consumer kernel spmv_pcrow (tests lower it to route rows there).
int pc_row_threshold() {
  const char* v = std::getenv("MPSP_PC_T");
  return v ? std::atoi(v) : INT_MAX;                 // opt-in (no faster yet)
}

template <int L>
struct WPrefetch { static constexpr bool on = (L <= 16); };

template <int L>
struct WEntry {
  uint32_t a[L], x[L];
  int32_t w, ex;
  uint32_t sx;
  bool valid;
};

// Entry jb + lane of the row; its column `col` was loaded one block earlier
// (the x gather never waits on the column load).
template <int L>
__device__ __forceinline__ void wload(const PartView& P, const XView& x, int64_t e0, int jb,
                                      int len, int lane, int col, WEntry<L>& E) {
  const int j = jb + lane;
  E.valid = j < len;
  if (!E.valid) {
#pragma unroll
    for (int i = 0; i < L; ++i) { E.a[i] = 0u; E.x[i] = 0u; }
    E.w = 0; E.ex = 0; E.sx = 0u;
    return;
  }
  const int64_t e = e0 + j;
  E.w = __ldg(P.expw + e);
  load_a<L>(P.limbs, e >> 5, lane, E.a);
  load_x<L>(x.limbs, col, E.x);
  E.ex = __ldg(x.exps + col);
  E.sx = __ldg(x.signs + col);
}

// DENSE (mpsp_dense_create): every row holds all n columns in order, so the
// column of entry j is j itself - no index array is read.
template <bool DENSE = false>
__device__ __forceinline__ int wcol(const PartView& P, int64_t e0, int jb, int len, int lane) {
  if constexpr (DENSE) return (jb + lane < len) ? jb + lane : 0;
  return (jb + lane < len) ? __ldg(P.col + e0 + jb + lane) : 0;
}

#ifndef MPSP_WROW_MINB
#define MPSP_WROW_MINB 1
#endif
template <int L, bool DENSE = false>
__global__ void __launch_bounds__(128, (L <= 8 ? MPSP_WROW_MINB : 1)) spmv_wrow(PartView P, XView x, YView y) {
  const int64_t w = P.npcrow + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= P.nwrow) return;
  const int64_t e0 = P.wrow_ptr[w];
  const int len = P.wrow_len[w];
  const int row = P.wrow_row[w];
  WChain<L> ch;
  ch.init();

  WEntry<L> nxt;
  int cnext = 0;                      // columns of the block after the prefetched one
  if (WPrefetch<L>::on) {
    wload<L>(P, x, e0, 0, len, lane, wcol<DENSE>(P, e0, 0, len, lane), nxt);
    cnext = wcol<DENSE>(P, e0, 32, len, lane);
  } else {
    cnext = wcol<DENSE>(P, e0, 0, len, lane);
  }
  for (int jb = 0; jb < len; jb += 32) {
    MP<L> t;
    {
      WEntry<L> cur;
      if constexpr (WPrefetch<L>::on) {
        cur = nxt;
        if (jb + 32 < len) {
          wload<L>(P, x, e0, jb + 32, len, lane, cnext, nxt);
          cnext = wcol<DENSE>(P, e0, jb + 64, len, lane);
        }
      } else {
        wload<L>(P, x, e0, jb, len, lane, cnext, cur);
        cnext = wcol<DENSE>(P, e0, jb + 32, len, lane);
      }
      const int32_t ea = (int32_t)((uint32_t)cur.w << 1) >> 1;
      mp_mul<L>(cur.a, ea, (uint32_t)cur.w >> 31, cur.x, cur.ex, cur.sx, t);
    }
    ch.consume(t, lane);
  }
  MP<L> s;
  ch.exact(s);
  if (lane == 0 && row >= 0) store_y<L>(y, row, s);
}

// --------------------------------------------------------------------------
// spmv_pcrow<L>: the longest rows, one CTA per row, products and chain in
// different warps.  U = pc_spl(L) producer warps: producer u computes, for
// every 32U-step chunk, the products of steps Uk + u (k = lane; consecutive
// entries in the chunk-permuted layout, layout.h) into a double-buffered
// shared-memory slot; FULL / EMPTY named barriers hand the slots over.  The
// chain warp runs WChainU::consume: lane k owns the U consecutive steps
// Uk .. Uk+U-1, so one block sum (one warp scan, one ballot) advances the
// chain 32U steps and the U per-lane alignments are independent (ILP).
// A tie on the grid is handled as a failing step (exact path).
// --------------------------------------------------------------------------
// Shared-memory chunk of the producer/consumer kernel: per step the raw
// product and its speculative alignment against the tag the producer read.
template <int L, int U>
struct PcSlot {
  uint32_t m[L][U][32];         // raw product mantissa (exact path)
  uint32_t e[U][32], s[U][32];
  uint32_t q[L + 2][U][32];     // aligned, rounded, signed Q
  int32_t h[U][32];
  uint32_t fl[U][32];           // bit0: pre (exact path), bit1: nonzero
  int32_t tagE[U];              // the tag each producer item aligned to
  uint32_t tagS[U], tagZ[U];
};

// The chain over one 32U-step chunk, lane k owning steps Uk .. Uk+U-1.  The
// first pass uses the producers' pre-aligned Q where their tag equals the
// chain's state; any restart (after an exact step changed the binade)
// re-aligns from the raw products.
template <int L, int U>
__device__ __forceinline__ void consume_slot(WChain<L>& ch, const PcSlot<L, U>& S, int lane) {
  constexpr int N = L + 2;
  constexpr int CS = 32 * U;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int32_t LO = 1 << (HB - 1), HI = 1 << HB;
  bool tz[U];
#pragma unroll
  for (int u = 0; u < U; ++u) tz[u] = !(S.fl[u][lane] & 2u);
  auto prod = [&](int u, MP<L>& t) {
#pragma unroll
    for (int i = 0; i < L; ++i) t.m[i] = S.m[i][u][lane];
    t.e = (int32_t)S.e[u][lane];
    t.s = S.s[u][lane];
  };
  bool first = true;
  int start = 0;
  while (start < CS) {
    if (ch.szero) {
      int fu = U;
#pragma unroll
      for (int u = U - 1; u >= 0; --u)
        if (!tz[u] && U * lane + u >= start) fu = u;
      const unsigned nzm = __ballot_sync(FULL, fu < U);
      if (nzm == 0u) break;
      const int kf = __ffs(nzm) - 1;
      const int uf = __shfl_sync(FULL, fu, kf);
      MP<L> tf;
#pragma unroll
      for (int i = 0; i < L; ++i) tf.m[i] = S.m[i][uf][kf];
      tf.e = (int32_t)S.e[uf][kf];
      tf.s = S.s[uf][kf];
      ch.reset_to(tf, lane);
      start = U * kf + uf + 1;
      first = false;
      continue;
    }
    uint32_t Q[U][N];
    int32_t h[U];
    bool act[U], pre[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      act[u] = (U * lane + u >= start) && !tz[u];
      const bool tag_ok = first && !S.tagZ[u] && S.tagE[u] == ch.E && S.tagS[u] == ch.sg;
      if (tag_ok) {                               // warp-uniform
#pragma unroll
        for (int i = 0; i < N; ++i) Q[u][i] = act[u] ? S.q[i][u][lane] : 0u;
        h[u] = act[u] ? S.h[u][lane] : 0;
        pre[u] = (S.fl[u][lane] & 1u) != 0u;
      } else {
        MP<L> t;
        prod(u, t);
        align_q<L>(t, act[u], ch.E, ch.sg, Q[u], h[u], pre[u]);
      }
    }
    first = false;
    int32_t Hx[U];
    int32_t tot = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) { Hx[u] = tot; tot += h[u]; }
    int32_t Pi = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t v = __shfl_up_sync(FULL, Pi, o);
      if (lane >= o) Pi += v;
    }
    const int32_t X = ch.Shi + Pi - tot;
    int fu = U;
#pragma unroll
    for (int u = U - 1; u >= 0; --u) {
      const int32_t LB = X + Hx[u];
      const int32_t ek = ch.err + U * lane + u;
      const bool ok = !act[u] || (!pre[u] && LB + h[u] - 1 >= LO && LB + ek + h[u] + 1 <= HI);
      if (!ok) fu = u;
    }
    const unsigned failM = __ballot_sync(FULL, fu < U);
    if (failM == 0u) {
#pragma unroll
      for (int u = 0; u < U; ++u) add_n<N>(ch.R, ch.R, Q[u]);
      ch.Shi += __shfl_sync(FULL, Pi, 31);
      ch.err = min(ch.err + CS, 1 << 28);
      break;
    }
    const int kf = __ffs(failM) - 1;
    const int uf = __shfl_sync(FULL, fu, kf);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (lane < kf || (lane == kf && u < uf)) add_n<N>(ch.R, ch.R, Q[u]);
    MP<L> sx, tf;
    ch.exact(sx);
#pragma unroll
    for (int i = 0; i < L; ++i) tf.m[i] = S.m[i][uf][kf];
    tf.e = (int32_t)S.e[uf][kf];
    tf.s = S.s[uf][kf];
    mp_add<L>(sx, tf);
    ch.reset_to(sx, lane);
    start = U * kf + uf + 1;
  }
}

__device__ __forceinline__ void bar_sync_n(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// --------------------------------------------------------------------------
// spmv_pcrow<L>: the longest rows, one CTA per row, products and chain in
// different warps.  U = pc_spl(L) producer warps: producer u computes, for
// every 32U-step chunk, the products of steps Uk + u (k = lane; consecutive
// entries in the chunk-permuted layout, layout.h) AND their grid alignment
// against the chain's last published tag (E, sign) - a speculation, since the
// binade changes rarely - into a double-buffered shared-memory slot handed
// over with FULL / EMPTY named barriers.  The chain warp (WChain, lane k
// owning steps Uk .. Uk+U-1) checks the tag, scans, bounds and commits a
// 32U-step block per pass; stale tags and restarts re-align locally from the
// raw products.  A grid tie takes the exact path.
// --------------------------------------------------------------------------
template <int L>
__global__ void __launch_bounds__(32 * (1 + pc_spl(L))) spmv_pcrow(PartView P, XView x, YView y) {
  constexpr int U = pc_spl(L);
  constexpr int CS = 32 * U;
  constexpr int NT = 32 * (U + 1);                   // barrier participants
  extern __shared__ __align__(16) unsigned char pc_smem[];
  PcSlot<L, U>* slot = reinterpret_cast<PcSlot<L, U>*>(pc_smem);   // [2]
  volatile int32_t* pub = reinterpret_cast<volatile int32_t*>(slot + 2);   // E, sign, zero
  const int64_t w = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e0 = P.wrow_ptr[w];
  const int len = P.wrow_len[w];
  const int nch = (len + CS - 1) / CS;
  if (threadIdx.x == 0) { pub[0] = 0; pub[1] = 0; pub[2] = 1; }
  __syncthreads();
  if (warp > 0) {
    // producer u: positions c*CS + 32u + lane, step c*CS + U*lane + u
    const int u = warp - 1;
    auto colof = [&](int c) {
      return (c * CS + U * lane + u < len) ? __ldg(P.col + e0 + c * CS + 32 * u + lane) : 0;
    };
    auto load = [&](int c, int col, WEntry<L>& E) {
      E.valid = c * CS + U * lane + u < len;
      if (!E.valid) {
#pragma unroll
        for (int i = 0; i < L; ++i) { E.a[i] = 0u; E.x[i] = 0u; }
        E.w = 0; E.ex = 0; E.sx = 0u;
        return;
      }
      const int64_t e = e0 + c * CS + 32 * u + lane;
      E.w = __ldg(P.expw + e);
      load_a<L>(P.limbs, e >> 5, lane, E.a);
      load_x<L>(x.limbs, col, E.x);
      E.ex = __ldg(x.exps + col);
      E.sx = __ldg(x.signs + col);
    };
    WEntry<L> nxt;
    int cnext = 0;
    if (nch > 0) {
      load(0, colof(0), nxt);
      cnext = colof(1);
    }
    for (int c = 0; c < nch; ++c) {
      const int j = c & 1;
      WEntry<L> cur = nxt;
      if (c + 1 < nch) {
        load(c + 1, cnext, nxt);
        cnext = colof(c + 2);
      }
      MP<L> t;
      const int32_t ea = (int32_t)((uint32_t)cur.w << 1) >> 1;
      mp_mul<L>(cur.a, ea, (uint32_t)cur.w >> 31, cur.x, cur.ex, cur.sx, t);
      // speculative alignment against the chain's last published tag
      const int32_t tE = pub[0];
      const uint32_t tS = (uint32_t)pub[1], tZ = (uint32_t)pub[2];
      const int32_t tE0 = __shfl_sync(0xffffffffu, tE, 0);          // one tag per item
      const uint32_t tS0 = __shfl_sync(0xffffffffu, tS, 0), tZ0 = __shfl_sync(0xffffffffu, tZ, 0);
      uint32_t Q[L + 2];
      int32_t h = 0;
      bool pre = true;
      const bool nz = !t.is_zero();
      if (!tZ0) align_q<L>(t, nz, tE0, tS0, Q, h, pre);
      if (c >= 2) bar_sync_n(3 + j, NT);                       // EMPTY(j)
      PcSlot<L, U>& S = slot[j];
#pragma unroll
      for (int k = 0; k < L; ++k) S.m[k][u][lane] = t.m[k];
      S.e[u][lane] = (uint32_t)t.e;
      S.s[u][lane] = t.s;
      if (!tZ0) {
#pragma unroll
        for (int k = 0; k < L + 2; ++k) S.q[k][u][lane] = Q[k];
        S.h[u][lane] = h;
      }
      S.fl[u][lane] = (pre ? 1u : 0u) | (nz ? 2u : 0u);
      if (lane == 0) { S.tagE[u] = tE0; S.tagS[u] = tS0; S.tagZ[u] = tZ0; }
      bar_arrive_n(1 + j, NT);                                 // FULL(j)
    }
    return;
  }
  WChain<L> ch;
  ch.init();
  for (int c = 0; c < nch; ++c) {
    const int j = c & 1;
    bar_sync_n(1 + j, NT);                                     // FULL(j)
    consume_slot<L, U>(ch, slot[j], lane);
    if (lane == 0) { pub[0] = ch.E; pub[1] = (int32_t)ch.sg; pub[2] = ch.szero ? 1 : 0; }
    if (c + 2 < nch) bar_arrive_n(3 + j, NT);                  // EMPTY(j)
  }
  MP<L> s;
  ch.exact(s);
  const int row = P.wrow_row[w];
  if (lane == 0 && row >= 0) store_y<L>(y, row, s);
}

template <int L>
static int launch_wrow_L(const PartView& P, const XView& x, const YView& y, cudaStream_t st,
                         bool dense) {
  const int64_t nw = P.nwrow - P.npcrow;
  if (nw <= 0) return 0;
  const int threads = 128;
  const int64_t blocks = (nw * 32 + threads - 1) / threads;
  if (dense)
    spmv_wrow<L, true><<<(unsigned)blocks, threads, 0, st>>>(P, x, y);
  else
    spmv_wrow<L><<<(unsigned)blocks, threads, 0, st>>>(P, x, y);
  launch_counter_add(1);
  return (int)cudaGetLastError();
}

template <int L>
static int launch_pcrow_L(const PartView& P, const XView& x, const YView& y, cudaStream_t st) {
  if (P.npcrow <= 0) return 0;
  constexpr int U = pc_spl(L);
  const size_t smem = 2 * sizeof(PcSlot<L, U>) + 16;
  static std::atomic<uint64_t> attr{0};
  if (int e = ensure_smem_attr((const void*)spmv_pcrow<L>, smem, attr)) return e;
  spmv_pcrow<L><<<(unsigned)P.npcrow, 32 * (1 + U), smem, st>>>(P, x, y);
  launch_counter_add(1);
  return (int)cudaGetLastError();
}

int launch_spmv_long(int L, const PartView& P, const XView& x, const YView& y, void* stream,
                     bool dense) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 1: return launch_wrow_L<1>(P, x, y, st, dense);
    case 2: return launch_wrow_L<2>(P, x, y, st, dense);
    case 4: return launch_wrow_L<4>(P, x, y, st, dense);
    case 8: return launch_wrow_L<8>(P, x, y, st, dense);
    case 16: return launch_wrow_L<16>(P, x, y, st, dense);
    case 32: return launch_wrow_L<32>(P, x, y, st, dense);
    default: return (int)cudaErrorInvalidValue;
  }
}

int launch_spmv_pc(int L, const PartView& P, const XView& x, const YView& y, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 1: return launch_pcrow_L<1>(P, x, y, st);
    case 2: return launch_pcrow_L<2>(P, x, y, st);
    case 4: return launch_pcrow_L<4>(P, x, y, st);
    case 8: return launch_pcrow_L<8>(P, x, y, st);
    case 16: return launch_pcrow_L<16>(P, x, y, st);
    case 32: return launch_pcrow_L<32>(P, x, y, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace mpsp
