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
  return v ? std::atoi(v) : 256;
}

// One step's operands (a_k, x_col) in registers.
template <int L>
struct WEntry {
  uint32_t a[L], x[L];
  int32_t w, ex;
  uint32_t sx;
};

// Step 32c + lane of a warp row: entry position e0 + 32c + lane, i.e. offset
// `off` = 32c from the lane's base pointers (32-bit offsets, no 64-bit index
// arithmetic per step).  Invalid steps (past the row end) load zero limbs.
template <int L>
struct WRowBase {
  using CT = typename Chunk<L>::T;
  static constexpr int NC = L / Chunk<L>::CW;
  const int32_t* expw;   // + e0 + lane
  const int32_t* col;    // + e0 + lane
  const CT* a;           // chunk (e0/32, c = 0, lane)
  __device__ __forceinline__ void init(const PartView& P, int64_t e0, int lane) {
    expw = P.expw + e0 + lane;
    col = P.col + e0 + lane;
    a = reinterpret_cast<const CT*>(P.limbs) + (e0 >> 5) * NC * 32 + lane;
  }
};

template <int L>
__device__ __forceinline__ void wload(const WRowBase<L>& B, const XView& x, int off, bool valid,
                                      int col, WEntry<L>& E) {
  if (!valid) {
#pragma unroll
    for (int i = 0; i < L; ++i) { E.a[i] = 0u; E.x[i] = 0u; }
    E.w = 0; E.ex = 0; E.sx = 0u;
    return;
  }
  constexpr int NC = WRowBase<L>::NC, CW = Chunk<L>::CW;
  E.w = __ldg(B.expw + off);
  const typename Chunk<L>::T* ap = B.a + (off >> 5) * (NC * 32);
#pragma unroll
  for (int c = 0; c < NC; ++c) unpack_chunk(__ldg(ap + c * 32), &E.a[c * CW]);
  load_x<L>(x.limbs, col, E.x);
  E.ex = __ldg(x.exps + col);
  E.sx = __ldg(x.signs + col);
}

#ifndef MPSP_WROW_MINB
#define MPSP_WROW_MINB 4
#endif
// threads per block (the warps of a block never cooperate: the block size
// only sets the granularity at which an SM's warp slots refill)
#ifndef MPSP_WROW_T
#define MPSP_WROW_T 128
#endif
// ---------------------------------------------------------------------------
// spmv_wrow<L>: one warp per row; per block of 32 steps each lane forms the
// product of its step and the chain advances by WChain::consume.  Operands
// of block c+1 are loaded while block c is processed, its columns one block
// earlier still.  DENSE (mpsp_dense_create): the column of step j is j
// itself - no index array is read.
// ---------------------------------------------------------------------------
template <int L, bool DENSE = false>
__global__ void __launch_bounds__(MPSP_WROW_T, (L <= 8 ? MPSP_WROW_MINB * (128 / MPSP_WROW_T) : 1)) spmv_wrow(PartView P, XView x, YView y) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= P.nwrow) return;
  const int64_t e0 = P.wrow_ptr[w];
  const int len = P.wrow_len[w];
  const int row = P.wrow_row[w];
  const int nb = (len + 31) / 32;
  WChain<L> ch;
  ch.init();
  WRowBase<L> B;
  B.init(P, e0, lane);
  auto valid = [&](int c) { return 32 * c + lane < len; };
  auto colof = [&](int c) -> int {
    if (!valid(c)) return 0;
    if constexpr (DENSE) return 32 * c + lane;
    return __ldg(B.col + 32 * c);
  };
  MP<L> t;
  if constexpr (L <= 16) {
    // operands of block c+1 loaded while block c is processed (registers)
    WEntry<L> nxt;
    int cn = 0;
    if (nb > 0) {
      wload<L>(B, x, 0, valid(0), colof(0), nxt);
      cn = colof(1);
    }
    for (int c = 0; c < nb; ++c) {
      const WEntry<L> cur = nxt;
      if (c + 1 < nb) {
        wload<L>(B, x, 32 * (c + 1), valid(c + 1), cn, nxt);
        cn = colof(c + 2);
      }
      mul_entry<L, true>(cur.a, cur.w, cur.x, cur.ex, cur.sx, t);
      ch.consume(t, lane);
    }
  } else {
    // L = 32: no register prefetch (the operands alone are 64 registers)
    int cn = nb > 0 ? colof(0) : 0;
    for (int c = 0; c < nb; ++c) {
      WEntry<L> cur;
      wload<L>(B, x, 32 * c, valid(c), cn, cur);
      cn = colof(c + 1);
      mul_entry<L, true>(cur.a, cur.w, cur.x, cur.ex, cur.sx, t);
      ch.consume(t, lane);
    }
  }
  MP<L> s;
  ch.exact(s);
  if (lane == 0 && row >= 0) store_y<L>(y, row, s);
}

template <int L>
static int launch_wrow_L(const PartView& P, const XView& x, const YView& y, cudaStream_t st,
                         bool dense) {
  const int64_t nw = P.nwrow;
  if (nw <= 0) return 0;
  const int threads = MPSP_WROW_T;
  const int64_t blocks = (nw * 32 + threads - 1) / threads;
  if (dense)
    spmv_wrow<L, true><<<(unsigned)blocks, threads, 0, st>>>(P, x, y);
  else
    spmv_wrow<L><<<(unsigned)blocks, threads, 0, st>>>(P, x, y);
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

}  // namespace mpsp

#ifdef MPSP_WSTATS
// tuning builds only: read and reset the warp-row chain counters (wchain.cuh)
extern "C" int mpsp_debug_wrow_stats(unsigned long long out[8]) {
  cudaError_t e = cudaMemcpyFromSymbol(out, mpsp::g_wstats, sizeof(unsigned long long) * 8);
  if (e != cudaSuccess) return (int)e;
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return (int)cudaMemcpyToSymbol(mpsp::g_wstats, z, sizeof(z));
}
#endif
