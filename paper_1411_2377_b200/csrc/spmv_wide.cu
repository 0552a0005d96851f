// spmv_wide.cu - SpMV at p > 1024 (p = 2048, 4096, 8192: L = 64, 128, 256;
// SURVEY.md 8(f) rank 3, the paper's solver precisions PAPER.md:388-390,
// 412-418).  One warp per row; every MP value is spread over the warp's
// lanes (lane j holds limbs jK .. jK+K-1, K = L/32), and each product
// t = RN(a x) and each add s = RN(s + t) is computed by the whole warp:
//
//  product: the 2L-1 Comba columns are split so that lane j owns columns
//    c = j + 32u and c + L (u < K): their term counts sum to L for every
//    lane, so the L^2 limb-MACs are balanced exactly (operands broadcast
//    from shared memory, conflict-free: lane j reads x[c - i], distinct
//    banks).  The three-word column sums are summed into limbs lane-locally
//    (lane j: limbs [2Kj, 2Kj+2K)); the lanes' carry words are passed up one
//    lane and the remaining one-bit ripple is resolved for all lanes at once
//    by the carry-lookahead identity on ballots (ripple()).  Normalisation
//    (<= 1 bit) and RNE as in mp_mul, with the sticky from a ballot.
//  add: compare (ballot of differing lanes), far path d >= p+2 returns the
//    larger operand (DESIGN.md far-path lemma), otherwise the smaller one is
//    aligned through shared memory with a 32-bit guard limb + sticky, added /
//    subtracted with the ballot ripple, normalised (carry: right 1; else
//    left by clz; >= 32 bits of cancellation via shared memory), RNE.
// Same values as the oracle's mul/add chain (tests/test_gpu_wide.py).
#include <cuda_runtime.h>

#include <cstdint>

#include "wide_mp.cuh"

namespace mpsp {
namespace wide {

constexpr int WARPS = 4;                       // warps (rows) per block

// One warp per row (the part's rows are all "warp rows", longest first);
// entries entry-major: entry E's L limbs at limbs[E*L ..].
template <int K, bool DENSE>
__global__ void __launch_bounds__(32 * WARPS) spmv_wide(PartView P, XView x, YView y) {
  constexpr int L = 32 * K;
  extern __shared__ uint32_t wsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* sA = wsm + warp * 8 * L;
  uint32_t* sX = sA + L;
  uint32_t* cs = sX + L;                           // 6L words
  const int64_t w = (int64_t)blockIdx.x * WARPS + warp;
  if (w >= P.nwrow) return;
  const int64_t e0 = P.wrow_ptr[w];
  const int len = P.wrow_len[w];
  const int row = P.wrow_row[w];
  WMP<K> s;
  wset_zero<K>(s);
  // entry j+1's operands are loaded while entry j is processed
  uint32_t na[K], nx[K];
  int32_t nw = 0, nex = 0;
  uint32_t nsx = 0u;
  auto fetch = [&](int j) {
    const int64_t e = e0 + j;
    const int col = DENSE ? j : __ldg(P.col + e);   // dense rows: column = position
    nw = __ldg(P.expw + e);
    load_k<K>(P.limbs + e * L + lane * K, na);
    load_k<K>(x.limbs + (int64_t)col * L + lane * K, nx);
    nex = __ldg(x.exps + col);
    nsx = __ldg(x.signs + col);
  };
  if (len > 0) fetch(0);
  for (int j = 0; j < len; ++j) {
    uint32_t a[K], xv[K];
#pragma unroll
    for (int i = 0; i < K; ++i) { a[i] = na[i]; xv[i] = nx[i]; }
    const int32_t wv = nw, exv = nex;
    const uint32_t sxv = nsx;
    if (j + 1 < len) fetch(j + 1);
    WMP<K> t;
    const int32_t ea = expw_exp(wv);
    wmul<K>(a, ea, (uint32_t)wv >> 31, xv, exv, sxv, sA, sX, cs, lane, t);
    wadd<K>(s, t, cs, lane);
    __syncwarp();
  }
  if (row < 0) return;
  const bool z = wzero<K>(s);
  uint32_t* yl = y.limbs + (int64_t)row * L + lane * K;
#pragma unroll
  for (int i = 0; i < K; ++i) yl[i] = s.m[i];
  if (lane == 0) {
    y.exps[row] = z ? 0 : s.e;
    y.signs[row] = z ? (uint8_t)0 : (uint8_t)s.s;
  }
}

template <int K, bool DENSE>
int launch(const PartView& P, const XView& x, const YView& y, cudaStream_t st) {
  if (P.nwrow <= 0) return 0;
  constexpr int L = 32 * K;
  const size_t smem = (size_t)WARPS * 8 * L * 4;
  static std::atomic<uint64_t> attr{0};
  if (int e = ensure_smem_attr((const void*)spmv_wide<K, DENSE>, smem, attr)) return e;
  const int64_t blocks = (P.nwrow + WARPS - 1) / WARPS;
  spmv_wide<K, DENSE><<<(unsigned)blocks, 32 * WARPS, smem, st>>>(P, x, y);
  launch_counter_add(1);
  return (int)cudaGetLastError();
}

}  // namespace wide

int launch_spmv_wide(int L, const PartView& P, const XView& x, const YView& y, void* stream,
                     bool dense) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L * 2 + (dense ? 1 : 0)) {
    case 128: return wide::launch<2, false>(P, x, y, st);
    case 129: return wide::launch<2, true>(P, x, y, st);
    case 256: return wide::launch<4, false>(P, x, y, st);
    case 257: return wide::launch<4, true>(P, x, y, st);
    case 512: return wide::launch<8, false>(P, x, y, st);
    case 513: return wide::launch<8, true>(P, x, y, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace mpsp
