// spmv_long.cu - warp-specialised kernel for long rows (hard
// part 2: the ordered add chain of a 5000-long row is a serial critical path).
//
// One CTA owns LR = 8 consecutive length-sorted rows (a quarter of a SELL
// slice).  Warp 0 is the CONSUMER: lane r runs row r's chain
//     s = RN(s + t_j),  j ascending.
// Warps 1..LPW are PRODUCERS: for positions in chunks of LC they compute the
// rounded products t_j = RN(a_j * x[col_j]) (Comba, IMAD.WIDE) and PRE-ALIGN
// them to the consumer's published accumulator exponent E_s (speculation:
// E_s changes in well under 1% of the steps of a long row).  A pre-aligned
// slot holds Y = |t| * 2^32 >> (E_s - E_t) as L+1 limbs (one guard limb) plus
// a sticky flag.  The consumer's fast step is then one (L)-limb carry chain:
//     R = S + Q(Y) + cin,   cin = complement carry + RNE increment,
// valid while the result stays in S's binade.  Everything else is exact
// fallback, never approximation:
//   * E_used != E_s (stale speculation): realign Y by |delta| <= 31 bits
//     (right: bits go to sticky; left, when adding or when the sticky tail is
//     empty: exact for rounding, since only the round bit and "anything
//     below" matter and both stay known);
//   * binade change (carry out / top bit lost) or |delta| > 31 or S == 0
//     without an exact slot: the step is recomputed from S (restored by
//     subtracting back) and the product reloaded, with the general mp_add.
// Chunks are double-buffered in shared memory; one __syncthreads per chunk.
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <cstdlib>

#include "kernel_common.cuh"

namespace mpsp {

constexpr int LR = 8;                      // rows per CTA (consumer lanes)
constexpr int LC = 24;                     // positions per chunk
constexpr int LPW = 3;                     // producer warps
constexpr int LTHREADS = 32 * (1 + LPW);
constexpr int LPROD_PER_LANE = LR * LC / (32 * LPW);   // = 2
static_assert(LR * LC == 32 * LPW * LPROD_PER_LANE, "chunk must tile the producers");
constexpr int32_t KEY_UNKNOWN = INT_MIN;

enum : uint32_t { F_SIGN = 1u, F_STK = 2u, F_ZERO = 4u, F_EXACT = 8u };

template <int L>
struct LongSlot {
  static constexpr int W = L + 3;          // Y[0..L], flags, E_used  (odd stride for even L)
};

// Read at every mpsp_csr_create (tests lower it to route all rows through
// this kernel).
int long_row_threshold() {
  const char* v = std::getenv("MPSP_LONG_T");
  return v ? std::atoi(v) : 64;
}

template <int L>
__device__ __forceinline__ void load_entry(const PartView& P, const XView& x, int64_t g, int l,
                                           uint32_t (&a)[L], int32_t& w, uint32_t (&xv)[L],
                                           int32_t& ex, uint32_t& sx) {
  const int col = __ldg(P.col + g * 32 + l);
  w = __ldg(P.expw + g * 32 + l);
  load_a<L>(P.limbs, g, l, a);
  load_x<L>(x.limbs, col, xv);
  ex = __ldg(x.exps + col);
  sx = __ldg(x.signs + col);
}

template <int L>
__device__ __forceinline__ void product_of(const uint32_t (&a)[L], int32_t w, const uint32_t (&xv)[L],
                                           int32_t ex, uint32_t sx, MP<L>& t) {
  const int32_t ea = (int32_t)((uint32_t)w << 1) >> 1;
  mp_mul<L>(a, ea, (uint32_t)w >> 31, xv, ex, sx, t);
}

// Producer: turn t into a slot aligned to `key` (the consumer's E_s).
template <int L>
__device__ __forceinline__ void write_slot(uint32_t* slot, const MP<L>& t, bool valid, int32_t key) {
  uint32_t Y[L + 1];
  Y[0] = 0u;
#pragma unroll
  for (int i = 0; i < L; ++i) Y[i + 1] = t.m[i];
  uint32_t fl, stk = 0u;
  int32_t eu;
  const bool zero = !valid || t.is_zero();
  int64_t d = (int64_t)key - (int64_t)t.e;
  if (zero) {
    fl = F_ZERO;
    eu = 0;
    d = 0;
  } else if (key == KEY_UNKNOWN || d < 0) {
    fl = F_EXACT | t.s;                    // exact copy of t (d = 0 w.r.t. its own exponent)
    eu = t.e;
    d = 0;
  } else {
    if (d > 32 * (L + 1)) d = 32 * (L + 1);
    fl = t.s | (d == 0 ? F_EXACT : 0u);
    eu = key;
  }
  shr_bits_sticky<L + 1>(Y, (uint32_t)d, stk);
  if (stk) fl |= F_STK;
#pragma unroll
  for (int i = 0; i <= L; ++i) slot[i] = zero ? 0u : Y[i];
  slot[L + 1] = fl;
  slot[L + 2] = (uint32_t)eu;
}

template <int L>
__global__ void __launch_bounds__(LTHREADS) spmv_long(PartView P, XView x, YView y) {
  extern __shared__ uint32_t smem[];
  constexpr int SW = LongSlot<L>::W;
  uint32_t* buf = smem;                                          // [2][LC][LR][SW]
  volatile int32_t* es_pub = (volatile int32_t*)(smem + 2 * LC * LR * SW);
  const int64_t s = blockIdx.x >> 2;
  const int sub = blockIdx.x & 3;
  const int64_t slot0 = s * 32 + sub * LR;
  const int64_t g0 = P.slice_ptr[s] >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int width = P.slot_len[slot0];                           // longest row (sorted)
  if (threadIdx.x < LR) es_pub[threadIdx.x] = KEY_UNKNOWN;
  __syncthreads();
  const int nchunks = (width + LC - 1) / LC;

  // ---- consumer state (warp 0, lanes < LR)
  MP<L> S;
  S.set_zero();
  const bool cons = (warp == 0 && lane < LR);
  // ---- producer constants (warps 1..LPW): row r = lane % LR, positions jj
  const int pr = lane % LR;
  const int pbase = ((warp - 1) * 32 + lane) / LR;               // jj for u = 0
  const int prowlen = (warp > 0) ? P.slot_len[slot0 + pr] : 0;

  for (int c = 0; c <= nchunks; ++c) {
    if (warp > 0 && c < nchunks) {
      uint32_t* B = buf + (c & 1) * (LC * LR * SW);
      const int32_t key = es_pub[pr];
      uint32_t a[LPROD_PER_LANE][L], xv[LPROD_PER_LANE][L];
      int32_t w[LPROD_PER_LANE], ex[LPROD_PER_LANE];
      uint32_t sx[LPROD_PER_LANE];
      bool valid[LPROD_PER_LANE];
#pragma unroll
      for (int u = 0; u < LPROD_PER_LANE; ++u) {
        const int jj = pbase + u * (32 * LPW / LR);
        const int j = c * LC + jj;
        valid[u] = j < prowlen;
        if (valid[u]) {
          load_entry<L>(P, x, g0 + j, sub * LR + pr, a[u], w[u], xv[u], ex[u], sx[u]);
        } else {
#pragma unroll
          for (int i = 0; i < L; ++i) { a[u][i] = 0u; xv[u][i] = 0u; }
          w[u] = 0; ex[u] = 0; sx[u] = 0u;
        }
      }
#pragma unroll
      for (int u = 0; u < LPROD_PER_LANE; ++u) {
        const int jj = pbase + u * (32 * LPW / LR);
        MP<L> t;
        product_of<L>(a[u], w[u], xv[u], ex[u], sx[u], t);
        write_slot<L>(B + (jj * LR + pr) * SW, t, valid[u], key);
      }
    }
    if (cons && c >= 1) {
      const int cc = c - 1;
      const uint32_t* B = buf + (cc & 1) * (LC * LR * SW);
      const int jn = min(LC, width - cc * LC);
      for (int jj = 0; jj < jn; ++jj) {
        const uint32_t* sl = B + (jj * LR + lane) * SW;
        const uint32_t fl = sl[L + 1];
        if (fl & F_ZERO) continue;
        const int32_t eu = (int32_t)sl[L + 2];
        uint32_t Y[L + 1];
#pragma unroll
        for (int i = 0; i <= L; ++i) Y[i] = sl[i];
        uint32_t stk = (fl >> 1) & 1u;
        const uint32_t st_sign = fl & F_SIGN;
        bool slow = false;
        if (S.is_zero()) {
          if (fl & F_EXACT) {                       // S = t exactly
#pragma unroll
            for (int i = 0; i < L; ++i) S.m[i] = Y[i + 1];
            S.e = eu;
            S.s = st_sign;
            es_pub[lane] = S.e;
            continue;
          }
          slow = true;
        } else {
          const int64_t delta = (int64_t)S.e - (int64_t)eu;
          if (delta > 0) {
            if (delta <= 31) {                      // right: shifted-out bits -> sticky
              const uint32_t r = (uint32_t)delta;
              stk |= (Y[0] << (32u - r)) != 0u;
#pragma unroll
              for (int i = 0; i < L; ++i) Y[i] = __funnelshift_r(Y[i], Y[i + 1], r);
              Y[L] >>= r;
            } else {
              slow = true;
            }
          } else if (delta < 0) {
            // left: exact for round/sticky purposes when adding, or when no
            // sticky bits exist (a subtracted sticky tail would borrow)
            const uint32_t r = (uint32_t)(-delta);
            const bool sub_with_stk = ((st_sign ^ S.s) != 0u) && stk;
            if (r <= 31 && __clz(Y[L]) >= (int)r && !sub_with_stk) {
#pragma unroll
              for (int i = L; i > 0; --i) Y[i] = __funnelshift_l(Y[i - 1], Y[i], r);
              Y[0] <<= r;
            } else {
              slow = true;
            }
          }
        }
        if (!slow) {
          // ---- fast step: R = S + Q + cin in S's binade
          const uint32_t opp = st_sign ^ S.s;
          uint32_t q0, c0;
          if (opp) {                                // Q = -(Y + stk) mod 2^(32(L+1))
            q0 = ~Y[0] + (1u - stk);
            c0 = (Y[0] == 0u && stk == 0u) ? 1u : 0u;
#pragma unroll
            for (int i = 1; i <= L; ++i) Y[i] = ~Y[i];
          } else {
            q0 = Y[0];
            c0 = 0u;
          }
          const uint32_t rb = q0 >> 31;
          const uint32_t st = (q0 << 1) | stk;
          const uint32_t lsb = (S.m[0] ^ Y[1] ^ c0) & 1u;
          const uint32_t inc = rb & ((st != 0u) | lsb);
          const uint32_t cin = c0 + inc;            // 0..2
          uint32_t co;
          {
            uint32_t dummy;
            // carry flag := (cin >= 1); second unit of cin folded into limb 0
            const uint32_t c1 = cin >> 1;
            asm volatile("add.cc.u32 %0, %1, 0xffffffff;" : "=r"(dummy) : "r"(cin & 1u));
            asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(S.m[0]) : "r"(Y[1]));
#pragma unroll
            for (int i = 1; i < L; ++i) asm volatile("addc.cc.u32 %0, %0, %1;" : "+r"(S.m[i]) : "r"(Y[i + 1]));
            asm volatile("addc.u32 %0, 0, 0;" : "=r"(co));
            if (c1) {                               // cin == 2 (complement carry + increment)
              uint32_t co2 = inc_n<L>(S.m, 1u);
              co += co2;
            }
          }
          bool bad;
          if (opp) bad = (co == 0u) || (S.m[L - 1] < 0x80000000u) || (S.m[L - 1] == 0x80000000u && inc);
          else bad = (co != 0u);
          if (bad) {
            // restore S: S = R - Q - cin (mod 2^(32L))
            uint32_t Qh[L];
#pragma unroll
            for (int i = 0; i < L; ++i) Qh[i] = Y[i + 1];
            sub_n<L>(S.m, S.m, Qh, 0u);
            uint32_t cinv[L];
            cinv[0] = cin;
#pragma unroll
            for (int i = 1; i < L; ++i) cinv[i] = 0u;
            sub_n<L>(S.m, S.m, cinv, 0u);
            slow = true;
          }
        }
        if (slow) {
          // ---- exact fallback: reload the entry, general product + add
          const int j = cc * LC + jj;
          uint32_t a[L], xv[L];
          int32_t w, ex;
          uint32_t sx;
          load_entry<L>(P, x, g0 + j, sub * LR + lane, a, w, xv, ex, sx);
          MP<L> t;
          product_of<L>(a, w, xv, ex, sx, t);
          mp_add<L>(S, t);
          es_pub[lane] = S.is_zero() ? KEY_UNKNOWN : S.e;
        }
      }
    }
    __syncthreads();
  }
  if (cons) {
    const int row = P.slot_row[slot0 + lane];
    if (row >= 0) store_y<L>(y, row, S);
  }
}

template <int L>
static int launch_long_L(const PartView& P, const XView& x, const YView& y, cudaStream_t st) {
  if (P.nlong <= 0) return 0;
  const size_t smem = (size_t)(2 * LC * LR * LongSlot<L>::W + LR) * 4;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(spmv_long<L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  spmv_long<L><<<(unsigned)(P.nlong * 4), LTHREADS, smem, st>>>(P, x, y);
  launch_counter_add(1);
  return (int)cudaGetLastError();
}

int launch_spmv_long(int L, const PartView& P, const XView& x, const YView& y, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  switch (L) {
    case 1: return launch_long_L<1>(P, x, y, st);
    case 2: return launch_long_L<2>(P, x, y, st);
    case 4: return launch_long_L<4>(P, x, y, st);
    case 8: return launch_long_L<8>(P, x, y, st);
    case 16: return launch_long_L<16>(P, x, y, st);
    case 32: return launch_long_L<32>(P, x, y, st);
    default: return (int)cudaErrorInvalidValue;
  }
}

}  // namespace mpsp
