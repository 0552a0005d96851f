// spmv_long.cu - warp-specialised kernel for long rows (hard
// part 2: the ordered add chain of a 5000-long row is a serial critical path).
//
// One CTA owns LR = 8 consecutive length-sorted rows (a quarter of a SELL
// slice).  One warp is the CONSUMER: lane r runs row r's chain
//     s = RN(s + t_j),  j ascending.
// The other LPW warps are PRODUCERS: for positions in chunks of LC they
// compute the rounded products t_j = RN(a_j * x[col_j]) (Comba, IMAD.WIDE)
// and PRE-ALIGN them against the consumer's published accumulator tag
// (E_s, sign_s) - a speculation, since E_s changes in about 1% of the steps
// of a long row.  For that tag the producer also forms the two's complement
// (opposite signs) and the round-to-nearest-even decision of the step, which
// only depends on the product once the accumulator's binade is fixed:
//     Q = +-(|t| * 2^32 >> (E_s - E_t))  (L+1 limbs, guard limb q0),
//     cin = c0 + [round up] + [tie] * lsb(S + Q),
// so the consumer's fast step is   S := S + Q_up + cin   in S's binade.
//
// The consumer keeps S in CARRY-SAVE form (limbs A_i plus one pending carry
// C_i per limb; carries out of the top limb are dropped, i.e. arithmetic is
// mod 2^(32L), which is exact while S stays in [2^(32L-1), 2^(32L))): a step
// is 2 independent ops per limb instead of an L-deep carry chain.  The lowest
// limb never has a pending carry, so the tie LSB is exact; the binade is
// checked conservatively on the top limb (true top in {T, T+1}).
//
// Everything outside the fast path is exact fallback, never approximation,
// handled in one warp-uniform rare block: stale tag (realign by <= 31 bits:
// right shifts feed the sticky; a left shift keeps the round bit, and a
// subtracted sticky tail < 2^r borrows exactly like the "-1" of the sticky
// trick because the low r bits are zero), zero accumulator, binade margin
// violated, or a binade change: S is restored exactly (resolve carries,
// subtract the step back) and the step redone with the general mp_add on the
// raw product kept in the slot.
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
constexpr int32_t E_UNKNOWN = INT_MIN;

#ifdef MPSP_LONG_PROFILE
// debug build only: per-chunk timestamps of CTA 0 (producer role 1 lane 0,
// consumer lane 0): [chunk][0..3] = prod start, prod end, cons start, cons end
__device__ long long g_long_prof[4096][6];
#define LPROF(c, k) do { if (blockIdx.x == 0 && (c) < 4096) g_long_prof[c][k] = clock64(); } while (0)
#else
#define LPROF(c, k) do { } while (0)
#endif

#ifdef MPSP_LONG_CHECK
// debug build only: first divergence between the fast/rare consumer and a
// reference chain (general mp_add of the raw products) - diagnostics
__device__ unsigned long long g_long_chk[64];
__device__ int g_long_chk_flag;
#endif

// info word bits
enum : uint32_t {
  I_C0 = 1u, I_INC = 2u, I_TIE = 4u, I_ZERO = 8u, I_OPP = 16u, I_STK = 32u, I_SIGNT = 64u,
  I_SU = 128u,
  // exponent gap 0: |Q| may reach 2^(32L), so a wrap mod 2^(32L) would not be
  // visible on the top limb -> always take the exact path
  I_RARE = 256u
};

// Slot (one product of one row).  Part A (read every step, 128-bit loads):
// Q_up[0..L-1], Y0 (magnitude guard limb), info, E_used.  Part B (rare
// path): M[0..L-1] (raw rounded product mantissa), E_t.
template <int L>
struct LongSlot {
  static constexpr int A = (L + 3 + 3) / 4 * 4;
  static constexpr int B = (L + 1 + 3) / 4 * 4;
  static constexpr int W0 = A + B;
  static constexpr int W = ((W0 / 4) % 2 == 1) ? W0 : W0 + 4;   // odd # of 16B -> no conflicts
  static constexpr int QU = 0, Y0 = L, INFO = L + 1, EU = L + 2;
  static constexpr int M = A, ET = A + L;
};

// Read at every mpsp_csr_create (tests lower it to route all rows through
// this kernel).
int long_row_threshold() {
  const char* v = std::getenv("MPSP_LONG_T");
  return v ? std::atoi(v) : 64;
}

template <int L>
struct Entry {
  uint32_t a[L], x[L];
  int32_t w, ex;
  uint32_t sx;
};

template <int L>
__device__ __forceinline__ void load_entry(const PartView& P, const XView& x, int64_t g, int l,
                                           bool valid, Entry<L>& E) {
  if (!valid) {
#pragma unroll
    for (int i = 0; i < L; ++i) { E.a[i] = 0u; E.x[i] = 0u; }
    E.w = 0; E.ex = 0; E.sx = 0u;
    return;
  }
  const int col = __ldg(P.col + g * 32 + l);
  E.w = __ldg(P.expw + g * 32 + l);
  load_a<L>(P.limbs, g, l, E.a);
  load_x<L>(x.limbs, col, E.x);
  E.ex = __ldg(x.exps + col);
  E.sx = __ldg(x.signs + col);
}

// Producer: t = RN(a*x), then its slot against the tag (ek, sk): the
// magnitude is aligned to E_used = ek - MARGIN (so the consumer only ever
// shifts RIGHT by delta = E_s - E_used in [0, 31]: E_s may drop by up to
// MARGIN or grow by up to 31 - MARGIN since the tag was read), the guard
// limb stays in magnitude form, the L upper limbs are complemented when the
// signs differ (Q_up = ~Y_up; the +1 of the two's complement is folded into
// the consumer's carry-in).
constexpr int MARGIN = 2;

template <int L>
__device__ __forceinline__ void produce_slot(uint32_t* slot, const Entry<L>& E, bool valid,
                                             int32_t ek, uint32_t sk) {
  using SL = LongSlot<L>;
  MP<L> t;
  const int32_t ea = (int32_t)((uint32_t)E.w << 1) >> 1;
  mp_mul<L>(E.a, ea, (uint32_t)E.w >> 31, E.x, E.ex, E.sx, t);
  const bool zero = !valid || t.is_zero();
  uint32_t Y[L + 1];
  Y[0] = 0u;
#pragma unroll
  for (int i = 0; i < L; ++i) Y[i + 1] = t.m[i];
  int64_t d = (int64_t)ek - MARGIN - (int64_t)t.e;    // shift used (>= 1 for the fast path)
  const bool rare = (ek == E_UNKNOWN) || d < 1;
  if (rare) d = 0;
  if (d > 32 * (L + 1)) d = 32 * (L + 1);
  uint32_t stk = 0u;
  shr_bits_sticky<L + 1>(Y, (uint32_t)d, stk);
  stk = stk ? 1u : 0u;
  const uint32_t su = rare ? t.s : sk;
  const uint32_t mask = 0u - (t.s ^ su);
  uint32_t info = (stk << 5) | (t.s << 6) | (su << 7) | (rare ? I_RARE : 0u);
  if (zero) info = I_ZERO;
  slot[SL::Y0] = zero ? 0u : Y[0];
#pragma unroll
  for (int i = 0; i < L; ++i) slot[SL::QU + i] = zero ? 0u : (Y[i + 1] ^ mask);
  slot[SL::INFO] = info;
  slot[SL::EU] = (uint32_t)(rare ? t.e : ek - MARGIN);
#pragma unroll
  for (int i = 0; i < L; ++i) slot[SL::M + i] = t.m[i];
  slot[SL::ET] = (uint32_t)t.e;
}

template <int L>
struct ProdPrefetch { static constexpr bool on = (L <= 8); };

// Consumer rare path: exact handling of one step from the exact accumulator
// S (value before the step): general add of the raw product in the slot.
template <int L>
__device__ __forceinline__ void exact_step(MP<L>& S, const uint32_t* sl, uint32_t info) {
  using SL = LongSlot<L>;
  if (info & I_ZERO) return;
  MP<L> t;
#pragma unroll
  for (int i = 0; i < L; ++i) t.m[i] = sl[SL::M + i];
  t.e = (int32_t)sl[SL::ET];
  t.s = (info >> 6) & 1u;
  mp_add<L>(S, t);
}

// One consumer step's branch-free arithmetic for this lane's K limbs of its
// row (LPR lanes per row): realign the slot by E_s - E_used, RNE decision,
// carry-save add with the bottom pending carry (ck > 0) or the carry-in
// (ck == 0).  BLOCK: the margin check assumes up to CG undelivered carries.
constexpr int CG = 4;                       // fast steps per block

template <int K>
struct StepOut {
  uint32_t A1[K], C1[K], Q[K];
  uint32_t co, cin, info;
  bool need, zslot, tag_ok;
};

template <int L, int LPR, int K, bool BLOCK>
__device__ __forceinline__ void cons_compute(const uint32_t* sl, int ck, const uint32_t (&Acs)[K],
                                             const uint32_t (&Ccs)[K], int32_t Ecur, uint32_t Scur,
                                             StepOut<K>& o) {
  using SL = LongSlot<L>;
  const uint32_t info = sl[SL::INFO];
  const int32_t eu = (int32_t)sl[SL::EU];
  const uint32_t Y0 = sl[SL::Y0];
  const uint32_t qw0 = sl[SL::QU];
  const uint32_t opp = ((info >> 6) ^ (info >> 7)) & 1u;     // sign_t != sign used
  const uint32_t mask = 0u - opp;
  uint32_t Qm[K + 1];
#pragma unroll
  for (int i = 0; i <= K; ++i) {
    const int idx = ck * K + i;
    const uint32_t v = sl[SL::QU + (idx < L ? idx : L - 1)];
    Qm[i] = idx < L ? v : mask;                      // sign fill above the top limb
  }
  const int32_t delta = Ecur - eu;
  const bool ok_shift = (delta >= 0) && (delta <= 31);
  const uint32_t r = ok_shift ? (uint32_t)delta : 0u;
  const uint32_t stk0 = (info >> 5) & 1u;
  const uint32_t y1 = qw0 ^ mask;
  const uint32_t y0 = __funnelshift_r(Y0, y1, r);
  const uint32_t stk = stk0 | ((r != 0u && (Y0 << (32u - r)) != 0u) ? 1u : 0u);
#pragma unroll
  for (int i = 0; i < K; ++i) o.Q[i] = __funnelshift_r(Qm[i], Qm[i + 1], r);
  const uint32_t nstk = stk ^ 1u;
  const uint32_t c0 = opp & ((y0 == 0u) ? 1u : 0u) & nstk;
  const uint32_t q0 = (y0 ^ mask) + (opp & nstk);
  const uint32_t rb = q0 >> 31;
  const uint32_t stn = ((q0 << 1) | stk) != 0u ? 1u : 0u;
  const uint32_t lsb = (Acs[0] ^ o.Q[0] ^ c0) & 1u;
  o.cin = c0 + (rb & (stn | lsb));                  // 0..2 (meaningful at ck 0)
  {
    const uint64_t t0 = (uint64_t)Acs[0] + o.Q[0] + (ck == 0 ? o.cin : Ccs[0]);
    o.A1[0] = (uint32_t)t0;
    uint32_t co = (uint32_t)(t0 >> 32);
#pragma unroll
    for (int i = 1; i < K; ++i) {
      o.C1[i] = co;
      const uint64_t ti = (uint64_t)Acs[i] + o.Q[i] + Ccs[i];
      o.A1[i] = (uint32_t)ti;
      co = (uint32_t)(ti >> 32);
    }
    o.co = co;
    o.C1[0] = 0u;
  }
  o.info = info;
  o.zslot = (info & I_ZERO) != 0u;
  o.tag_ok = ok_shift && (((info >> 7) & 1u) == Scur) && !(info & I_RARE);
  if (BLOCK) {
    // top lane: true top in [T, T + 1 + undelivered carries] (the latter only
    // reach the top limb directly when K == 1)
    const uint64_t T = (uint64_t)o.A1[K - 1] + (K > 1 ? o.C1[K - 1] : 0u);
    const uint64_t hi = (K == 1) ? 0xFFFFFFFEull - CG : 0xFFFFFFFEull;
    const bool safe = (ck != LPR - 1) || ((T >= 0x80000001ull) && (T <= hi));
    o.need = !(safe && (o.zslot || o.tag_ok));
  } else {
    o.need = false;                                  // careful mode checks after delivery
  }
}

template <int L>
__global__ void __launch_bounds__(LTHREADS) spmv_long(PartView P, XView x, YView y) {
  extern __shared__ uint32_t smem[];
  using SL = LongSlot<L>;
  constexpr int SW = SL::W;
  uint32_t* buf = smem;                                          // [2][LC][LR][SW]
  // published tag per row: low 32 bits E_s, high 32 bits sign_s (one 64-bit word)
  volatile unsigned long long* key_pub = (volatile unsigned long long*)(smem + 2 * LC * LR * SW);
  const int64_t s = blockIdx.x >> 2;
  const int sub = blockIdx.x & 3;
  const int64_t slot0 = s * 32 + sub * LR;
  const int64_t g0 = P.slice_ptr[s] >> 5;
  // the consumer role rotates over the CTA's warps so that consumers of
  // co-resident CTAs spread over the SM's four schedulers
  const int cw = (int)(blockIdx.x & 3);
  const int hw = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp = (hw - cw + 4) & 3;                            // role: 0 = consumer
  const int width = P.slot_len[slot0];                           // longest row (sorted)
  if (threadIdx.x < LR) key_pub[threadIdx.x] = (unsigned long long)(uint32_t)E_UNKNOWN;
  __syncthreads();
  const int nchunks = (width + LC - 1) / LC;

  // ---- consumer (role 0): LPR lanes per row, K limbs per lane; each row's
  // accumulator S in carry-save form spread over its lanes
  constexpr int LPR = L < 4 ? L : 4;
  constexpr int K = L / LPR;
  const int crow = lane / LPR;                       // row of this lane (>= LR: idle)
  const int ck = lane % LPR;                         // limb group: limbs [ck*K, ck*K+K)
  const bool cons = (warp == 0 && crow < LR);
  const int crw = crow < LR ? crow : 0;              // idle lanes mirror row 0, never commit
  uint32_t Acs[K], Ccs[K];                           // limbs, pending carries into them
#pragma unroll
  for (int i = 0; i < K; ++i) { Acs[i] = 0u; Ccs[i] = 0u; }
  int32_t Ecur = E_UNKNOWN;                          // replicated over the row's lanes
  uint32_t Scur = 0u;
  bool szero = true;
#ifdef MPSP_LONG_CHECK
  MP<L> Sref;
  Sref.set_zero();
#endif
  // ---- producer constants: row r = lane % LR, positions jj
  const int pr = lane % LR;
  const int pbase = ((warp - 1) * 32 + lane) / LR;               // jj for u = 0
  const int prowlen = (warp > 0) ? P.slot_len[slot0 + pr] : 0;
  constexpr int JSTEP = 32 * LPW / LR;
  Entry<L> pre[ProdPrefetch<L>::on ? LPROD_PER_LANE : 1];
  if (ProdPrefetch<L>::on && warp > 0 && nchunks > 0) {
#pragma unroll
    for (int u = 0; u < LPROD_PER_LANE; ++u) {
      const int j = pbase + u * JSTEP;
      load_entry<L>(P, x, g0 + j, sub * LR + pr, j < prowlen, pre[u]);
    }
  }

  for (int c = 0; c <= nchunks; ++c) {
    if (warp > 0 && c < nchunks) {
      if (warp == 1 && lane == 0) LPROF(c, 0);
      uint32_t* B = buf + (c & 1) * (LC * LR * SW);
      const unsigned long long kw = key_pub[pr];
      const int2 key = make_int2((int32_t)(uint32_t)kw, (int32_t)(kw >> 32));
      if constexpr (ProdPrefetch<L>::on) {
        Entry<L> cur[LPROD_PER_LANE];
#pragma unroll
        for (int u = 0; u < LPROD_PER_LANE; ++u) cur[u] = pre[u];
        if (c + 1 < nchunks) {
#pragma unroll
          for (int u = 0; u < LPROD_PER_LANE; ++u) {
            const int j = (c + 1) * LC + pbase + u * JSTEP;
            load_entry<L>(P, x, g0 + j, sub * LR + pr, j < prowlen, pre[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < LPROD_PER_LANE; ++u) {
          const int jj = pbase + u * JSTEP;
          produce_slot<L>(B + (jj * LR + pr) * SW, cur[u], c * LC + jj < prowlen, key.x,
                          (uint32_t)key.y);
        }
      } else {
        Entry<L> cur[LPROD_PER_LANE];
#pragma unroll
        for (int u = 0; u < LPROD_PER_LANE; ++u) {
          const int j = c * LC + pbase + u * JSTEP;
          load_entry<L>(P, x, g0 + j, sub * LR + pr, j < prowlen, cur[u]);
        }
#pragma unroll
        for (int u = 0; u < LPROD_PER_LANE; ++u) {
          const int jj = pbase + u * JSTEP;
          produce_slot<L>(B + (jj * LR + pr) * SW, cur[u], c * LC + jj < prowlen, key.x,
                          (uint32_t)key.y);
        }
      }
      if (warp == 1 && lane == 0) LPROF(c, 1);
    }
    if (warp == 0 && c >= 1) {
      const int cc = c - 1;
      if (lane == 0) LPROF(cc, 2);
      const uint32_t* B = buf + (cc & 1) * (LC * LR * SW);
      const int jn = min(LC, width - cc * LC);
      // careful per-step mode (per-step carry delivery and checks, exact
      // rare path) for the rows in `rrow`, steps [jb, jb+gn)
      auto careful = [&](int jb, int gn, bool rrow) {
        for (int u = 0; u < gn; ++u) {
          const uint32_t* sl = B + ((jb + u) * LR + crw) * SW;
          StepOut<K> o;
          cons_compute<L, LPR, K, false>(sl, ck, Acs, Ccs, Ecur, Scur, o);
          uint32_t cup = __shfl_up_sync(0xffffffffu, o.co, 1);
          if (ck == 0) cup = 0u;
          o.C1[0] = cup;
          const uint64_t T = (uint64_t)o.A1[K - 1] + o.C1[K - 1];
          const bool safe = (ck != LPR - 1) || ((T >= 0x80000001ull) && (T <= 0xFFFFFFFEull));
          const bool need_lane = rrow && (szero ? !o.zslot : !(safe && (o.zslot || o.tag_ok)));
          if (rrow) {
#pragma unroll
            for (int i = 0; i < K; ++i) { Acs[i] = o.A1[i]; Ccs[i] = o.C1[i]; }
          }
          const unsigned bal2 = __ballot_sync(0xffffffffu, need_lane);
          if (bal2 != 0u) {
            const bool need_row = rrow && ((bal2 >> (crow * LPR)) & ((1u << LPR) - 1u)) != 0u;
            uint32_t Af[L], Cf[L], Qf[L];
#pragma unroll
            for (int i = 0; i < L; ++i) {
              const int src = crw * LPR + i / K;
              Af[i] = __shfl_sync(0xffffffffu, Acs[i % K], src);
              Cf[i] = __shfl_sync(0xffffffffu, Ccs[i % K], src);
              Qf[i] = __shfl_sync(0xffffffffu, o.Q[i % K], src);
            }
            const uint32_t cin_row = __shfl_sync(0xffffffffu, o.cin, crw * LPR);
            if (need_row) {
              MP<L> S;
              if (szero) {
                S.set_zero();
              } else {
                add_n<L>(S.m, Af, Cf);               // resolve carries (mod 2^(32L))
                sub_n<L>(S.m, S.m, Qf, 0u);
                uint32_t cv[L];
                cv[0] = cin_row;
#pragma unroll
                for (int i = 1; i < L; ++i) cv[i] = 0u;
                sub_n<L>(S.m, S.m, cv, 0u);
                S.e = Ecur;
                S.s = Scur;
              }
              exact_step<L>(S, sl, o.info);
#pragma unroll
              for (int i = 0; i < K; ++i) {
                uint32_t v = S.m[i];
#pragma unroll
                for (int g = 1; g < LPR; ++g) v = (ck == g) ? S.m[g * K + i] : v;
                Acs[i] = v;
                Ccs[i] = 0u;
              }
              szero = S.is_zero();
              const int32_t Enew = szero ? E_UNKNOWN : S.e;
              const uint32_t Snew = szero ? 0u : S.s;
              if (ck == 0 && (Enew != Ecur || Snew != Scur))
                key_pub[crow] = ((unsigned long long)Snew << 32) | (uint32_t)Enew;
              Ecur = Enew;
              Scur = Snew;
            }
          }
        }
      };
      const int nfull = jn / CG;
      for (int b = 0; b < nfull; ++b) {
        const int jb = b * CG;
        // ---- block of CG fast steps, straight-line code: no branch, vote or
        // shuffle inside; cross-lane carries are counted, delivered at the end
        uint32_t As0[K], Cs0[K];
#pragma unroll
        for (int i = 0; i < K; ++i) { As0[i] = Acs[i]; Cs0[i] = Ccs[i]; }
        bool nacc = false;
        uint32_t cacc = 0u;
#pragma unroll
        for (int u = 0; u < CG; ++u) {
          const uint32_t* sl = B + ((jb + u) * LR + crw) * SW;
          StepOut<K> o;
          cons_compute<L, LPR, K, true>(sl, ck, Acs, Ccs, Ecur, Scur, o);
#ifdef MPSP_LONG_PROFILE
          if (blockIdx.x == 0 && cons && ck == 0 && cc < 4096 && !o.zslot) {
            const int32_t dl = Ecur - (int32_t)sl[SL::EU];
            atomicAdd((unsigned long long*)&g_long_prof[cc][5], (unsigned long long)(dl != MARGIN) << 20);
          }
#endif
#pragma unroll
          for (int i = 0; i < K; ++i) { Acs[i] = o.A1[i]; Ccs[i] = o.C1[i]; }
          Ccs[0] = 0u;                                     // bottom pending consumed
          cacc += o.co;
          nacc = nacc || (cons && (szero ? !o.zslot : o.need));
        }
        {
          uint32_t cup = __shfl_up_sync(0xffffffffu, cacc, 1);
          if (ck == 0) cup = 0u;
          Ccs[0] += cup;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, nacc);
#ifdef MPSP_LONG_PROFILE
        if (blockIdx.x == 0 && lane == 0 && cc < 4096) {
          g_long_prof[cc][4] += (bal != 0u);
          g_long_prof[cc][5] += __popc(bal);
        }
#endif
        if (bal != 0u) {
          const bool rrow = cons && ((bal >> (crow * LPR)) & ((1u << LPR) - 1u)) != 0u;
          if (rrow) {
#pragma unroll
            for (int i = 0; i < K; ++i) { Acs[i] = As0[i]; Ccs[i] = Cs0[i]; }
          }
          careful(jb, CG, rrow);
        }
      }
      if (nfull * CG < jn) careful(nfull * CG, jn - nfull * CG, cons);
      {
        const int jb = 0, gn = jn;
#ifdef MPSP_LONG_CHECK
        for (int u = 0; u < gn; ++u) {
          const uint32_t* sl = B + ((jb + u) * LR + crw) * SW;
          const uint32_t info = sl[SL::INFO];
          if (cons && ck == 0 && !(info & I_ZERO)) {
            MP<L> t;
#pragma unroll
            for (int i = 0; i < L; ++i) t.m[i] = sl[SL::M + i];
            t.e = (int32_t)sl[SL::ET];
            t.s = (info >> 6) & 1u;
            mp_add<L>(Sref, t);
          }
        }
        {
          uint32_t Af[L], Cf[L];
#pragma unroll
          for (int i = 0; i < L; ++i) {
            const int src = crw * LPR + i / K;
            Af[i] = __shfl_sync(0xffffffffu, Acs[i % K], src);
            Cf[i] = __shfl_sync(0xffffffffu, Ccs[i % K], src);
          }
          if (cons && ck == 0) {
            MP<L> Sc;
            add_n<L>(Sc.m, Af, Cf);
            if (szero) Sc.set_zero();
            bool diff = (Sc.is_zero() != Sref.is_zero());
            if (!Sref.is_zero()) {
              for (int i = 0; i < L; ++i) diff |= Sc.m[i] != Sref.m[i];
              diff |= (Ecur != Sref.e) || (Scur != Sref.s);
            }
            if (diff && atomicExch(&g_long_chk_flag, 1) == 0) {
              g_long_chk[0] = blockIdx.x; g_long_chk[1] = crow; g_long_chk[2] = cc * LC + jb;
              g_long_chk[8] = (uint32_t)Ecur; g_long_chk[9] = Scur; g_long_chk[10] = (uint32_t)Sref.e;
              g_long_chk[11] = Sref.s;
              for (int i = 0; i < L && i < 8; ++i) { g_long_chk[16 + i] = Sc.m[i]; g_long_chk[24 + i] = Sref.m[i]; }
            }
          }
        }
#endif
        (void)jb;
        (void)gn;
      }
      if (lane == 0) LPROF(cc, 3);
    }
    __syncthreads();
  }
  if (warp == 0) {
    uint32_t Af[L], Cf[L];
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const int src = crw * LPR + i / K;
      Af[i] = __shfl_sync(0xffffffffu, Acs[i % K], src);
      Cf[i] = __shfl_sync(0xffffffffu, Ccs[i % K], src);
    }
    if (cons && ck == 0) {
      const int row = P.slot_row[slot0 + crow];
      if (row >= 0) {
        MP<L> S;
        add_n<L>(S.m, Af, Cf);
        if (szero) S.set_zero();
        S.e = Ecur;
        S.s = Scur;
        store_y<L>(y, row, S);
      }
    }
  }
}

template <int L>
static int launch_long_L(const PartView& P, const XView& x, const YView& y, cudaStream_t st) {
  if (P.nlong <= 0) return 0;
  const size_t smem = (size_t)(2 * LC * LR * LongSlot<L>::W + 2 * LR) * 4;
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

#ifdef MPSP_LONG_CHECK
extern "C" int mpsp_debug_long_check(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, mpsp::g_long_chk, 64 * sizeof(unsigned long long));
}
#endif
#ifdef MPSP_LONG_PROFILE
extern "C" int mpsp_debug_long_profile(long long* out, int nchunks) {
  if (nchunks > 4096) nchunks = 4096;
  return (int)cudaMemcpyFromSymbol(out, mpsp::g_long_prof, (size_t)nchunks * 6 * sizeof(long long));
}
#endif
