// xchg.cu - packing of MP vector elements into one (4L+4)-byte record for
// the multi-GPU x exchange (BASELINE.json
// north_star (4): x replicated by NCCL over NVLink before each application).
//
// A record is L limb words followed by one word expw = (sign << 31) |
// (exp & 0x7fffffff) - the same packing as A's exponent word (layout.h).  The
// exchange moves records (one NCCL call per peer or one all-gather per
// application instead of three); mpsp_vec_unpack scatters received records
// into the ABI vector (limbs / exps / signs) the SpMV kernels read.
// Bit-exact for every valid value (|exp| <= 2^29 fits the 31-bit field).
#include <cuda_runtime.h>

#include <cstdint>

#include "layout.h"

namespace mpsp {

// one thread per record word: coalesced on the record side, and on the limb
// side (consecutive words of consecutive elements are consecutive limbs)
template <int L>
__global__ void vec_pack_kernel(int64_t count, const uint32_t* __restrict__ limbs,
                                const int32_t* __restrict__ exps, const uint8_t* __restrict__ signs,
                                uint32_t* __restrict__ rec) {
  constexpr int R = L + 1;
  const int64_t total = count * R;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / R;
    const int w = (int)(t - i * R);
    rec[t] = w < L ? limbs[i * L + w]
                   : (((uint32_t)signs[i] & 1u) << 31) | ((uint32_t)exps[i] & 0x7fffffffu);
  }
}

template <int L>
__global__ void vec_unpack_kernel(int64_t count, const uint32_t* __restrict__ rec,
                                  uint32_t* __restrict__ limbs, int32_t* __restrict__ exps,
                                  uint8_t* __restrict__ signs) {
  constexpr int R = L + 1;
  const int64_t total = count * R;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / R;
    const int w = (int)(t - i * R);
    const uint32_t v = rec[t];
    if (w < L) {
      limbs[i * L + w] = v;
    } else {
      exps[i] = (int32_t)(v << 1) >> 1;
      signs[i] = (uint8_t)(v >> 31);
    }
  }
}

static unsigned grid_for(int64_t words) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (words + 255) / 256;
  const int64_t cap = (int64_t)sms * 8;          // grid-stride beyond 8 blocks per SM
  return (unsigned)(want < cap ? (want > 0 ? want : 1) : cap);
}

template <int L>
static int pack_L(bool unpack, int64_t count, const uint32_t* limbs_in, const int32_t* exps_in,
                  const uint8_t* signs_in, const uint32_t* rec_in, uint32_t* rec_out,
                  uint32_t* limbs_out, int32_t* exps_out, uint8_t* signs_out, cudaStream_t st) {
  const unsigned g = grid_for(count * (L + 1));
  if (unpack)
    vec_unpack_kernel<L><<<g, 256, 0, st>>>(count, rec_in, limbs_out, exps_out, signs_out);
  else
    vec_pack_kernel<L><<<g, 256, 0, st>>>(count, limbs_in, exps_in, signs_in, rec_out);
  launch_counter_add(1);
  return (int)cudaGetLastError();
}

int launch_vec_pack(int L, bool unpack, int64_t count, const uint32_t* limbs_in,
                    const int32_t* exps_in, const uint8_t* signs_in, const uint32_t* rec_in,
                    uint32_t* rec_out, uint32_t* limbs_out, int32_t* exps_out, uint8_t* signs_out,
                    void* stream) {
  if (count <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
#define MPSP_PACK_CASE(LL)                                                                    \
  case LL:                                                                                    \
    return pack_L<LL>(unpack, count, limbs_in, exps_in, signs_in, rec_in, rec_out, limbs_out, \
                      exps_out, signs_out, st);
  switch (L) {
    MPSP_PACK_CASE(1)
    MPSP_PACK_CASE(2)
    MPSP_PACK_CASE(4)
    MPSP_PACK_CASE(8)
    MPSP_PACK_CASE(16)
    MPSP_PACK_CASE(32)
    MPSP_PACK_CASE(64)
    MPSP_PACK_CASE(128)
    MPSP_PACK_CASE(256)
    default: return (int)cudaErrorInvalidValue;
  }
#undef MPSP_PACK_CASE
}

}  // namespace mpsp
