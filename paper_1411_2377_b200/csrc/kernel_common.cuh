// kernel_common.cuh - load/store helpers shared by the SpMV kernels
// (layout.h describes the device layout).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "layout.h"
#include "mp_device.cuh"

namespace mpsp {

// cudaFuncSetAttribute applies to the CURRENT device only: the opt-in to more
// than 48 KB of dynamic shared memory is remembered per device ordinal (a
// process may hold handles on several GPUs).
inline int ensure_smem_attr(const void* fn, size_t bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return (int)e;
  const uint64_t bit = 1ull << (dev & 63);
  if (dev < 64 && (done.load(std::memory_order_relaxed) & bit)) return 0;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return (int)e;
  if (dev < 64) done.fetch_or(bit);
  return 0;
}

// SM count of the current device (the runtime caches the attribute)
inline int current_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

template <int L>
struct Chunk;  // CW-word vector type
template <> struct Chunk<1> { using T = uint32_t; static constexpr int CW = 1; };
template <> struct Chunk<2> { using T = uint2; static constexpr int CW = 2; };
template <int L> struct Chunk { using T = uint4; static constexpr int CW = 4; };

__device__ __forceinline__ void unpack_chunk(uint32_t v, uint32_t* d) { d[0] = v; }
__device__ __forceinline__ void unpack_chunk(const uint2& v, uint32_t* d) { d[0] = v.x; d[1] = v.y; }
__device__ __forceinline__ void unpack_chunk(const uint4& v, uint32_t* d) {
  d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
}

// A entry limbs of group g, lane l.
template <int L>
__device__ __forceinline__ void load_a(const uint32_t* __restrict__ limbs, int64_t g, int l,
                                       uint32_t (&a)[L]) {
  using C = Chunk<L>;
  constexpr int NC = L / C::CW;
  const typename C::T* base = reinterpret_cast<const typename C::T*>(limbs) + g * NC * 32 + l;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    typename C::T v = __ldg(base + c * 32);
    unpack_chunk(v, &a[c * C::CW]);
  }
}

// x element `col` (element-major limbs).
template <int L>
__device__ __forceinline__ void load_x(const uint32_t* __restrict__ xl, int col, uint32_t (&x)[L]) {
  using C = Chunk<L>;
  constexpr int NC = L / C::CW;
  const typename C::T* base = reinterpret_cast<const typename C::T*>(xl) + (int64_t)col * NC;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    typename C::T v = __ldg(base + c);
    unpack_chunk(v, &x[c * C::CW]);
  }
}

// A's packed exponent word (layout.h): bit 31 sign, bits 0-30 the exponent.
__device__ __forceinline__ int32_t expw_exp(int32_t w) { return (int32_t)((uint32_t)w << 1) >> 1; }
__device__ __forceinline__ uint32_t expw_sign(int32_t w) { return (uint32_t)w >> 31; }

// t = RN(a_k * x_col) for one stored entry.  At L = 32 a power-of-two a
// (M_a = 2^(p-1): the product is exact, t is x with the exponent moved) skips
// the multiplication when every active lane's entry is one (a warp-uniform
// branch; C5's diagonal 4 sits at the same step of every interior row).  The
// test reads the loaded limbs (an OR over L-1 limbs, ~L/3 instructions; at
// L = 16 it measured 8% slower on C3, whose entries are never powers of two).
template <int L, bool FW = false>
__device__ __forceinline__ void mul_entry(const uint32_t (&a)[L], int32_t w, const uint32_t (&x)[L],
                                          int32_t ex, uint32_t sx, MP<L>& t) {
  const int32_t ea = expw_exp(w);
  const uint32_t sa = expw_sign(w);
  if constexpr (L >= 32) {
    uint32_t lo = 0u;
#pragma unroll
    for (int i = 0; i < L - 1; ++i) lo |= a[i];
    if (__all_sync(FW ? 0xffffffffu : __activemask(), (lo == 0u) & (a[L - 1] == 0x80000000u))) {
      // a = 2^(ea-1): a x = M_x 2^(ex + ea - 1 - p), exact
      const bool xz = x[L - 1] == 0u;
#pragma unroll
      for (int i = 0; i < L; ++i) t.m[i] = x[i];
      t.e = xz ? 0 : ex + ea - 1;
      t.s = xz ? 0u : (sa ^ sx);
      return;
    }
  }
  mp_mul<L, FW>(a, ea, sa, x, ex, sx, t);
}

template <int L>
__device__ __forceinline__ void store_y(const YView& y, int row, const MP<L>& s) {
  using C = Chunk<L>;
  constexpr int NC = L / C::CW;
  typename C::T* base = reinterpret_cast<typename C::T*>(y.limbs) + (int64_t)row * NC;
  const bool z = s.is_zero();
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    typename C::T v;
    if constexpr (C::CW == 1) {
      v = s.m[c];
    } else if constexpr (C::CW == 2) {
      v = make_uint2(s.m[2 * c], s.m[2 * c + 1]);
    } else {
      v = make_uint4(s.m[4 * c], s.m[4 * c + 1], s.m[4 * c + 2], s.m[4 * c + 3]);
    }
    base[c] = v;
  }
  y.exps[row] = z ? 0 : s.e;
  y.signs[row] = z ? (uint8_t)0 : (uint8_t)s.s;
}

}  // namespace mpsp
