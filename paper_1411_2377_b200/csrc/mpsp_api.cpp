// mpsp_api.cpp - the C ABI of include/mpsp.h: validation, transpose, row
// binning / SELL repack, device upload, argument checks and launches.
//
// Host side of SURVEY.md 8(a) rows a1-a3 (one-off, outside the timed loop):
//   a1 validate + pack: CSR invariants, value encodings
//      (MSB set, |exp| <= 2^29), limbs repacked into the chunk-major SELL
//      layout of layout.h, sign packed into the exponent word.
//   a2 transpose: stable counting sort on column -> ascending row index of A
//      inside each transposed row (BASELINE.json north_star (3)).
//   a3 binning: rows sorted by length (descending, stable) into slices of 32.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <thread>
#include <vector>

#include "../../include/mpsp.h"
#include "layout.h"

using namespace mpsp;

namespace {

thread_local char g_cuda_err[256] = "no error";

int cuda_fail(cudaError_t e) {
  std::snprintf(g_cuda_err, sizeof g_cuda_err, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
  cudaGetLastError();  // clear sticky-free errors
  return MPSP_E_CUDA;
}

template <class F>
void parallel_for(int64_t n, F f) {
  unsigned hw = std::thread::hardware_concurrency();
  int64_t nt = std::max<int64_t>(1, std::min<int64_t>(hw ? hw : 1, 32));
  if (n < (1 << 16)) nt = 1;
  if (nt == 1) { f(0, n); return; }
  std::vector<std::thread> th;
  const int64_t chunk = (n + nt - 1) / nt;
  for (int64_t t = 0; t < nt; ++t) {
    int64_t b = t * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    th.emplace_back([=] { f(b, e); });
  }
  for (auto& x : th) x.join();
}

struct DevPart {
  int64_t nrows = 0, nnz = 0, nslices = 0, nentries = 0, nwrow = 0;
  int32_t max_len = 0;
  int64_t* slice_ptr = nullptr;
  int32_t* slot_row = nullptr;
  int32_t* slot_len = nullptr;
  int32_t* slice_order = nullptr;  // device launch order (null: stored order)
  int64_t* wrow_ptr = nullptr;
  int32_t* wrow_row = nullptr;
  int32_t* wrow_len = nullptr;
  int32_t* col = nullptr;
  int32_t* expw = nullptr;
  uint32_t* limbs = nullptr;
  size_t bytes = 0;
  // row chunks (host pipeline of mpsp_spmv_host): chunk c = local rows
  // [crow[c], crow[c+1]), its SELL slices [cslice[c], cslice[c+1]); its rows
  // read x only below chi[c].  One chunk unless build_part chunked the part.
  std::vector<int64_t> crow, cslice, chi;

  // the part restricted to chunk c's SELL slices (no warp rows)
  PartView chunk_view(int c) const {
    PartView v = view();
    const int64_t s0 = cslice[(size_t)c], s1 = cslice[(size_t)c + 1];
    v.slice_ptr = slice_ptr + s0;
    v.slot_row = slot_row + 32 * s0;
    v.slot_len = slot_len + 32 * s0;
    v.nslices = s1 - s0;
    v.nslots = 32 * (s1 - s0);
    v.slice_order = nullptr;
    v.nwrow = 0;
    return v;
  }

  PartView view() const {
    PartView v;
    v.slice_ptr = slice_ptr; v.slot_row = slot_row; v.slot_len = slot_len;
    v.col = col; v.expw = expw; v.limbs = limbs;
    v.nslices = nslices; v.nslots = nslices * 32;
    v.slice_order = slice_order;
    v.nwrow = nwrow; v.wrow_ptr = wrow_ptr; v.wrow_row = wrow_row; v.wrow_len = wrow_len;
    return v;
  }
  void release() {
    cudaFree(slice_ptr); cudaFree(slot_row); cudaFree(slot_len); cudaFree(slice_order);
    cudaFree(wrow_ptr); cudaFree(wrow_row); cudaFree(wrow_len);
    cudaFree(col); cudaFree(expw); cudaFree(limbs);
    slice_ptr = nullptr; slot_row = nullptr; slot_len = nullptr; slice_order = nullptr;
    wrow_ptr = nullptr; wrow_row = nullptr; wrow_len = nullptr;
    col = nullptr; expw = nullptr; limbs = nullptr;
  }
};

}  // namespace

struct mpsp_csr {
  int dev = 0;
  int p = 0, L = 0;
  int64_t n = 0, rb = 0, re = 0;
  uint32_t flags = 0;
  bool has_t = false;
  bool dense = false;   // mpsp_dense_create: every row holds all n columns
  mutable const void* ptr_ok[6] = {};   // x/y pointers of the last mpsp_spmv(_t) call that passed the checks
  DevPart A, T;
  // fork/join for running the long-row and short-row kernels concurrently
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // host-buffer API workspace (lazily allocated): compute stream, copy
  // streams and per-chunk events of the H2D / kernels / D2H pipeline
  cudaStream_t stream = nullptr, s_h2d = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_x, ev_y;
  void* ws = nullptr;
  size_t ws_bytes = 0;
};

namespace {

bool supported_L(int L) {
  return L == 1 || L == 2 || L == 4 || L == 8 || L == 16 || L == 32 || L == 64 || L == 128 || L == 256;
}

// Build one part (rows [0,nrows) of a local CSR whose entry e of local row r
// is source entry src(r, e)).
//   lrp : local rowptr (int64, nrows+1), entries in order (ascending column)
//   lcol: local column of entry e
//   srck: source index k into (limbs, exps, signs) of entry e (or nullptr:
//         k = k0 + e)
template <class Dummy = void>
int build_part(DevPart& P, int L, int64_t nrows, const int64_t* lrp, const int32_t* lcol,
               const int64_t* srck, int64_t k0, const uint32_t* limbs, const int32_t* exps,
               const uint8_t* signs, bool dense = false, uint64_t* host_check = nullptr) {
  P.nrows = nrows;
  P.nnz = lrp[nrows] - lrp[0];
  // --- a3: stable counting sort of rows by length, descending
  int32_t maxlen = 0;
  for (int64_t r = 0; r < nrows; ++r) maxlen = std::max<int32_t>(maxlen, (int32_t)(lrp[r + 1] - lrp[r]));
  P.max_len = maxlen;
  std::vector<int64_t> cnt((size_t)maxlen + 2, 0);
  for (int64_t r = 0; r < nrows; ++r) cnt[(size_t)(maxlen - (lrp[r + 1] - lrp[r]))]++;
  int64_t acc = 0;
  for (auto& c : cnt) { int64_t t = c; c = acc; acc += t; }
  std::vector<int32_t> order((size_t)nrows);
  for (int64_t r = 0; r < nrows; ++r) order[(size_t)cnt[(size_t)(maxlen - (lrp[r + 1] - lrp[r]))]++] = (int32_t)r;
  // warp rows: the rows longer than the threshold (a prefix of `order`);
  // at p > 1024 (spmv_wide) every row is a warp row, entries entry-major
  const bool wide = L > 32;
  // (few rows - under ~32k - cannot fill the GPU one thread per row: their
  // chains are latency-bound, so rows over 32 entries take a warp each)
  const char* tv = std::getenv("MPSP_LONG_T");
  const int64_t T = (wide || dense) ? -1 : (tv || nrows >= 32768 ? long_row_threshold() : 32);
  int64_t nw = 0;
  while (nw < nrows && lrp[order[(size_t)nw] + 1] - lrp[order[(size_t)nw]] > T) ++nw;
  // Row chunks: a part of short rows only (no warp rows) with many rows is
  // length-sorted within C contiguous row chunks instead of globally, so the
  // host-buffer entry point can pipeline H2D of x, the chunk kernels and D2H
  // of y (mpsp_spmv_host); short rows make the sort scope irrelevant to the
  // device path.  Env MPSP_CHUNKS overrides C (1: no chunks).
  int64_t C = 1;
  if (nw == 0 && !wide && !dense && nrows >= 2 * 65536) C = std::min<int64_t>(8, nrows / 65536);
  if (const char* vc = std::getenv("MPSP_CHUNKS")) C = std::max<int64_t>(1, std::min<int64_t>(64, std::atoll(vc)));
  if (nw > 0 || wide || dense || nrows == 0) C = 1;
  P.crow.assign((size_t)C + 1, 0);
  P.chi.assign((size_t)C, 0);
  for (int64_t c = 0; c <= C; ++c) P.crow[(size_t)c] = nrows * c / C;
  if (C > 1) {
    for (int64_t c = 0; c < C; ++c) {               // stable counting sort per chunk
      const int64_t r0 = P.crow[(size_t)c], r1 = P.crow[(size_t)c + 1];
      std::fill(cnt.begin(), cnt.end(), 0);
      for (int64_t r = r0; r < r1; ++r) cnt[(size_t)(maxlen - (lrp[r + 1] - lrp[r]))]++;
      int64_t a2 = r0;
      for (auto& cc : cnt) { int64_t t = cc; cc = a2; a2 += t; }
      for (int64_t r = r0; r < r1; ++r) order[(size_t)cnt[(size_t)(maxlen - (lrp[r + 1] - lrp[r]))]++] = (int32_t)r;
    }
  }
  for (int64_t c = 0; c < C; ++c) {                 // x window end of each chunk
    int64_t hi = 0;
    for (int64_t r = P.crow[(size_t)c]; r < P.crow[(size_t)c + 1]; ++r)
      if (lrp[r + 1] > lrp[r]) hi = std::max<int64_t>(hi, (int64_t)lcol[lrp[r + 1] - 1 - lrp[0]] + 1);
    P.chi[(size_t)c] = hi;
  }
  P.nwrow = nw;
  std::vector<int64_t> wptr((size_t)nw);
  std::vector<int32_t> wrow((size_t)nw), wlen((size_t)nw);
  int64_t ew = 0;
  for (int64_t i = 0; i < nw; ++i) {
    const int32_t r = order[(size_t)i];
    wptr[(size_t)i] = ew;
    wrow[(size_t)i] = r;
    wlen[(size_t)i] = (int32_t)(lrp[r + 1] - lrp[r]);
    const int64_t cs = wide ? 1 : 32;
    ew += (wlen[(size_t)i] + cs - 1) / cs * cs;
  }
  // SELL slices of the remaining rows (chunk by chunk: a chunk's last slice
  // may be partial)
  P.cslice.assign((size_t)C + 1, 0);
  int64_t nslices = 0;
  for (int64_t c = 0; c < C; ++c) {
    const int64_t m = (c == 0 ? P.crow[1] - nw : P.crow[(size_t)c + 1] - P.crow[(size_t)c]);
    P.cslice[(size_t)c] = nslices;
    nslices += (m + 31) / 32;
  }
  P.cslice[(size_t)C] = nslices;
  P.nslices = nslices;
  std::vector<int64_t> sp((size_t)nslices + 1, 0);
  std::vector<int32_t> srow((size_t)nslices * 32, -1), slen((size_t)nslices * 32, 0);
  sp[0] = ew;
  for (int64_t c = 0; c < C; ++c) {
    const int64_t o0 = (c == 0 ? nw : P.crow[(size_t)c]), o1 = P.crow[(size_t)c + 1];
    for (int64_t s = P.cslice[(size_t)c]; s < P.cslice[(size_t)c + 1]; ++s) {
      int64_t w = 0;
      for (int l = 0; l < 32; ++l) {
        const int64_t slot = s * 32 + l;
        const int64_t oi = o0 + (s - P.cslice[(size_t)c]) * 32 + l;
        if (oi < o1) {
          int32_t r = order[(size_t)oi];
          srow[(size_t)slot] = r;
          slen[(size_t)slot] = (int32_t)(lrp[r + 1] - lrp[r]);
          w = std::max<int64_t>(w, slen[(size_t)slot]);
        }
      }
      sp[(size_t)s + 1] = sp[(size_t)s] + 32 * w;
    }
  }
  const int64_t nent = sp[(size_t)nslices];
  P.nentries = nent;
  const int CW = L < 4 ? L : 4, NC = L / CW;
  // --- a1: repack (host), zero-filled padding
  std::vector<int32_t> hcol, hexp;
  std::vector<uint32_t> hl;
  try {
    hcol.assign((size_t)nent, 0);
    hexp.assign((size_t)nent, 0);
    hl.assign((size_t)nent * (size_t)L, 0u);
  } catch (const std::bad_alloc&) {
    return MPSP_E_NOMEM;
  }
  // entry E <- local entry e: column, packed exponent word, chunk-major limbs
  auto put = [&](int64_t E, int64_t e) {
    const int64_t k = srck ? srck[e] : k0 + e;    // source entry
    const int64_t g = E / 32;
    const int l = (int)(E % 32);
    hcol[(size_t)E] = lcol[e];
    const uint32_t* src = limbs + (size_t)k * L;
    const bool nz = src[L - 1] != 0u;
    hexp[(size_t)E] = nz ? (int32_t)(((uint32_t)signs[k] << 31) | ((uint32_t)exps[k] & 0x7fffffffu)) : 0;
    if (wide) {
      for (int i = 0; i < L; ++i) hl[(size_t)E * L + i] = nz ? src[i] : 0u;
      return;
    }
    for (int c = 0; c < NC; ++c)
      for (int w = 0; w < CW; ++w)
        hl[(size_t)(((g * NC + c) * 32 + l) * CW + w)] = nz ? src[c * CW + w] : 0u;
  };
  parallel_for(nw, [&](int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i) {
      const int32_t r = wrow[(size_t)i];
      for (int64_t j = 0; j < wlen[(size_t)i]; ++j) put(wptr[(size_t)i] + j, lrp[r] + j);
    }
  });
  parallel_for(nslices, [&](int64_t s0, int64_t s1) {
    for (int64_t s = s0; s < s1; ++s) {
      for (int l = 0; l < 32; ++l) {
        const int64_t slot = s * 32 + l;
        const int32_t r = srow[(size_t)slot];
        if (r < 0) continue;
        const int64_t len = slen[(size_t)slot];
        for (int64_t j = 0; j < len; ++j) put((sp[(size_t)s] / 32 + j) * 32 + l, lrp[r] + j);
      }
    }
  });
  if (host_check) {
    // host-only build (mpsp_debug_host_build): no device memory; a checksum
    // of the device arrays instead of the upload
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* d, size_t bytes) {
      const unsigned char* c = (const unsigned char*)d;
      for (size_t i = 0; i < bytes; ++i) h = (h ^ c[i]) * 1099511628211ull;
    };
    mix(sp.data(), sp.size() * 8); mix(srow.data(), srow.size() * 4); mix(slen.data(), slen.size() * 4);
    mix(wptr.data(), wptr.size() * 8); mix(wrow.data(), wrow.size() * 4); mix(wlen.data(), wlen.size() * 4);
    mix(hcol.data(), hcol.size() * 4); mix(hexp.data(), hexp.size() * 4); mix(hl.data(), hl.size() * 4);
    *host_check = h;
    return MPSP_OK;
  }
  // --- upload
  auto up = [&](void** dst, const void* src, size_t bytes) -> int {
    if (bytes == 0) bytes = 16;  // keep pointers valid for empty parts
    cudaError_t e = cudaMalloc(dst, bytes);
    if (e != cudaSuccess) { cudaGetLastError(); return e == cudaErrorMemoryAllocation ? MPSP_E_NOMEM : cuda_fail(e); }
    P.bytes += bytes;
    if (src) {
      e = cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
      if (e != cudaSuccess) return cuda_fail(e);
    }
    return MPSP_OK;
  };
  int rc;
  if ((rc = up((void**)&P.slice_ptr, sp.data(), sp.size() * 8)) ||
      (rc = up((void**)&P.slot_row, srow.data(), srow.size() * 4)) ||
      (rc = up((void**)&P.slot_len, slen.data(), slen.size() * 4)) ||
      (rc = up((void**)&P.wrow_ptr, wptr.data(), wptr.size() * 8)) ||
      (rc = up((void**)&P.wrow_row, wrow.data(), wrow.size() * 4)) ||
      (rc = up((void**)&P.wrow_len, wlen.data(), wlen.size() * 4)) ||
      (rc = up((void**)&P.col, hcol.data(), hcol.size() * 4)) ||
      (rc = up((void**)&P.expw, hexp.data(), hexp.size() * 4)) ||
      (rc = up((void**)&P.limbs, hl.data(), hl.size() * 4)))
    return rc;
  if (C > 1 && nslices > 1) {
    // the device entry point launches every chunk's slices at once: widest
    // first across the chunks, so the longest thread chains start first (in
    // stored order each chunk's widest slices would start one chunk later;
    // C3 measured 226 vs 215 us)
    std::vector<int32_t> ord((size_t)nslices);
    for (int64_t i = 0; i < nslices; ++i) ord[(size_t)i] = (int32_t)i;
    std::stable_sort(ord.begin(), ord.end(), [&](int32_t a, int32_t b) {
      return sp[(size_t)a + 1] - sp[(size_t)a] > sp[(size_t)b + 1] - sp[(size_t)b];
    });
    if ((rc = up((void**)&P.slice_order, ord.data(), ord.size() * 4))) return rc;
  }
  return MPSP_OK;
}

bool env_validate() {
  const char* v = std::getenv("MPSP_VALIDATE");
  return v && v[0] == '1';
}

bool overlap(const void* a, size_t na, const void* b, size_t nb) {
  if (!a || !b || !na || !nb) return false;
  const char* pa = (const char*)a;
  const char* pb = (const char*)b;
  return pa < pb + nb && pb < pa + na;
}

int check_device_ptr(const void* p, int dev) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); return MPSP_E_ARG; }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) return MPSP_E_ARG;
  if (at.device != dev) return MPSP_E_DEVICE;
  return MPSP_OK;
}

__attribute__((unused)) int validate_x_host(int L, int64_t n, const uint32_t* xl, const int32_t* xe) {
  for (int64_t i = 0; i < n; ++i) {
    const uint32_t top = xl[(size_t)i * L + L - 1];
    bool nz = false;
    for (int c = 0; c < L; ++c) nz |= xl[(size_t)i * L + c] != 0u;
    if (nz && !(top >> 31)) return MPSP_E_VALUE;
    if (nz && (xe[i] > (1 << 29) || xe[i] < -(1 << 29))) return MPSP_E_VALUE;
  }
  return MPSP_OK;
}

int do_spmv(const mpsp_csr* A, bool transpose, const uint32_t* xl, const int32_t* xe,
            const uint8_t* xs, uint32_t* yl, int32_t* ye, uint8_t* ys, void* stream,
            bool check_ptrs) {
  if (!A) return MPSP_E_ARG;
  if (transpose && !A->has_t) return MPSP_E_NOTRANS;
  const int L = A->L;
  // empty x / y may be passed as NULL
  if ((A->n > 0 && (!xl || !xe || !xs)) || (A->re > A->rb && (!yl || !ye || !ys))) return MPSP_E_ARG;
  if (A->n == 0 && A->re == A->rb) return MPSP_OK;
  const size_t align = (size_t)(L >= 4 ? 16 : 4 * L);
  if (((uintptr_t)xl % align) || ((uintptr_t)yl % align)) return MPSP_E_ARG;
  const int64_t n = A->n, r = A->re - A->rb;
  const size_t xb[3] = {(size_t)n * L * 4, (size_t)n * 4, (size_t)n};
  const size_t yb[3] = {(size_t)r * L * 4, (size_t)r * 4, (size_t)r};
  const void* xp[3] = {xl, xe, xs};
  const void* yp[3] = {yl, ye, ys};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (overlap(xp[i], xb[i], yp[j], yb[j])) return MPSP_E_ALIAS;
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_fail(e);
  if (cur != A->dev) return MPSP_E_DEVICE;
  // (the six pointers of the last call that passed are remembered: a solver
  // or bench loop re-applying to the same buffers skips the attribute
  // queries.  MPSP_PTR_CACHE=0 queries on every call - for callers that free
  // and re-allocate buffers between calls, include/mpsp.h)
  const void* cur6[6] = {xp[0], xp[1], xp[2], yp[0], yp[1], yp[2]};
  static const bool no_cache = [] {
    const char* v = std::getenv("MPSP_PTR_CACHE");
    return v && v[0] == '0';
  }();
  if (check_ptrs && (no_cache || std::memcmp(cur6, A->ptr_ok, sizeof cur6) != 0)) {
    for (int i = 0; i < 3; ++i) {
      int rc = n > 0 ? check_device_ptr(xp[i], A->dev) : MPSP_OK;
      if (rc) return rc;
      rc = r > 0 ? check_device_ptr(yp[i], A->dev) : MPSP_OK;
      if (rc) return rc;
    }
    std::memcpy(A->ptr_ok, cur6, sizeof cur6);
  }
  if (env_validate() && n > 0) {
    std::vector<uint32_t> hl((size_t)n * L);
    std::vector<int32_t> he((size_t)n);
    if (cudaMemcpy(hl.data(), xl, hl.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(he.data(), xe, he.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
      return cuda_fail(cudaGetLastError());
    int rc = validate_x_host(L, n, hl.data(), he.data());
    if (rc) return rc;
  }
  if (r == 0) return MPSP_OK;
  const DevPart& P = transpose ? A->T : A->A;
  XView xv{xl, xe, xs};
  YView yv{yl, ye, ys};
  const PartView pv = P.view();
  if (L > 32 || A->dense) {       // p > 1024: warp-cooperative kernel; dense: warp rows
    const int err = L > 32 ? launch_spmv_wide(L, pv, xv, yv, stream, A->dense)
                           : launch_spmv_long(L, pv, xv, yv, stream, true);
    return err ? cuda_fail((cudaError_t)err) : MPSP_OK;
  }
  const bool has_w = pv.nwrow > 0, has_s = pv.nslots > 0;
  cudaStream_t us = (cudaStream_t)stream;
  cudaError_t ce;
  int err;
  // tuning knob MPSP_FORK (read per call): 1 (default) warp rows on the
  // high-priority aux stream, 2 short rows there instead, 0 both in order on
  // the caller's stream
  static const int fork_mode = [] {
    const char* v = std::getenv("MPSP_FORK");
    return v ? std::atoi(v) : 1;
  }();
  if (has_w && has_s && A->aux && fork_mode != 0) {
    // one kind of rows on the high-priority aux stream (default: the warp
    // rows - the longest rows are the critical path), the other on the
    // caller's stream; joined back there
    const bool w_aux = fork_mode != 2;
    if ((ce = cudaEventRecord(A->ev_fork, us)) != cudaSuccess) return cuda_fail(ce);
    if ((ce = cudaStreamWaitEvent(A->aux, A->ev_fork, 0)) != cudaSuccess) return cuda_fail(ce);
    if ((err = w_aux ? launch_spmv_long(L, pv, xv, yv, A->aux) : launch_spmv(L, pv, xv, yv, A->aux)) != 0)
      return cuda_fail((cudaError_t)err);
    if ((ce = cudaEventRecord(A->ev_join, A->aux)) != cudaSuccess) return cuda_fail(ce);
    if ((err = w_aux ? launch_spmv(L, pv, xv, yv, stream) : launch_spmv_long(L, pv, xv, yv, stream)) != 0)
      return cuda_fail((cudaError_t)err);
    if ((ce = cudaStreamWaitEvent(us, A->ev_join, 0)) != cudaSuccess) return cuda_fail(ce);
    return MPSP_OK;
  }
  if ((err = launch_spmv_long(L, pv, xv, yv, stream)) != 0) return cuda_fail((cudaError_t)err);
  if ((err = launch_spmv(L, pv, xv, yv, stream)) != 0) return cuda_fail((cudaError_t)err);
  return MPSP_OK;
}

}  // namespace

extern "C" {

const char* mpsp_strerror(int code) {
  switch (code) {
    case MPSP_OK: return "ok";
    case MPSP_E_ARG: return "invalid argument (null pointer, bad size or range, misaligned)";
    case MPSP_E_PREC: return "unsupported precision (p must be 32, 64, ..., 8192, a power of two times 32; the solvers: 128 <= p <= 1024)";
    case MPSP_E_CSR: return "invalid CSR structure (rowptr/colidx)";
    case MPSP_E_UNSORTED: return "column indices not strictly increasing within a row";
    case MPSP_E_VALUE: return "invalid value (unnormalised nonzero mantissa or |exp| > 2^29)";
    case MPSP_E_NOMEM: return "out of memory";
    case MPSP_E_CUDA: return "CUDA error";
    case MPSP_E_ALIAS: return "x and y storage overlap";
    case MPSP_E_DEVICE: return "wrong CUDA device for this handle";
    case MPSP_E_NOTRANS: return "handle built without MPSP_WITH_TRANSPOSE";
    default: return "unknown error code";
  }
}

const char* mpsp_last_cuda_error(void) { return g_cuda_err; }

int mpsp_supported_precision(int p_bits) { return p_bits > 0 && p_bits % 32 == 0 && supported_L(p_bits / 32); }

int64_t mpsp_launch_count(void) { return launch_counter_get(); }

static int create_impl(mpsp_csr** out, int p_bits, int64_t n, const int64_t* rowptr,
                       const int32_t* colidx, const uint32_t* limbs, const int32_t* exps,
                       const uint8_t* signs, int64_t row_begin, int64_t row_end, uint32_t flags,
                       bool dense);

int mpsp_csr_create(mpsp_csr** out, int p_bits, int64_t n, const int64_t* rowptr,
                    const int32_t* colidx, const uint32_t* limbs, const int32_t* exps,
                    const uint8_t* signs, int64_t row_begin, int64_t row_end, uint32_t flags) {
  return create_impl(out, p_bits, n, rowptr, colidx, limbs, exps, signs, row_begin, row_end, flags,
                     false);
}

int mpsp_dense_create(mpsp_csr** out, int p_bits, int64_t n, const uint32_t* limbs,
                      const int32_t* exps, const uint8_t* signs, int64_t row_begin,
                      int64_t row_end, uint32_t flags) {
  if (!out) return MPSP_E_ARG;
  *out = nullptr;
  if (n < 0 || row_begin < 0 || row_end < row_begin || row_end > n) return MPSP_E_ARG;
  if (n > 46340) return MPSP_E_CSR;                       // n^2 entries <= 2^31-1
  if (n > 0 && (!limbs || !exps || !signs)) return MPSP_E_ARG;
  // the full pattern: row i holds columns 0..n-1 in order (entry i*n + j)
  std::vector<int64_t> rp;
  std::vector<int32_t> ci;
  try {
    rp.resize((size_t)n + 1);
    ci.resize((size_t)(n * n));
  } catch (const std::bad_alloc&) {
    return MPSP_E_NOMEM;
  }
  for (int64_t i = 0; i <= n; ++i) rp[(size_t)i] = i * n;
  parallel_for(n, [&](int64_t i0, int64_t i1) {
    for (int64_t i = i0; i < i1; ++i)
      for (int64_t j = 0; j < n; ++j) ci[(size_t)(i * n + j)] = (int32_t)j;
  });
  return create_impl(out, p_bits, n, rp.data(), ci.data(), limbs, exps, signs, row_begin, row_end,
                     flags, true);
}

// a1: argument, CSR-invariant and value-encoding checks of mpsp_csr_create
// (include/mpsp.h lists the codes).
static int validate_csr(int p_bits, int64_t n, const int64_t* rowptr, const int32_t* colidx,
                        const uint32_t* limbs, const int32_t* exps, const uint8_t* signs,
                        int64_t row_begin, int64_t row_end, uint32_t flags) {
  if (n < 0 || !rowptr || row_begin < 0 || row_end < row_begin || row_end > n) return MPSP_E_ARG;
  if (flags & ~MPSP_WITH_TRANSPOSE) return MPSP_E_ARG;
  if (!mpsp_supported_precision(p_bits)) return MPSP_E_PREC;
  if (n > INT32_MAX) return MPSP_E_CSR;
  const int L = p_bits / 32;
  if (rowptr[0] != 0) return MPSP_E_CSR;
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) return MPSP_E_CSR;
  const int64_t nnz = rowptr[n];
  if (nnz > INT32_MAX) return MPSP_E_CSR;
  if (nnz > 0 && (!colidx || !limbs || !exps || !signs)) return MPSP_E_ARG;
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      if (colidx[k] < 0 || colidx[k] >= n) return MPSP_E_CSR;
    }
  }
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rowptr[i] + 1; k < rowptr[i + 1]; ++k)
      if (colidx[k] <= colidx[k - 1]) return MPSP_E_UNSORTED;
  std::atomic<int> bad{0};
  parallel_for(nnz, [&](int64_t k0, int64_t k1) {
    for (int64_t k = k0; k < k1; ++k) {
      const uint32_t* m = limbs + (size_t)k * L;
      bool nz = false;
      for (int c = 0; c < L; ++c) nz |= m[c] != 0u;
      if (!nz) continue;
      if (!(m[L - 1] >> 31) || exps[k] > (1 << 29) || exps[k] < -(1 << 29)) bad.store(1);
    }
  });
  return bad.load() ? MPSP_E_VALUE : MPSP_OK;
}

// a2 + a3: rows [row_begin, row_end) of A, and of A^T with MPSP_WITH_TRANSPOSE
// (stable counting sort on column: ascending row index of A inside each
// transposed row), binned and repacked.  check != nullptr: host only (no
// device memory), check[0] / check[1] receive the parts' array checksums.
static int build_parts(mpsp_csr* H, int L, int64_t n, const int64_t* rowptr, const int32_t* colidx,
                       const uint32_t* limbs, const int32_t* exps, const uint8_t* signs,
                       int64_t row_begin, int64_t row_end, uint32_t flags, bool dense,
                       uint64_t* check) {
  const int64_t nnz = rowptr[n];
  const int64_t nrows = row_end - row_begin;
  int rc = MPSP_OK;
  {
    std::vector<int64_t> lrp((size_t)nrows + 1);
    const int64_t k0 = rowptr[row_begin];
    for (int64_t r = 0; r <= nrows; ++r) lrp[(size_t)r] = rowptr[row_begin + r] - k0;
    rc = build_part(H->A, L, nrows, lrp.data(), colidx + k0, nullptr, k0, limbs, exps, signs, dense,
                    check ? &check[0] : nullptr);
  }
  if (rc == MPSP_OK && (flags & MPSP_WITH_TRANSPOSE)) {
    H->has_t = true;
    try {
      std::vector<int64_t> tcnt((size_t)n + 1, 0);
      for (int64_t k = 0; k < nnz; ++k) tcnt[(size_t)colidx[k] + 1]++;
      for (int64_t j = 0; j < n; ++j) tcnt[(size_t)j + 1] += tcnt[(size_t)j];
      const int64_t t0 = tcnt[(size_t)row_begin], t1 = tcnt[(size_t)row_end];
      std::vector<int64_t> next(tcnt.begin(), tcnt.end() - 1);
      std::vector<int32_t> tcol((size_t)(t1 - t0));
      std::vector<int64_t> tsrc((size_t)(t1 - t0));
      for (int64_t i = 0; i < n; ++i) {          // ascending row index of A
        for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
          const int64_t j = colidx[k];
          if (j < row_begin || j >= row_end) continue;
          const int64_t pos = next[(size_t)j]++ - t0;
          tcol[(size_t)pos] = (int32_t)i;
          tsrc[(size_t)pos] = k;
        }
      }
      std::vector<int64_t> lrp((size_t)nrows + 1);
      for (int64_t r = 0; r <= nrows; ++r) lrp[(size_t)r] = tcnt[(size_t)(row_begin + r)] - t0;
      rc = build_part(H->T, L, nrows, lrp.data(), tcol.data(), tsrc.data(), 0, limbs, exps, signs,
                      dense, check ? &check[1] : nullptr);
    } catch (const std::bad_alloc&) {
      rc = MPSP_E_NOMEM;
    }
  }
  return rc;
}

static int create_impl(mpsp_csr** out, int p_bits, int64_t n, const int64_t* rowptr,
                       const int32_t* colidx, const uint32_t* limbs, const int32_t* exps,
                       const uint8_t* signs, int64_t row_begin, int64_t row_end, uint32_t flags,
                       bool dense) {
  if (!out) return MPSP_E_ARG;
  *out = nullptr;
  int rc = validate_csr(p_bits, n, rowptr, colidx, limbs, exps, signs, row_begin, row_end, flags);
  if (rc) return rc;
  const int L = p_bits / 32;
  int dev = 0;
  cudaError_t ce = cudaGetDevice(&dev);
  if (ce != cudaSuccess) return cuda_fail(ce);
  mpsp_csr* H = new (std::nothrow) mpsp_csr();
  if (!H) return MPSP_E_NOMEM;
  H->dev = dev; H->p = p_bits; H->L = L; H->n = n; H->rb = row_begin; H->re = row_end;
  H->flags = flags;
  H->dense = dense;
  rc = build_parts(H, L, n, rowptr, colidx, limbs, exps, signs, row_begin, row_end, flags, dense,
                   nullptr);
  if (rc == MPSP_OK && (H->A.nwrow > 0 || H->T.nwrow > 0)) {
    int prio_lo = 0, prio_hi = 0;
    cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
    if ((ce = cudaStreamCreateWithPriority(&H->aux, cudaStreamNonBlocking, prio_hi)) != cudaSuccess ||
        (ce = cudaEventCreateWithFlags(&H->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (ce = cudaEventCreateWithFlags(&H->ev_join, cudaEventDisableTiming)) != cudaSuccess)
      rc = cuda_fail(ce);
  }
  if (rc == MPSP_OK) {
    ce = cudaDeviceSynchronize();
    if (ce != cudaSuccess) rc = cuda_fail(ce);
  }
  if (rc != MPSP_OK) {
    mpsp_destroy(H);
    return rc;
  }
  *out = H;
  return MPSP_OK;
}

int mpsp_debug_host_build(int p_bits, int64_t n, const int64_t* rowptr, const int32_t* colidx,
                          const uint32_t* limbs, const int32_t* exps, const uint8_t* signs,
                          int64_t row_begin, int64_t row_end, uint32_t flags, int64_t out[12]) {
  if (!out) return MPSP_E_ARG;
  int rc = validate_csr(p_bits, n, rowptr, colidx, limbs, exps, signs, row_begin, row_end, flags);
  if (rc) return rc;
  mpsp_csr H;
  uint64_t check[2] = {0, 0};
  rc = build_parts(&H, p_bits / 32, n, rowptr, colidx, limbs, exps, signs, row_begin, row_end, flags,
                   false, check);
  if (rc) return rc;
  const DevPart* ps[2] = {&H.A, &H.T};
  for (int i = 0; i < 2; ++i) {
    out[6 * i + 0] = ps[i]->nnz;
    out[6 * i + 1] = ps[i]->nentries;
    out[6 * i + 2] = ps[i]->nwrow;
    out[6 * i + 3] = ps[i]->nslices;
    out[6 * i + 4] = (int64_t)ps[i]->crow.size() - 1;
    out[6 * i + 5] = (int64_t)check[i];
  }
  return MPSP_OK;
}

void mpsp_destroy(mpsp_csr* A) {
  if (!A) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(A->dev);
  cudaDeviceSynchronize();
  A->A.release();
  A->T.release();
  if (A->ws) cudaFree(A->ws);
  if (A->stream) cudaStreamDestroy(A->stream);
  if (A->s_h2d) cudaStreamDestroy(A->s_h2d);
  if (A->s_d2h) cudaStreamDestroy(A->s_d2h);
  for (cudaEvent_t e : A->ev_x) cudaEventDestroy(e);
  for (cudaEvent_t e : A->ev_y) cudaEventDestroy(e);
  if (A->aux) cudaStreamDestroy(A->aux);
  if (A->ev_fork) cudaEventDestroy(A->ev_fork);
  if (A->ev_join) cudaEventDestroy(A->ev_join);
  cudaSetDevice(cur);
  cudaGetLastError();
  delete A;
}

int mpsp_spmv(const mpsp_csr* A, const uint32_t* x_limbs, const int32_t* x_exps,
              const uint8_t* x_signs, uint32_t* y_limbs, int32_t* y_exps, uint8_t* y_signs,
              void* cuda_stream) {
  return do_spmv(A, false, x_limbs, x_exps, x_signs, y_limbs, y_exps, y_signs, cuda_stream, true);
}

int mpsp_spmv_t(const mpsp_csr* A, const uint32_t* x_limbs, const int32_t* x_exps,
                const uint8_t* x_signs, uint32_t* y_limbs, int32_t* y_exps, uint8_t* y_signs,
                void* cuda_stream) {
  return do_spmv(A, true, x_limbs, x_exps, x_signs, y_limbs, y_exps, y_signs, cuda_stream, true);
}

static int spmv_host(mpsp_csr* A, bool transpose, const uint32_t* xl, const int32_t* xe,
                     const uint8_t* xs, uint32_t* yl, int32_t* ye, uint8_t* ys) {
  if (!A) return MPSP_E_ARG;
  if (transpose && !A->has_t) return MPSP_E_NOTRANS;
  const int L = A->L;
  const int64_t n = A->n, r = A->re - A->rb;
  if ((n > 0 && (!xl || !xe || !xs)) || (r > 0 && (!yl || !ye || !ys))) return MPSP_E_ARG;
  if (n == 0 && r == 0) return MPSP_OK;
  const size_t xb[3] = {(size_t)n * L * 4, (size_t)n * 4, (size_t)n};
  const size_t yb[3] = {(size_t)r * L * 4, (size_t)r * 4, (size_t)r};
  const void* xp[3] = {xl, xe, xs};
  const void* yp[3] = {yl, ye, ys};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      if (overlap(xp[i], xb[i], yp[j], yb[j])) return MPSP_E_ALIAS;
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_fail(e);
  if (cur != A->dev) return MPSP_E_DEVICE;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t need = al(xb[0]) + al(xb[1]) + al(xb[2]) + al(yb[0]) + al(yb[1]) + al(yb[2]) + 256;
  if (!A->stream) {
    e = cudaStreamCreateWithFlags(&A->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e);
  }
  if (A->ws_bytes < need) {
    if (A->ws) cudaFree(A->ws);
    A->ws = nullptr;
    A->ws_bytes = 0;
    e = cudaMalloc(&A->ws, need);
    if (e != cudaSuccess) { cudaGetLastError(); return MPSP_E_NOMEM; }
    A->ws_bytes = need;
  }
  char* base = (char*)A->ws;
  void* dx[3];
  void* dy[3];
  size_t off = 0;
  for (int i = 0; i < 3; ++i) { dx[i] = base + off; off += al(xb[i]); }
  for (int i = 0; i < 3; ++i) { dy[i] = base + off; off += al(yb[i]); }
  const DevPart& P = transpose ? A->T : A->A;
  const int64_t C = (int64_t)P.crow.size() - 1;
  if (C <= 1 || L > 32 || A->dense) {
    for (int i = 0; i < 3; ++i)
      if (xb[i] && (e = cudaMemcpyAsync(dx[i], xp[i], xb[i], cudaMemcpyHostToDevice, A->stream)) != cudaSuccess)
        return cuda_fail(e);
    int rc = do_spmv(A, transpose, (const uint32_t*)dx[0], (const int32_t*)dx[1], (const uint8_t*)dx[2],
                     (uint32_t*)dy[0], (int32_t*)dy[1], (uint8_t*)dy[2], A->stream, false);
    if (rc) return rc;
    void* hy[3] = {yl, ye, ys};
    for (int i = 0; i < 3; ++i)
      if (yb[i] && (e = cudaMemcpyAsync(hy[i], dy[i], yb[i], cudaMemcpyDeviceToHost, A->stream)) != cudaSuccess)
        return cuda_fail(e);
    e = cudaStreamSynchronize(A->stream);
    return e == cudaSuccess ? MPSP_OK : cuda_fail(e);
  }
  // Row-chunk pipeline: chunk c's kernels start once x is
  // on the device up to the chunk's window end chi[c] (H2D in increasing
  // index order on s_h2d), and its y rows go back on s_d2h while the next
  // chunks compute - H2D, kernels and D2H overlap (full duplex on the link).
  if (!A->s_h2d) {
    if ((e = cudaStreamCreateWithFlags(&A->s_h2d, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&A->s_d2h, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e);
  }
  while ((int64_t)A->ev_x.size() < C) {
    cudaEvent_t a = nullptr, b = nullptr;
    if ((e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming)) != cudaSuccess) {
      cudaEventDestroy(a);
      return cuda_fail(e);
    }
    A->ev_x.push_back(a);
    A->ev_y.push_back(b);
  }
  XView xv{(const uint32_t*)dx[0], (const int32_t*)dx[1], (const uint8_t*)dx[2]};
  YView yv{(uint32_t*)dy[0], (int32_t*)dy[1], (uint8_t*)dy[2]};
  int64_t copied = 0, scopied = 0, xneed = 0;
  const size_t esz[3] = {(size_t)L * 4, 4, 1};
  // MPSP_E2E_SMALL (default 1): the exponent and sign arrays (1/(4L+5) of the
  // bytes) move in few copies - x's for the first chunk's window, then the
  // rest at the second chunk, y's after the last chunk - instead of two small
  // DMA transfers per chunk and direction; 0 keeps them per chunk.
  const char* vb = std::getenv("MPSP_E2E_SMALL");
  const bool batch = !(vb && vb[0] == '0');
  auto h2d = [&](int i, int64_t lo, int64_t hi) -> cudaError_t {
    if (hi <= lo) return cudaSuccess;
    return cudaMemcpyAsync((char*)dx[i] + lo * esz[i], (const char*)xp[i] + lo * esz[i],
                           (size_t)(hi - lo) * esz[i], cudaMemcpyHostToDevice, A->s_h2d);
  };
  void* hy[3] = {yl, ye, ys};
  auto d2h = [&](int i, int64_t lo, int64_t hi) -> cudaError_t {
    if (hi <= lo) return cudaSuccess;
    return cudaMemcpyAsync((char*)hy[i] + lo * esz[i], (const char*)dy[i] + lo * esz[i],
                           (size_t)(hi - lo) * esz[i], cudaMemcpyDeviceToHost, A->s_d2h);
  };
  for (int64_t c = 0; c < C; ++c) {
    xneed = std::min<int64_t>(n, std::max<int64_t>(xneed, P.chi[(size_t)c]));
    if ((e = h2d(0, copied, xneed)) != cudaSuccess) return cuda_fail(e);
    copied = std::max(copied, xneed);
    // small arrays: the first chunk's window, then the rest of x at once
    const int64_t sneed = (batch && c > 0) ? n : xneed;
    for (int i = 1; i < 3; ++i)
      if ((e = h2d(i, scopied, sneed)) != cudaSuccess) return cuda_fail(e);
    scopied = std::max(scopied, sneed);
    if ((e = cudaEventRecord(A->ev_x[(size_t)c], A->s_h2d)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaStreamWaitEvent(A->stream, A->ev_x[(size_t)c], 0)) != cudaSuccess) return cuda_fail(e);
    const int err = launch_spmv(L, P.chunk_view((int)c), xv, yv, A->stream);
    if (err) return cuda_fail((cudaError_t)err);
    if ((e = cudaEventRecord(A->ev_y[(size_t)c], A->stream)) != cudaSuccess) return cuda_fail(e);
    if ((e = cudaStreamWaitEvent(A->s_d2h, A->ev_y[(size_t)c], 0)) != cudaSuccess) return cuda_fail(e);
    const int64_t r0 = P.crow[(size_t)c], r1 = P.crow[(size_t)c + 1];
    for (int i = 0; i < 3; ++i) {
      if (batch && i > 0) {
        if (c == C - 1 && (e = d2h(i, 0, r)) != cudaSuccess) return cuda_fail(e);
        continue;
      }
      if ((e = d2h(i, r0, r1)) != cudaSuccess) return cuda_fail(e);
    }
  }
  if ((e = cudaStreamSynchronize(A->s_d2h)) != cudaSuccess) return cuda_fail(e);
  if ((e = cudaStreamSynchronize(A->stream)) != cudaSuccess) return cuda_fail(e);
  return MPSP_OK;
}

int mpsp_spmv_host(mpsp_csr* A, const uint32_t* x_limbs, const int32_t* x_exps,
                   const uint8_t* x_signs, uint32_t* y_limbs, int32_t* y_exps, uint8_t* y_signs) {
  return spmv_host(A, false, x_limbs, x_exps, x_signs, y_limbs, y_exps, y_signs);
}

int mpsp_spmv_t_host(mpsp_csr* A, const uint32_t* x_limbs, const int32_t* x_exps,
                     const uint8_t* x_signs, uint32_t* y_limbs, int32_t* y_exps, uint8_t* y_signs) {
  return spmv_host(A, true, x_limbs, x_exps, x_signs, y_limbs, y_exps, y_signs);
}

static int vec_pack_impl(int p_bits, int64_t count, bool unpack, const uint32_t* limbs_in,
                         const int32_t* exps_in, const uint8_t* signs_in, const uint32_t* rec_in,
                         uint32_t* rec_out, uint32_t* limbs_out, int32_t* exps_out,
                         uint8_t* signs_out, void* stream) {
  if (!mpsp_supported_precision(p_bits)) return MPSP_E_PREC;
  if (count < 0) return MPSP_E_ARG;
  if (count == 0) return MPSP_OK;
  const int L = p_bits / 32;
  const void* ptrs[4] = {unpack ? (const void*)rec_in : (const void*)limbs_in,
                         unpack ? (const void*)limbs_out : (const void*)exps_in,
                         unpack ? (const void*)exps_out : (const void*)signs_in,
                         unpack ? (const void*)signs_out : (const void*)rec_out};
  for (const void* q : ptrs)
    if (!q) return MPSP_E_ARG;
  const size_t rb = (size_t)count * (L + 1) * 4;
  if (unpack ? (overlap(rec_in, rb, limbs_out, (size_t)count * L * 4) ||
                overlap(rec_in, rb, exps_out, (size_t)count * 4) ||
                overlap(rec_in, rb, signs_out, (size_t)count))
             : (overlap(rec_out, rb, limbs_in, (size_t)count * L * 4) ||
                overlap(rec_out, rb, exps_in, (size_t)count * 4) ||
                overlap(rec_out, rb, signs_in, (size_t)count)))
    return MPSP_E_ALIAS;
  const int e = launch_vec_pack(L, unpack, count, limbs_in, exps_in, signs_in, rec_in, rec_out,
                                limbs_out, exps_out, signs_out, stream);
  return e ? cuda_fail((cudaError_t)e) : MPSP_OK;
}

int mpsp_vec_pack(int p_bits, int64_t count, const uint32_t* limbs, const int32_t* exps,
                  const uint8_t* signs, uint32_t* rec, void* cuda_stream) {
  return vec_pack_impl(p_bits, count, false, limbs, exps, signs, nullptr, rec, nullptr, nullptr,
                       nullptr, cuda_stream);
}

int mpsp_vec_unpack(int p_bits, int64_t count, const uint32_t* rec, uint32_t* limbs,
                    int32_t* exps, uint8_t* signs, void* cuda_stream) {
  return vec_pack_impl(p_bits, count, true, nullptr, nullptr, nullptr, rec, nullptr, limbs, exps,
                       signs, cuda_stream);
}

int mpsp_csr_info(const mpsp_csr* A, int64_t info[10]) {
  if (!A || !info) return MPSP_E_ARG;
  info[0] = A->p;
  info[1] = A->n;
  info[2] = A->rb;
  info[3] = A->re;
  info[4] = A->A.nnz;
  info[5] = A->has_t ? A->T.nnz : -1;
  info[6] = (int64_t)(A->A.bytes + A->T.bytes + A->ws_bytes);
  info[7] = A->dev;
  info[8] = A->A.nentries;
  info[9] = A->A.max_len;
  return MPSP_OK;
}

// ---------------------------------------------------------------- BiCG
// PAPER.md:249-297 (Fig. 4, K = I) and 375-380 (parity-tested against the
// test suite's CPU reference of the same steps).
namespace {

int check_vec_args(int p_bits, int64_t n, const void* a, const void* b, const void* c) {
  if (!mpsp_supported_precision(p_bits) || n < 0) return n < 0 ? MPSP_E_ARG : MPSP_E_PREC;
  if (n > 0 && (!a || !b || !c)) return MPSP_E_ARG;
  return MPSP_OK;
}

// exact integer k >= 0 -> ABI limbs/exp/sign at precision p (no rounding: k
// must fit in p bits, which holds for 1, 10^20 and 10^50 at p >= 128)
void encode_int(int L, uint32_t* limbs, int32_t* e, uint8_t* s, const std::vector<uint32_t>& mag) {
  // mag: little-endian 32-bit words of k
  int top = (int)mag.size() - 1;
  while (top >= 0 && mag[(size_t)top] == 0u) --top;
  for (int i = 0; i < L; ++i) limbs[i] = 0u;
  *e = 0; *s = 0;
  if (top < 0) return;
  const int bl = 32 * top + 32 - __builtin_clz(mag[(size_t)top]);
  const int sh = 32 * L - bl;                         // left shift into the mantissa
  for (int i = 0; i <= top; ++i) {
    const uint64_t v = (uint64_t)mag[(size_t)i];
    const int pos = 32 * i + sh;
    const int w = pos / 32, b = pos % 32;
    if (w < L) limbs[w] |= (uint32_t)(v << b);
    if (b && w + 1 < L) limbs[w + 1] |= (uint32_t)(v >> (32 - b));
  }
  *e = bl;
}

std::vector<uint32_t> pow10_words(int k) {
  std::vector<uint32_t> m{1u};
  for (int i = 0; i < k; ++i) {
    uint64_t c = 0;
    for (auto& w : m) {
      const uint64_t t = (uint64_t)w * 10u + c;
      w = (uint32_t)t;
      c = t >> 32;
    }
    if (c) m.push_back((uint32_t)c);
  }
  return m;
}

}  // namespace

int mpsp_dot(int p_bits, int64_t n, const uint32_t* u_limbs, const int32_t* u_exps,
             const uint8_t* u_signs, const uint32_t* v_limbs, const int32_t* v_exps,
             const uint8_t* v_signs, uint32_t* out_limbs, int32_t* out_exps, uint8_t* out_signs,
             void* cuda_stream) {
  int rc = check_vec_args(p_bits, n, u_limbs, v_limbs, out_limbs);
  if (rc) return rc;
  if (!out_limbs || !out_exps || !out_signs) return MPSP_E_ARG;
  const int L = p_bits / 32;
  VecIn u{u_limbs, u_exps, u_signs}, v{v_limbs, v_exps, v_signs};
  YView o{out_limbs, out_exps, out_signs};
  // segmented parallel evaluation needs a scratch buffer (stream-ordered)
  cudaStream_t st = (cudaStream_t)cuda_stream;
  void* work = nullptr;
  const char* ns = std::getenv("MPSP_DOT_ONEWARP");           // debug: plain one-warp chain
  const size_t wb = (ns && ns[0] == '1' && L <= 32) ? 0 : krylov_dot_work_bytes(L, n);
  if (wb && cudaMallocAsync(&work, wb, st) != cudaSuccess) { cudaGetLastError(); return MPSP_E_NOMEM; }
  const int e = krylov_dot(L, n, u, v, o, nullptr, cuda_stream, work);
  if (work) cudaFreeAsync(work, st);
  return e ? cuda_fail((cudaError_t)e) : MPSP_OK;
}

int mpsp_axpy(int p_bits, int64_t n, const uint32_t* a_limbs, const int32_t* a_exps,
              const uint8_t* a_signs, int negate, const uint32_t* x_limbs, const int32_t* x_exps,
              const uint8_t* x_signs, const uint32_t* y_limbs, const int32_t* y_exps,
              const uint8_t* y_signs, uint32_t* z_limbs, int32_t* z_exps, uint8_t* z_signs,
              void* cuda_stream) {
  int rc = check_vec_args(p_bits, n, x_limbs, y_limbs, z_limbs);
  if (rc) return rc;
  if (!a_limbs || !a_exps || !a_signs) return MPSP_E_ARG;
  const int L = p_bits / 32;
  VecIn a{a_limbs, a_exps, a_signs}, x{x_limbs, x_exps, x_signs}, y{y_limbs, y_exps, y_signs};
  YView z{z_limbs, z_exps, z_signs};
  const int e = krylov_axpy(L, n, a, negate ? 1 : 0, x, y, z, nullptr, cuda_stream);
  return e ? cuda_fail((cudaError_t)e) : MPSP_OK;
}

int mpsp_bicg(mpsp_csr* A, const uint32_t* b_limbs, const int32_t* b_exps, const uint8_t* b_signs,
              uint32_t* x_limbs, int32_t* x_exps, uint8_t* x_signs, int max_iter, int* iters,
              int* status, void* cuda_stream) {
  if (!A || !iters || !status || max_iter < 0) return MPSP_E_ARG;
  if (!A->has_t) return MPSP_E_NOTRANS;
  if (A->rb != 0 || A->re != A->n) return MPSP_E_ARG;   // needs the whole matrix
  if (A->p < 128) return MPSP_E_PREC;                     // 10^50 exact in p bits
  const int L = A->L;
  const int64_t n = A->n;
  *iters = 0;
  *status = MPSP_BICG_MAXITER;
  if (n > 0 && (!b_limbs || !b_exps || !b_signs || !x_limbs || !x_exps || !x_signs)) return MPSP_E_ARG;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  cudaError_t ce;
  // workspace: r, rt, p, pt, z, zt (ABI vectors), KS_N scalars, KF_N flags
  const size_t vl = (size_t)n * L * 4, ve = (size_t)n * 4, vs = (size_t)n;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t per = al(vl) + al(ve) + al(vs);
  const size_t sbytes = al((size_t)KS_N * L * 4) + al((size_t)KS_N * 4) + al(KS_N) + 256;
  const size_t dbytes = al(krylov_dot_work_bytes(L, n));
  char* ws = nullptr;
  if ((ce = cudaMalloc(&ws, 6 * per + sbytes + 2 * dbytes)) != cudaSuccess) { cudaGetLastError(); return MPSP_E_NOMEM; }
  void* dwork = dbytes ? (void*)(ws + 6 * per + sbytes) : nullptr;
  void* dwork2 = dbytes ? (void*)(ws + 6 * per + sbytes + dbytes) : nullptr;
  // (r, r) and the next iteration's rho = (r~, r) are independent: forked
  // onto two streams (own workspaces) and joined back on st
  cudaStream_t fs[2] = {};
  cudaEvent_t fe[3] = {};
  const char* nf = std::getenv("MPSP_NOFORK");               // tuning knob: 1 = no forked dots
  bool conc = !(nf && nf[0] == '1');
  for (int j = 0; j < 2 && conc; ++j)
    conc = cudaStreamCreateWithFlags(&fs[j], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&fe[j], cudaEventDisableTiming) == cudaSuccess;
  conc = conc && cudaEventCreateWithFlags(&fe[2], cudaEventDisableTiming) == cudaSuccess;
  if (!conc) cudaGetLastError();
  struct V { uint32_t* l; int32_t* e; uint8_t* s; };
  V vec[6];
  for (int i = 0; i < 6; ++i) {
    char* b0 = ws + i * per;
    vec[i] = V{(uint32_t*)b0, (int32_t*)(b0 + al(vl)), (uint8_t*)(b0 + al(vl) + al(ve))};
  }
  char* sb = ws + 6 * per;
  YView S{(uint32_t*)sb, (int32_t*)(sb + al((size_t)KS_N * L * 4)),
          (uint8_t*)(sb + al((size_t)KS_N * L * 4) + al((size_t)KS_N * 4))};
  int* fl = (int*)(sb + al((size_t)KS_N * L * 4) + al((size_t)KS_N * 4) + al(KS_N));
  V &r = vec[0], &rt = vec[1], &pv = vec[2], &pt = vec[3], &z = vec[4], &zt = vec[5];
  auto in = [](const V& v) { return VecIn{v.l, v.e, v.s}; };
  auto out = [](const V& v) { return YView{v.l, v.e, v.s}; };
  auto sc_in = [&](int i) { return VecIn{S.limbs + (size_t)i * L, S.exps + i, S.signs + i}; };
  auto sc_out = [&](int i) { return YView{S.limbs + (size_t)i * L, S.exps + i, S.signs + i}; };
  int rc = MPSP_OK;
  auto K = [&](int e) { if (e && rc == MPSP_OK) rc = cuda_fail((cudaError_t)e); };
  auto cp = [&](const V& src, const V& dst) {
    if (n == 0) return;
    K((int)cudaMemcpyAsync(dst.l, src.l, vl, cudaMemcpyDeviceToDevice, st));
    K((int)cudaMemcpyAsync(dst.e, src.e, ve, cudaMemcpyDeviceToDevice, st));
    K((int)cudaMemcpyAsync(dst.s, src.s, vs, cudaMemcpyDeviceToDevice, st));
  };
  // constants 1, 10^20, 10^50 (exact integers) and flags
  {
    std::vector<uint32_t> hl((size_t)KS_N * L, 0u);
    std::vector<int32_t> he(KS_N, 0);
    std::vector<uint8_t> hs(KS_N, 0);
    encode_int(L, &hl[(size_t)KS_ONE * L], &he[KS_ONE], &hs[KS_ONE], {1u});
    encode_int(L, &hl[(size_t)KS_T20 * L], &he[KS_T20], &hs[KS_T20], pow10_words(20));
    encode_int(L, &hl[(size_t)KS_T50 * L], &he[KS_T50], &hs[KS_T50], pow10_words(50));
    K((int)cudaMemcpyAsync(S.limbs, hl.data(), hl.size() * 4, cudaMemcpyHostToDevice, st));
    K((int)cudaMemcpyAsync(S.exps, he.data(), he.size() * 4, cudaMemcpyHostToDevice, st));
    K((int)cudaMemcpyAsync(S.signs, hs.data(), hs.size(), cudaMemcpyHostToDevice, st));
    K((int)cudaMemsetAsync(fl, 0, KF_N * sizeof(int), st));
    // synchronous: the host vectors above must outlive the copies
    K((int)cudaStreamSynchronize(st));
  }
  // x_0 = 0, r_0 = b, r~_0 = r_0
  if (n > 0) {
    K((int)cudaMemsetAsync(x_limbs, 0, vl, st));
    K((int)cudaMemsetAsync(x_exps, 0, ve, st));
    K((int)cudaMemsetAsync(x_signs, 0, vs, st));
  }
  V bv{(uint32_t*)b_limbs, (int32_t*)b_exps, (uint8_t*)b_signs};
  V xv{x_limbs, x_exps, x_signs};
  cp(bv, r);
  cp(bv, rt);
  // rr = (r, r) -> KS_RR and rho = (r~, r) -> slot `rslot`, concurrently
  auto rr_rho = [&](int rslot) {
    if (!conc) {
      K(krylov_dot(L, n, in(r), in(r), sc_out(KS_RR), fl, st, dwork));
      K(krylov_dot(L, n, in(rt), in(r), sc_out(rslot), fl, st, dwork2));
      return;
    }
    K((int)cudaEventRecord(fe[2], st));
    K((int)cudaStreamWaitEvent(fs[0], fe[2], 0));
    K((int)cudaStreamWaitEvent(fs[1], fe[2], 0));
    K(krylov_dot(L, n, in(r), in(r), sc_out(KS_RR), fl, fs[0], dwork));
    K(krylov_dot(L, n, in(rt), in(r), sc_out(rslot), fl, fs[1], dwork2));
    K((int)cudaEventRecord(fe[0], fs[0]));
    K((int)cudaEventRecord(fe[1], fs[1]));
    K((int)cudaStreamWaitEvent(st, fe[0], 0));
    K((int)cudaStreamWaitEvent(st, fe[1], 0));
  };
  rr_rho(KS_RHO);
  K(krylov_scalar(L, S, fl, 0, st));
  int hfl[KF_N] = {0, 0, 0, 0};
  for (int i = 1; i <= max_iter && rc == MPSP_OK; ++i) {
    K(krylov_scalar(L, S, fl, 1, st));                       // rho == 0 -> stop
    if (i == 1) {
      cp(r, pv);
      cp(rt, pt);
    } else {
      K(krylov_scalar(L, S, fl, 2, st));                     // beta
      K(krylov_axpy(L, n, sc_in(KS_BETA), 0, in(pv), in(r), out(pv), fl, st));
      K(krylov_axpy(L, n, sc_in(KS_BETA), 0, in(pt), in(rt), out(pt), fl, st));
    }
    for (int tr = 0; tr < 2 && rc == MPSP_OK; ++tr) {          // z = A p, z~ = A^T p~
      const V& src = tr ? pt : pv;
      const V& dst = tr ? zt : z;
      const int e = do_spmv(A, tr == 1, src.l, src.e, src.s, dst.l, dst.e, dst.s, cuda_stream, false);
      if (e != MPSP_OK) rc = e;
    }
    K(krylov_dot(L, n, in(pt), in(z), sc_out(KS_SIGMA), fl, st, dwork));
    K(krylov_scalar(L, S, fl, 3, st));                       // alpha (sigma == 0 -> stop)
    K(krylov_axpy(L, n, sc_in(KS_ALPHA), 0, in(pv), in(xv), out(xv), fl, st));
    K(krylov_axpy(L, n, sc_in(KS_ALPHA), 1, in(z), in(r), out(r), fl, st));
    K(krylov_axpy(L, n, sc_in(KS_ALPHA), 1, in(zt), in(rt), out(rt), fl, st));
    rr_rho(KS_TAU);                                          // rr, next rho (KS_TAU: unused here)
    K(krylov_scalar(L, S, fl, 4, st));                       // ||r|| <= thr -> stop; rho_prev = rho
    {                                                        // rho := the next rho
      K((int)cudaMemcpyAsync(S.limbs + (size_t)KS_RHO * L, S.limbs + (size_t)KS_TAU * L, (size_t)L * 4,
                             cudaMemcpyDeviceToDevice, st));
      K((int)cudaMemcpyAsync(S.exps + KS_RHO, S.exps + KS_TAU, 4, cudaMemcpyDeviceToDevice, st));
      K((int)cudaMemcpyAsync(S.signs + KS_RHO, S.signs + KS_TAU, 1, cudaMemcpyDeviceToDevice, st));
    }
    K((int)cudaMemcpyAsync(hfl, fl, sizeof hfl, cudaMemcpyDeviceToHost, st));
    K((int)cudaStreamSynchronize(st));
    if (rc != MPSP_OK) break;
    if (hfl[KF_BREAK]) { *status = MPSP_BICG_BREAKDOWN; break; }
    *iters = i;
    if (hfl[KF_CONV]) { *status = MPSP_BICG_CONVERGED; break; }
  }
  cudaStreamSynchronize(st);
  for (int j = 0; j < 2; ++j) {
    if (fs[j]) cudaStreamDestroy(fs[j]);
    if (fe[j]) cudaEventDestroy(fe[j]);
  }
  if (fe[2]) cudaEventDestroy(fe[2]);
  cudaFree(ws);
  return rc;
}

int mpsp_gpbicg(mpsp_csr* A, const uint32_t* b_limbs, const int32_t* b_exps, const uint8_t* b_signs,
                uint32_t* x_limbs, int32_t* x_exps, uint8_t* x_signs, int max_iter, int* iters,
                int* status, void* cuda_stream) {
  if (!A || !iters || !status || max_iter < 0) return MPSP_E_ARG;
  if (A->rb != 0 || A->re != A->n) return MPSP_E_ARG;   // needs the whole matrix
  if (A->p < 128) return MPSP_E_PREC;
  const int L = A->L;
  const int64_t n = A->n;
  *iters = 0;
  *status = MPSP_BICG_MAXITER;
  if (n > 0 && (!b_limbs || !b_exps || !b_signs || !x_limbs || !x_exps || !x_signs)) return MPSP_E_ARG;
  cudaStream_t st = (cudaStream_t)cuda_stream;
  cudaError_t ce;
  constexpr int NV = 12;        // r rt u z p q t v w s y zero, + 2 temporaries
  const size_t vl = (size_t)n * L * 4, ve = (size_t)n * 4, vs = (size_t)n;
  auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t per = al(vl) + al(ve) + al(vs);
  const size_t sbytes = al((size_t)KS_N * L * 4) + al((size_t)KS_N * 4) + al(KS_N) + 256;
  const size_t dbytes = al(krylov_dot_work_bytes(L, n));
  constexpr int ND = 5;         // the five independent inner products mu1..mu5 run concurrently
  char* ws = nullptr;
  if ((ce = cudaMalloc(&ws, (NV + 2) * per + sbytes + ND * dbytes)) != cudaSuccess) {
    cudaGetLastError();
    return MPSP_E_NOMEM;
  }
  void* dwk[ND];
  for (int j = 0; j < ND; ++j) dwk[j] = dbytes ? (void*)(ws + (NV + 2) * per + sbytes + j * dbytes) : nullptr;
  void* dwork = dwk[0];
  cudaStream_t dst_[ND] = {};
  cudaEvent_t dev_[ND + 1] = {};
  const char* nf = std::getenv("MPSP_NOFORK");               // tuning knob: 1 = no forked dots
  bool conc = !(nf && nf[0] == '1');
  for (int j = 0; j < ND && conc; ++j)
    conc = cudaStreamCreateWithFlags(&dst_[j], cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&dev_[j], cudaEventDisableTiming) == cudaSuccess;
  conc = conc && cudaEventCreateWithFlags(&dev_[ND], cudaEventDisableTiming) == cudaSuccess;
  if (!conc) cudaGetLastError();
  struct V { uint32_t* l; int32_t* e; uint8_t* s; };
  V vec[NV + 2];
  for (int i = 0; i < NV + 2; ++i) {
    char* b0 = ws + i * per;
    vec[i] = V{(uint32_t*)b0, (int32_t*)(b0 + al(vl)), (uint8_t*)(b0 + al(vl) + al(ve))};
  }
  char* sb = ws + (NV + 2) * per;
  YView S{(uint32_t*)sb, (int32_t*)(sb + al((size_t)KS_N * L * 4)),
          (uint8_t*)(sb + al((size_t)KS_N * L * 4) + al((size_t)KS_N * 4))};
  int* fl = (int*)(sb + al((size_t)KS_N * L * 4) + al((size_t)KS_N * 4) + al(KS_N));
  V &r = vec[0], &rt = vec[1], &u = vec[2], &z = vec[3], &pv = vec[4], &q = vec[5], &t = vec[6],
    &v = vec[7], &w = vec[8], &sv = vec[9], &y = vec[10], &zero = vec[11], &t1 = vec[12], &t2 = vec[13];
  V xv{x_limbs, x_exps, x_signs};
  V bv{(uint32_t*)b_limbs, (int32_t*)b_exps, (uint8_t*)b_signs};
  auto in = [](const V& a) { return VecIn{a.l, a.e, a.s}; };
  auto out = [](const V& a) { return YView{a.l, a.e, a.s}; };
  auto sc_in = [&](int i) { return VecIn{S.limbs + (size_t)i * L, S.exps + i, S.signs + i}; };
  auto sc_out = [&](int i) { return YView{S.limbs + (size_t)i * L, S.exps + i, S.signs + i}; };
  int rc = MPSP_OK;
  auto K = [&](int e) { if (e && rc == MPSP_OK) rc = cuda_fail((cudaError_t)e); };
  auto zero_v = [&](const V& a) {
    if (n == 0) return;
    K((int)cudaMemsetAsync(a.l, 0, vl, st));
    K((int)cudaMemsetAsync(a.e, 0, ve, st));
    K((int)cudaMemsetAsync(a.s, 0, vs, st));
  };
  auto cp = [&](const V& src, const V& dst) {
    if (n == 0) return;
    K((int)cudaMemcpyAsync(dst.l, src.l, vl, cudaMemcpyDeviceToDevice, st));
    K((int)cudaMemcpyAsync(dst.e, src.e, ve, cudaMemcpyDeviceToDevice, st));
    K((int)cudaMemcpyAsync(dst.s, src.s, vs, cudaMemcpyDeviceToDevice, st));
  };
  // out = RN(y + RN(+-c x)): the one vector kernel every update is built from
  auto ax = [&](int c, bool neg, const V& xx, const V& yy, const V& oo) {
    K(krylov_axpy(L, n, sc_in(c), neg ? 1 : 0, in(xx), in(yy), out(oo), fl, st));
  };
  auto spmv = [&](const V& src, const V& dst) {
    const int e = do_spmv(A, false, src.l, src.e, src.s, dst.l, dst.e, dst.s, cuda_stream, false);
    if (e != MPSP_OK && rc == MPSP_OK) rc = e;
  };
  auto dotv = [&](const V& a, const V& b2, int slot) {
    K(krylov_dot(L, n, in(a), in(b2), sc_out(slot), fl, st, dwork));
  };
  auto scal = [&](int op) { K(krylov_scalar(L, S, fl, op, st)); };
  // mu1..mu5: forked onto ND streams (own workspaces), joined back on st
  auto dot5 = [&](const V* xa, const V* xb, const int* slot) {
    if (!conc) {
      for (int j = 0; j < ND; ++j) K(krylov_dot(L, n, in(xa[j]), in(xb[j]), sc_out(slot[j]), fl, st, dwk[j]));
      return;
    }
    K((int)cudaEventRecord(dev_[ND], st));
    for (int j = 0; j < ND; ++j) {
      K((int)cudaStreamWaitEvent(dst_[j], dev_[ND], 0));
      K(krylov_dot(L, n, in(xa[j]), in(xb[j]), sc_out(slot[j]), fl, dst_[j], dwk[j]));
      K((int)cudaEventRecord(dev_[j], dst_[j]));
    }
    for (int j = 0; j < ND; ++j) K((int)cudaStreamWaitEvent(st, dev_[j], 0));
  };
  {
    std::vector<uint32_t> hl((size_t)KS_N * L, 0u);
    std::vector<int32_t> he(KS_N, 0);
    std::vector<uint8_t> hs(KS_N, 0);
    encode_int(L, &hl[(size_t)KS_ONE * L], &he[KS_ONE], &hs[KS_ONE], {1u});
    encode_int(L, &hl[(size_t)KS_T20 * L], &he[KS_T20], &hs[KS_T20], pow10_words(20));
    encode_int(L, &hl[(size_t)KS_T50 * L], &he[KS_T50], &hs[KS_T50], pow10_words(50));
    K((int)cudaMemcpyAsync(S.limbs, hl.data(), hl.size() * 4, cudaMemcpyHostToDevice, st));
    K((int)cudaMemcpyAsync(S.exps, he.data(), he.size() * 4, cudaMemcpyHostToDevice, st));
    K((int)cudaMemcpyAsync(S.signs, hs.data(), hs.size(), cudaMemcpyHostToDevice, st));
    K((int)cudaMemsetAsync(fl, 0, KF_N * sizeof(int), st));
    K((int)cudaStreamSynchronize(st));
  }
  zero_v(xv); zero_v(u); zero_v(z); zero_v(zero);
  cp(bv, r);
  cp(bv, rt);
  dotv(r, r, KS_RR);
  scal(0);                                                    // c1, c2, thr
  int hfl[KF_N] = {0, 0, 0, 0};
  for (int i = 1; i <= max_iter && rc == MPSP_OK; ++i) {
    dotv(rt, r, KS_RHO);
    scal(1);                                                  // rho == 0
    if (i == 1) {
      cp(r, pv);
      spmv(pv, q);
      dotv(rt, q, KS_SIGMA);
      scal(3);                                                // alpha = rho / (r~, q)
      ax(KS_ALPHA, true, q, r, t);                            // t = r - alpha q
      spmv(t, v);
      ax(KS_ALPHA, false, q, zero, t1);                       // y = alpha q - r
      ax(KS_ONE, true, r, t1, y);
      dotv(v, t, KS_MU2);
      dotv(v, v, KS_MU5);
      scal(5);                                                // zeta, eta = 0
      ax(KS_ZETA, false, q, zero, u);                         // u = zeta q
    } else {
      scal(6);                                                // beta
      ax(KS_BETA, false, q, v, w);                            // w = v + beta q
      ax(KS_ONE, true, u, pv, t1);                            // p = r + beta (p - u)
      ax(KS_BETA, false, t1, r, pv);
      spmv(pv, q);
      dotv(rt, q, KS_SIGMA);
      scal(3);                                                // alpha
      ax(KS_ONE, true, r, t, sv);                             // s = t - r
      ax(KS_ALPHA, true, q, r, t);                            // t = r - alpha q
      spmv(t, v);
      ax(KS_ONE, true, q, w, t1);                             // y = s - alpha (w - q)
      ax(KS_ALPHA, true, t1, sv, y);
      {
        const V xa[ND] = {y, v, y, v, v}, xb[ND] = {y, t, t, y, v};
        const int slot[ND] = {KS_MU1, KS_MU2, KS_MU3, KS_MU4, KS_MU5};
        dot5(xa, xb, slot);
      }
      scal(7);                                                // tau, zeta, eta
      ax(KS_BETA, false, u, sv, t1);                          // u = zeta q + eta (s + beta u)
      ax(KS_ZETA, false, q, zero, t2);
      ax(KS_ETA, false, t1, t2, u);
    }
    ax(KS_ZETA, false, r, zero, t1);                          // z = zeta r + eta z - alpha u
    ax(KS_ETA, false, z, t1, t1);
    ax(KS_ALPHA, true, u, t1, z);
    ax(KS_ALPHA, false, pv, xv, t1);                          // x = x + alpha p + z
    ax(KS_ONE, false, z, t1, xv);
    ax(KS_ETA, true, y, t, t1);                               // r = t - eta y - zeta v
    ax(KS_ZETA, true, v, t1, r);
    dotv(r, r, KS_RR);
    scal(8);                                                  // converged / zeta == 0
    K((int)cudaMemcpyAsync(hfl, fl, sizeof hfl, cudaMemcpyDeviceToHost, st));
    K((int)cudaStreamSynchronize(st));
    if (rc != MPSP_OK) break;
    if (hfl[KF_BREAK]) { *status = MPSP_BICG_BREAKDOWN; break; }
    *iters = i;
    if (hfl[KF_CONV]) { *status = MPSP_BICG_CONVERGED; break; }
    if (hfl[KF_BRK2]) { *status = MPSP_BICG_BREAKDOWN; break; }
  }
  cudaStreamSynchronize(st);
  for (int j = 0; j < ND; ++j) {
    if (dst_[j]) cudaStreamDestroy(dst_[j]);
    if (dev_[j]) cudaEventDestroy(dev_[j]);
  }
  if (dev_[ND]) cudaEventDestroy(dev_[ND]);
  cudaFree(ws);
  return rc;
}

int mpsp_debug_dot_stats(unsigned long long out[2]) {
  if (!out) return MPSP_E_ARG;
  int e = krylov_dot_stats(out);
  if (e) return cuda_fail((cudaError_t)e);
  unsigned long long w[2] = {0ull, 0ull};
  e = krylov_wide_dot_stats(w);
  if (e) return cuda_fail((cudaError_t)e);
  out[0] += w[0];
  out[1] += w[1];
  return MPSP_OK;
}

int mpsp_imad_bench(double out[5]) {
  if (!out) return MPSP_E_ARG;
  int e = run_imad_bench(out);
  if (e != 0) return cuda_fail((cudaError_t)e);
  return MPSP_OK;
}

}  // extern "C"
