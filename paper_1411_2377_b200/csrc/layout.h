// layout.h - device layout of one row block of A (or A^T), shared by the
// host builder and the kernels.
//
// Rows are sorted by length (descending, stable) and cut into SELL slices of
// 32 rows; slice s holds w_s = (longest row in the slice) positions.  Entry
// (slice s, position j, lane l) has entry index E = slice_ptr[s] + 32*j + l,
// i.e. it lives in "group" g = E/32 = slice_ptr[s]/32 + j.
//   col[E], expw[E]   : int32 column index and packed exponent word
//                       expw = (sign << 31) | (exp & 0x7fffffff)
//   limbs             : group-major, then chunk-major, then lane:
//                       word (g, c, l, w) at ((g*NC + c)*32 + l)*CW + w,
//                       limb number c*CW + w, CW = min(L,4), NC = L/CW.
//                       A warp loading chunk c of one position reads
//                       32*CW*4 contiguous bytes (512 B at L >= 4).
//   slot_row[slot], slot_len[slot] : output row (local, -1 = padding) and
//                       length of the row held by slot = 32*s + l.
// Zero entries of A are stored with all limbs 0 (their product is zero).
#pragma once
#include <cstdint>

namespace mpsp {

struct PartView {
  const int64_t* slice_ptr;   // [nslices+1] entry offsets (multiples of 32)
  const int32_t* slot_row;    // [nslots]
  const int32_t* slot_len;    // [nslots]
  const int32_t* col;         // [nentries]
  const int32_t* expw;        // [nentries]
  const uint32_t* limbs;      // [nentries * L]
  int64_t nslots;             // 32 * nslices
  int64_t nslices;
  int64_t nlong;              // slices [0, nlong) hold rows longer than the
                              // long-row threshold (spmv_long); the rest
                              // go to spmv_sell
};

struct XView {
  const uint32_t* limbs;      // [n * L] element-major
  const int32_t* exps;        // [n]
  const uint8_t* signs;       // [n]
};

struct YView {
  uint32_t* limbs;            // [rows * L]
  int32_t* exps;
  uint8_t* signs;
};

// Launch the SpMV over one part on `stream`; returns a cudaError_t value.
int launch_spmv(int L, const PartView& P, const XView& x, const YView& y, void* stream);
// Long-row kernel over slices [0, P.nlong); returns a cudaError_t value.
int launch_spmv_long(int L, const PartView& P, const XView& x, const YView& y, void* stream);
// Row-length threshold above which a slice goes to the long-row kernel.
int long_row_threshold();
// Launch counter increment (shared by the kernel files).
void launch_counter_add(int64_t k);
// Integer-MAC microbenchmark (roofline denominator); returns cudaError_t.
int run_imad_bench(double out[3]);
// Launches this process has made.
int64_t launch_counter_get();

}  // namespace mpsp
