// layout.h - device layout of one row block of A (or A^T), shared by the
// host builder and the kernels.
//
// Rows are sorted by length (descending, stable).  The rows longer than the
// long-row threshold come first as WARP ROWS (one warp per row, spmv_wrow):
// warp row i owns entries [wrow_ptr[i], wrow_ptr[i] + len rounded up to 32),
// entry j of the row at E = wrow_ptr[i] + j, i.e. group g = E/32 and lane
// l = j % 32 in the limb formula below, so a warp's 32 consecutive entries
// load as coalesced 512 B chunks.  The remaining rows are cut into SELL
// slices of 32 rows; slice s holds w_s = (longest row in the slice) positions.  Entry
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
  int64_t nslots;             // 32 * nslices (SELL part: short rows)
  int64_t nslices;
  // launch order of the slices (widest first across the row chunks), or
  // null: the stored order (one chunk, or a chunk view of the host pipeline)
  const int32_t* slice_order;
  // warp rows (rows longer than the long-row threshold), longest first
  int64_t nwrow;
  const int64_t* wrow_ptr;    // [nwrow] first entry (multiple of 32)
  const int32_t* wrow_row;    // [nwrow] output row (local)
  const int32_t* wrow_len;    // [nwrow]
};

struct XView {
  const uint32_t* limbs;      // [n * L] element-major
  const int32_t* exps;        // [n]
  const uint8_t* signs;       // [n]
};

struct VecIn {                // a read-only MP vector (ABI format)
  const uint32_t* limbs;
  const int32_t* exps;
  const uint8_t* signs;
};

struct YView {
  uint32_t* limbs;            // [rows * L]
  int32_t* exps;
  uint8_t* signs;
};

// Launch the SpMV over one part on `stream`; returns a cudaError_t value.
int launch_spmv(int L, const PartView& P, const XView& x, const YView& y, void* stream);
// p > 1024 (L = 64, 128, 256): one warp per row over all P.nwrow rows
// (entry-major limbs), MP arithmetic spread across the lanes (spmv_wide.cu).
// dense = true: mpsp_dense_create's rows (column of entry j = j, no col reads).
int launch_spmv_wide(int L, const PartView& P, const XView& x, const YView& y, void* stream,
                     bool dense = false);
// Warp-row kernel over the P.nwrow long rows; returns a cudaError_t value.
int launch_spmv_long(int L, const PartView& P, const XView& x, const YView& y, void* stream,
                     bool dense = false);
// Row-length threshold above which a row goes to the warp-row kernel.
int long_row_threshold();
// Launch counter increment (shared by the kernel files).
void launch_counter_add(int64_t k);
// BiCG building blocks (krylov.cu); each returns a cudaError_t value.
// Scalars / flags: the BiCG state arrays of mpsp_api.cpp (enum in krylov.cu).
int krylov_dot(int L, int64_t n, const VecIn& u, const VecIn& v, const YView& out, const int* stop,
               void* stream, void* work);   // work: krylov_dot_work_bytes, or null (one warp)
size_t krylov_dot_work_bytes(int L, int64_t n);
int krylov_dot_stats(unsigned long long out[2]);   // [sequential, validated] segments, reset
int krylov_wide_dot_stats(unsigned long long out[2]);   // the same for p > 1024
// exclusive fp64 prefix of per-segment sums, in place (one 1024-thread block)
int launch_dot_prefix(double* segsum, int64_t nseg, const int* stop, void* stream);
int krylov_axpy(int L, int64_t n, const VecIn& al, int neg, const VecIn& x, const VecIn& y,
                const YView& z, const int* stop, void* stream);
int krylov_scalar(int L, const YView& S, int* fl, int op, void* stream);
// the same at L = 64, 128, 256 (krylov_wide.cu; the dot always needs `work`)
int krylov_wide_dot(int L, int64_t n, const VecIn& u, const VecIn& v, const YView& out,
                    const int* stop, void* stream, void* work);
size_t krylov_wide_dot_work_bytes(int L, int64_t n);
int krylov_wide_axpy(int L, int64_t n, const VecIn& al, int neg, const VecIn& x, const VecIn& y,
                     const YView& z, const int* stop, void* stream);
int krylov_wide_scalar(int L, const YView& S, int* fl, int op, void* stream);
enum { KS_RHO, KS_RHOP, KS_SIGMA, KS_ALPHA, KS_BETA, KS_RR, KS_NRM, KS_THR, KS_C1, KS_C2, KS_ONE,
       KS_T20, KS_T50, KS_ALPHAP, KS_ZETA, KS_ETA, KS_MU1, KS_MU2, KS_MU3, KS_MU4, KS_MU5, KS_TAU,
       KS_N };
// KF_BRK2: breakdown detected after the iteration's update (GPBiCG zeta = 0)
enum { KF_STOP, KF_BREAK, KF_CONV, KF_BRK2, KF_N };
// x exchange records (xchg.cu): pack count elements into (L+1)-word records
// (L limbs + expw) or unpack records into an ABI vector; cudaError_t value.
int launch_vec_pack(int L, bool unpack, int64_t count, const uint32_t* limbs_in,
                    const int32_t* exps_in, const uint8_t* signs_in, const uint32_t* rec_in,
                    uint32_t* rec_out, uint32_t* limbs_out, int32_t* exps_out, uint8_t* signs_out,
                    void* stream);
// Integer-MAC microbenchmark (roofline denominator); returns cudaError_t.
int run_imad_bench(double out[5]);
// Launches this process has made.
int64_t launch_counter_get();

}  // namespace mpsp
