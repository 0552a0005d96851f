/*
 * mpsp.h - C ABI of libmpsp: multiple-precision CSR sparse matrix-vector
 * multiplication on NVIDIA B200 (sm_100a).
 *
 * Operation (arXiv 1411.2377, PAPER.md:119-133 CSR storage of the nonzero
 * elements; PAPER.md:182-186 the product A^(s,p) b; PAPER.md:282-284 (Fig. 4,
 * BiCG) z = A p and z~ = A^T p~; BASELINE.json north_star for the rounding
 * and order):
 *
 *     y_i = chain_i(A, x):  s = +0;  for k = rowptr[i] .. rowptr[i+1]-1
 *                                     (ascending column index):
 *                                 s = RN_p( s + RN_p( A_k * x[colidx[k]] ) )
 *
 * RN_p = round to nearest, ties to even, to p significant bits, after every
 * multiply and every add (PAPER.md:84-85 lists RN among MPFR's modes; reading
 * c1 in DESIGN.md).  A^T x uses the same chain over column j of A in
 * ascending row index of A.  Results are bit-exact: every limb, exponent and
 * sign is a pure function of (A, x), independent of launch configuration,
 * binning and GPU count.
 *
 * VALUE ENCODING (packed host/device format):
 *   A nonzero value is (-1)^sign * (M / 2^p) * 2^exp with 2^(p-1) <= M < 2^p
 *   (MPFR convention).  M is stored as L = p/32 uint32 limbs, limb 0 least
 *   significant, so the MSB of limb L-1 is set.  exp is int32, sign is uint8
 *   in {0,1}.  Zero is "all limbs 0" (its exp and sign are ignored on input;
 *   written as exp 0, sign 0 on output; no -0 is ever produced).  There is no
 *   NaN/Inf/subnormal.  Input exponents must satisfy |exp| <= 2^29, which
 *   makes int32 overflow impossible inside the chain.
 *
 * Element layouts: limbs arrays are element-major ("AoS"): element i's limbs
 * are limbs[i*L .. i*L+L-1].  exps/signs are one entry per element.
 *
 * THREAD SAFETY: one handle per host thread at a time; distinct handles are
 * independent.  All functions return MPSP_OK (0) or a negative error code.
 */
#ifndef MPSP_H
#define MPSP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ------------------------------------------------------ */
#define MPSP_OK            0
#define MPSP_E_ARG        -1   /* null pointer, n < 0, bad row range, misaligned */
#define MPSP_E_PREC       -2   /* p % 32 != 0 or p outside the supported set */
#define MPSP_E_CSR        -3   /* rowptr[0]!=0, non-monotone, rowptr[n] > 2^31-1,
                                  colidx outside [0, n) */
#define MPSP_E_UNSORTED   -4   /* colidx not strictly increasing within a row
                                  (covers duplicates); the library does not sort */
#define MPSP_E_VALUE      -5   /* nonzero value without MSB of limb L-1 set,
                                  or |exp| > 2^29 */
#define MPSP_E_NOMEM      -6   /* host or device allocation failed */
#define MPSP_E_CUDA       -7   /* CUDA runtime error (see mpsp_strerror / mpsp_last_cuda_error) */
#define MPSP_E_ALIAS      -8   /* x and y storage overlap */
#define MPSP_E_DEVICE     -9   /* current device (or a pointer's device) differs from the handle's */
#define MPSP_E_NOTRANS   -10   /* spmv_t on a handle built without MPSP_WITH_TRANSPOSE */

/* ---- flags for mpsp_csr_create ---------------------------------------- */
#define MPSP_WITH_TRANSPOSE  0x1u  /* also build rows [row_begin,row_end) of A^T */

typedef struct mpsp_csr mpsp_csr;

/*
 * mpsp_csr_create - validate a CSR matrix and build its device form.
 *
 *   out        receives the handle (NULL on error; nothing leaks on error).
 *   p_bits     precision p in bits; supported: 32, 64, 128, 256, 512, 1024
 *              (L = p/32 in {1,2,4,8,16,32}) and the paper's solver
 *              precisions 2048, 4096, 8192 (L = 64, 128, 256;
 *              one warp per row with the limbs
 *              spread across the lanes).
 *   n          A is n x n (n >= 0).
 *   rowptr     host int64[n+1]: CSR row pointers (rowptr[0] = 0, monotone).
 *   colidx     host int32[nnz], nnz = rowptr[n] <= 2^31-1; strictly
 *              increasing within each row, values in [0, n).
 *   limbs      host uint32[nnz*L] element-major mantissas (see encoding).
 *   exps       host int32[nnz]; signs host uint8[nnz].
 *   row_begin, row_end
 *              the handle computes rows [row_begin, row_end) of y (and, with
 *              MPSP_WITH_TRANSPOSE, of A^T x).  0 <= row_begin <= row_end <= n.
 *              Single GPU: 0, n.  Row-block multi-GPU: one block per rank.
 *   flags      MPSP_WITH_TRANSPOSE or 0.
 *
 * The full global CSR is passed in host memory; the handle copies what it
 * needs (the caller may free or modify the inputs on return) and owns all
 * device memory, allocated on the CURRENT CUDA device.  Explicit zero entries
 * are kept (they contribute +0).  One-off cost: O(nnz*L) host work plus one
 * host-to-device copy; it synchronises the device before returning.
 *
 * Errors: MPSP_E_ARG, MPSP_E_PREC, MPSP_E_CSR, MPSP_E_UNSORTED, MPSP_E_VALUE,
 * MPSP_E_NOMEM, MPSP_E_CUDA.
 */
int mpsp_csr_create(mpsp_csr **out, int p_bits, int64_t n,
                    const int64_t *rowptr, const int32_t *colidx,
                    const uint32_t *limbs, const int32_t *exps, const uint8_t *signs,
                    int64_t row_begin, int64_t row_end, uint32_t flags);

/*
 * mpsp_dense_create - a handle for a DENSE n x n matrix: the dense MP matrix-
 * vector product of the paper's section 3 (the Lotkin
 * dense-vs-sparse comparison).
 *
 *   limbs      host uint32[n*n*L] row-major (entry (i, j) at i*n + j), the
 *              element encoding above; zeros are all-zero limbs.
 *   exps, signs host int32[n*n], uint8[n*n].
 *   p_bits, row_begin, row_end, flags: as for mpsp_csr_create (n <= 46340,
 *              so n^2 <= 2^31 - 1).
 * mpsp_spmv / mpsp_spmv_t on the handle compute y_i = the ordered chain over
 * ALL n columns j (zeros included; their products are +0 and leave s
 * unchanged, so the result equals mpsp_spmv on the CSR of the nonzeros bit
 * for bit).  The kernel reads no column indices (column = position).
 * Errors: MPSP_E_ARG, MPSP_E_PREC, MPSP_E_CSR (n too large), MPSP_E_VALUE,
 * MPSP_E_NOMEM, MPSP_E_CUDA.  Release with mpsp_destroy.
 */
int mpsp_dense_create(mpsp_csr **out, int p_bits, int64_t n,
                      const uint32_t *limbs, const int32_t *exps, const uint8_t *signs,
                      int64_t row_begin, int64_t row_end, uint32_t flags);

/*
 * mpsp_spmv - y[i - row_begin] = chain_i(A, x) for i in [row_begin, row_end).
 *
 * All pointers are DEVICE pointers on the handle's device:
 *   x_limbs uint32[n*L], x_exps int32[n], x_signs uint8[n]   (the full x)
 *   y_limbs uint32[r*L], y_exps int32[r], y_signs uint8[r]   (r = row_end-row_begin)
 * limbs pointers must be aligned to min(16, 4L) bytes.  x and y must not
 * overlap.  Pointers to empty arrays (n = 0, or an empty row range) may be
 * NULL.  The work is enqueued on `cuda_stream` (a cudaStream_t; NULL =
 * legacy default stream) and the call returns without synchronising; x and y
 * are caller-owned and must stay alive until the stream work completes.
 * x contents are not validated (an unnormalised nonzero x is undefined
 * behaviour) unless the environment variable MPSP_VALIDATE=1 is set.
 * The pointer checks (device memory on the handle's device) are skipped when
 * the six x/y pointers equal those of the handle's last call that passed
 * them; a caller that frees buffers and passes a new allocation at the same
 * address without it being device memory of that device must set
 * MPSP_PTR_CACHE=0 (check every call).
 *
 * Errors: MPSP_E_ARG, MPSP_E_ALIAS, MPSP_E_DEVICE, MPSP_E_VALUE (validation
 * mode only), MPSP_E_CUDA (launch failure).
 */
int mpsp_spmv(const mpsp_csr *A,
              const uint32_t *x_limbs, const int32_t *x_exps, const uint8_t *x_signs,
              uint32_t *y_limbs, int32_t *y_exps, uint8_t *y_signs, void *cuda_stream);

/*
 * mpsp_spmv_t - y[j - row_begin] = chainT_j(A, x): over i ascending with
 * (i, j) stored, s = RN(s + RN(A_ij * x_i)), for j in [row_begin, row_end).
 * Same arguments and errors as mpsp_spmv, plus MPSP_E_NOTRANS.
 */
int mpsp_spmv_t(const mpsp_csr *A,
                const uint32_t *x_limbs, const int32_t *x_exps, const uint8_t *x_signs,
                uint32_t *y_limbs, int32_t *y_exps, uint8_t *y_signs, void *cuda_stream);

/*
 * mpsp_spmv_host / mpsp_spmv_t_host - the same operations on HOST buffers
 * (pageable or pinned).  Copies x to a device workspace owned by the handle,
 * runs the kernel on the handle's internal stream, copies y back and
 * synchronises before returning.  Same errors as the device variants
 * (MPSP_E_ALIAS is checked on the host ranges).
 */
int mpsp_spmv_host(mpsp_csr *A,
                   const uint32_t *x_limbs, const int32_t *x_exps, const uint8_t *x_signs,
                   uint32_t *y_limbs, int32_t *y_exps, uint8_t *y_signs);
int mpsp_spmv_t_host(mpsp_csr *A,
                     const uint32_t *x_limbs, const int32_t *x_exps, const uint8_t *x_signs,
                     uint32_t *y_limbs, int32_t *y_exps, uint8_t *y_signs);

/* mpsp_destroy - synchronise the handle's device and free everything. NULL-safe. */
void mpsp_destroy(mpsp_csr *A);

/* mpsp_strerror - static, library-owned description of an error code. */
const char *mpsp_strerror(int code);

/* Text of the last CUDA error seen by this thread (static storage). */
const char *mpsp_last_cuda_error(void);

/*
 * mpsp_csr_info - sizes of a handle, for bindings and reporting.
 *   info[0] = p_bits, info[1] = n, info[2] = row_begin, info[3] = row_end,
 *   info[4] = nnz of the row block of A, info[5] = nnz of the row block of A^T
 *   (-1 without transpose), info[6] = device bytes owned by the handle,
 *   info[7] = device ordinal, info[8] = stored slots of A incl. padding,
 *   info[9] = max row length in the block of A.
 * Errors: MPSP_E_ARG.
 */
int mpsp_csr_info(const mpsp_csr *A, int64_t info[10]);

/* ---- x exchange records (multi-GPU) ---------
 * Before each multi-GPU application x must be replicated wherever a rank's
 * rows read it (BASELINE.json north_star (4): NCCL over NVLink).  To move
 * each element as ONE record - one NCCL call per peer, or one all-gather,
 * instead of three - an element is packed into L + 1 uint32 words: its L limbs
 * then expw = (sign << 31) | (exp & 0x7fffffff).  Bit-exact for every valid
 * value (|exp| <= 2^29).  All pointers are DEVICE pointers; asynchronous on
 * cuda_stream.
 *
 * mpsp_vec_pack   - rec[i*(L+1) ..] <- element i of (limbs, exps, signs),
 *                   i in [0, count).
 * mpsp_vec_unpack - element i of (limbs, exps, signs) <- rec[i*(L+1) ..].
 * Errors: MPSP_E_PREC (p not supported), MPSP_E_ARG (count < 0, null
 * pointer), MPSP_E_ALIAS (record and vector storage overlap), MPSP_E_CUDA. */
int mpsp_vec_pack(int p_bits, int64_t count, const uint32_t *limbs, const int32_t *exps,
                  const uint8_t *signs, uint32_t *rec, void *cuda_stream);
int mpsp_vec_unpack(int p_bits, int64_t count, const uint32_t *rec, uint32_t *limbs,
                    int32_t *exps, uint8_t *signs, void *cuda_stream);

/*
 * mpsp_debug_host_build - the host half of mpsp_csr_create without a GPU:
 * the same validation (same error codes), transpose, row binning, row chunks
 * and repack, then a checksum of the device arrays instead of the upload.
 * For host-side tests (address / undefined-behaviour sanitizers, SURVEY.md
 * 4 T6).  out[0..5] = part A: nnz, stored entries incl. padding, warp rows,
 * SELL slices, row chunks, checksum; out[6..11] = the same for A^T (zeros
 * without MPSP_WITH_TRANSPOSE).  Errors: those of mpsp_csr_create except
 * MPSP_E_CUDA; MPSP_E_ARG for out == NULL.
 */
int mpsp_debug_host_build(int p_bits, int64_t n, const int64_t *rowptr, const int32_t *colidx,
                          const uint32_t *limbs, const int32_t *exps, const uint8_t *signs,
                          int64_t row_begin, int64_t row_end, uint32_t flags, int64_t out[12]);

/* Number of kernels this library has launched in this process (monotone). */
int64_t mpsp_launch_count(void);

/* ---- BiCG ------------------------------------------
 * PAPER.md:249-297 (Fig. 4, BiCG; no preconditioner, K = I) from x_0 = 0, and
 * PAPER.md:375-380 (stop when ||r_i||_2 <= 1e-20 ||r_0||_2 + 1e-50).  Every
 * operation is one p-bit round-to-nearest-even operation in the order Fig. 4
 * writes it (readings c26-c31): a dot product is the ordered chain
 * s = RN(s + RN(u_k v_k)), k ascending, from +0; "a + beta b" is
 * RN(a + RN(beta b)); ||v|| = RN(sqrt((v, v))); the constants are RN(10^-20)
 * and RN(10^-50).  All vectors are DEVICE pointers in the element layout
 * above; scalars are 1-element vectors.  Asynchronous on cuda_stream except
 * mpsp_bicg, which synchronises once per iteration (3-int flag read).
 */
#define MPSP_BICG_CONVERGED  0
#define MPSP_BICG_BREAKDOWN  1   /* rho = 0 or (p~, z) = 0 */
#define MPSP_BICG_MAXITER    2

/* The vector and solver calls below support every precision mpsp_csr_create
 * does (mpsp_bicg / mpsp_gpbicg: p >= 128); at p > 1024 they run on
 * warp-distributed values (krylov_wide.cu); other p -> MPSP_E_PREC. */

/* out = (u, v): ordered rounded chain over k = 0..n-1 (one element, device). */
int mpsp_dot(int p_bits, int64_t n,
             const uint32_t *u_limbs, const int32_t *u_exps, const uint8_t *u_signs,
             const uint32_t *v_limbs, const int32_t *v_exps, const uint8_t *v_signs,
             uint32_t *out_limbs, int32_t *out_exps, uint8_t *out_signs, void *cuda_stream);

/* z_k = RN(y_k + RN(+-alpha x_k)), k = 0..n-1 (negate != 0: minus).  alpha is
 * a 1-element device vector; z may alias y (element-wise in place). */
int mpsp_axpy(int p_bits, int64_t n,
              const uint32_t *a_limbs, const int32_t *a_exps, const uint8_t *a_signs, int negate,
              const uint32_t *x_limbs, const int32_t *x_exps, const uint8_t *x_signs,
              const uint32_t *y_limbs, const int32_t *y_exps, const uint8_t *y_signs,
              uint32_t *z_limbs, int32_t *z_exps, uint8_t *z_signs, void *cuda_stream);

/* Solve A x = b by BiCG.  A: a handle over ALL rows built with
 * MPSP_WITH_TRANSPOSE, p >= 128 (else MPSP_E_NOTRANS / MPSP_E_ARG /
 * MPSP_E_PREC).  b, x: device n-vectors (x is overwritten; on breakdown it
 * holds the last complete iterate).  *iters = completed iterations, *status =
 * MPSP_BICG_*.  Workspace: 6 n-vectors, allocated and freed per call. */
int mpsp_bicg(mpsp_csr *A,
              const uint32_t *b_limbs, const int32_t *b_exps, const uint8_t *b_signs,
              uint32_t *x_limbs, int32_t *x_exps, uint8_t *x_signs,
              int max_iter, int *iters, int *status, void *cuda_stream);

/* Solve A x = b by GPBiCG (Fig. 4 right; K = I; readings
 * c32-c35 in DESIGN.md: left-to-right RN evaluation of every compound
 * update, the figure's "zeta z" / "zeta u" read as eta z / zeta v).
 * Transpose-free: A needs no MPSP_WITH_TRANSPOSE.  Same arguments, status
 * and errors as mpsp_bicg (breakdown also on tau = 0 or zeta = 0).
 * Workspace: 14 n-vectors, allocated and freed per call. */
int mpsp_gpbicg(mpsp_csr *A,
                const uint32_t *b_limbs, const int32_t *b_exps, const uint8_t *b_signs,
                uint32_t *x_limbs, int32_t *x_exps, uint8_t *x_signs,
                int max_iter, int *iters, int *status, void *cuda_stream);

/* Diagnostics of the segmented dot: out[0] = segments the
 * chain warp evaluated step by step, out[1] = segments committed from their
 * speculative sums, since the last call (counters are then reset); the
 * p <= 1024 and p > 1024 chains' counts are summed. */
int mpsp_debug_dot_stats(unsigned long long out[2]);

/*
 * mpsp_imad_bench - measures the sustained 32x32->64 limb-MAC rate of the
 * current device, all SMs busy, per-lane operands, in two instruction forms:
 * the Comba (product-scanning) pattern the SpMV kernels use (IMAD.WIDE.U32
 * with carry-out) and operand scanning (IMAD + IMAD.HI with carry chains).
 *   out[0] = limb-MACs per second of the faster form (the peak),
 *   out[1] = its kernel seconds, out[2] = SM count,
 *   out[3] = Comba limb-MACs per second, out[4] = operand-scanning rate.
 * out[0] is the roofline denominator for the integer-bound configurations.
 * Errors: MPSP_E_ARG (out NULL), MPSP_E_CUDA.
 */
int mpsp_imad_bench(double out[5]);

/* Supported precisions query: returns 1 if p_bits is supported, else 0. */
int mpsp_supported_precision(int p_bits);

#ifdef __cplusplus
}
#endif

#endif /* MPSP_H */
