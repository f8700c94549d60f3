// Internal interfaces between the rfgpu orchestrator (rfgpu_api.cu) and the
// kernel translation units. Not part of the C ABI (see include/rfgpu.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace rfgpu {

// Count of rfgpu kernel launches issued by this process (every launch site
// bumps it; rfgpu_launch_count reports the delta per context).
int64_t launch_counter();
void count_launch(int n = 1);

// ---- tall-skinny FP64 GEMM (gemm_f64.cu) --------------------------------
struct GemmPlan {
  bool sym;        // Gram-type product: only upper tiles are computed, then mirrored
  int64_t units;   // CTA tiles per split
  int ntiles;      // CTA columns along N
  int nt;          // 8-wide MMA tiles per warp along N (CTA tile N = 16*nt)
  int mtiles;      // CTA rows along M (128 each)
  int splits;      // K splits (1: direct store)
  int64_t ktiles;  // ceil(K / 32)
};

GemmPlan plan_gemm(int64_t M, int64_t N, int64_t K, int num_sms, int force_splits = 0, bool sym = false);
size_t gemm_workspace_bytes(int64_t M, int64_t N, const GemmPlan& p);

// trans_a = false: C = A(MxK) * B(KxN); true: C = A(KxM)^T * B(KxN).
// sumsq_partials (NN only, may be null): receives splits*mtiles partial sums
// of squares of A (each A element counted once).
cudaError_t gemm_f64(bool trans_a, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc, double* workspace,
                     size_t workspace_bytes, double* sumsq_partials, const GemmPlan& p, cudaStream_t st,
                     bool tri_b = false);

cudaError_t sum_array(const double* x, int64_t n, double* out, cudaStream_t st);

// ---- FP64 passes on the INT8 tensor cores (ozaki.cu) -----------------------
// Digit planes of A (m x n, FP64 or FP32) for Y = A X and Z = A^T Q (Ozaki
// scheme, 7 (FP64) / 4 (FP32) balanced 8-bit digits per operand, tcgen05
// kind::i8, FP64 recombination).
struct OzakiA {
  int8_t* rs;   // [digits][n_pad][m_pad] digits of A(i,j) 2^-rowexp[i] (column-major; A X reads them
                // M-major; A^T Q reads them K-major when `shared`)
  int8_t* cs;   // digits of A(i,j) 2^-colexp[j] (A^T Q when !shared; caller-bound): [digits][m_pad][n_pad]
                // (row-major, read M-major) when cs_rowmajor, else [digits][n_pad][m_pad] (read K-major)
  int* rowexp;  // m_pad: |A(i,:)| < 2^rowexp[i]
  int* colexp;  // [nchunks][n_pad]: |A(rows of chunk c, j)| < 2^colexp[c][j]
  int* ext;     // 2 (+pad): max column exponent, -min column exponent (non-zero columns)
  uint32_t* rowhi;    // m_pad row maxima (high words of |A(i,:)|)
  uint32_t* colpart;  // (m_pad / 256) x n_pad per-block column maxima (high words)
  int64_t m, n, m_pad, n_pad;
  int digits;   // 7 (FP64 A) or 4 (FP32 A)
  bool shared;     // one digit set (rs) serves both passes
  bool shared_ok;  // the column scales allow it (ozaki_col_exponents)
  int emax;     // max column exponent (shared mode's thin-operand shift)
  bool cs_rowmajor;
  int64_t chunk_rows, nchunks;  // colexp is [nchunks][n_pad]: column exponents per row chunk (= A^T Q K-split)
};
int64_t ozaki_chunk_rows();  // rows per column-exponent chunk (the A^T Q split; a multiple of 256)
bool ozaki_cs_rowmajor();  // layout of the column-scaled set (RFGPU_OZAKI_TNMN=0: column-major)
bool ozaki_enabled(int64_t m, int64_t n);  // RFGPU_OZAKI=0/1 overrides the size rule
OzakiA ozaki_layout(int64_t m, int64_t n, int digits);  // shapes only (no buffers)
size_t ozaki_set_bytes(int64_t m, int64_t n, int digits);  // one digit set (rs or cs)
size_t ozaki_a_bytes(int64_t m, int64_t n, int digits);    // rs + exponents + maxima (not cs)
void ozaki_bind(void* work, int64_t m, int64_t n, int digits, OzakiA* out);  // carve ozaki_a_bytes
int64_t ozaki_ssq_slots(int64_t rows, int64_t n);  // ||A||_F^2 partials of a row block
// Rows [r0, r1) (r0 a multiple of 256): row exponents, ||A||_F^2 partials
// (ozaki_ssq_slots(r1 - r0, n) of them), column maxima of these rows, and, with
// slice_rows, the row-scaled digits of these rows (all A X needs).
cudaError_t ozaki_prepare_rows(const void* A, bool f32, int64_t lda, int64_t r0, int64_t r1, const OzakiA& a,
                               double* ssq_part, bool slice_rows, cudaStream_t st);
// After every row block's stats: column exponents and whether one shared
// digit set could serve A^T Q too (shared_ok; shared is set only when forced
// by RFGPU_OZAKI_SHARED=1). With decide, synchronises the stream to read the
// exponent range (h_ext: 2 pinned ints); without, only launches the kernel.
cudaError_t ozaki_col_exponents(OzakiA* a, cudaStream_t st, int* h_ext, bool decide = true);
// Column exponents of the chunks completed by rows [r0, r1) and those rows'
// column-scaled digits (streamed upload; r0, r1 chunk-aligned or r1 = m).
cudaError_t ozaki_slice_cols_rows(const void* A, bool f32, int64_t lda, const OzakiA& a, int64_t r0, int64_t r1,
                                  cudaStream_t st);
// One read of A writing the row-scaled (rows) and / or column-scaled (cols) digits.
cudaError_t ozaki_slice_sets(const void* A, bool f32, int64_t lda, const OzakiA& a, bool rows, bool cols,
                             cudaStream_t st);
size_t ozaki_nn_work_bytes(const OzakiA& a, int64_t rows, int64_t ell);
// Y(r0:r1, 0:ell) = A(r0:r1, :) X  (X n x ell, col-major)
cudaError_t ozaki_nn(const OzakiA& a, int64_t r0, int64_t r1, const double* X, int64_t ldx, int64_t ell, double* Y,
                     int64_t ldy, void* work, cudaStream_t st);
size_t ozaki_tn_work_bytes(const OzakiA& a, int64_t ell);
// Z (n x ell) = A^T Q  (Q m x ell, col-major); presliced: Q's digits are already in work (ozaki_slice_thin)
cudaError_t ozaki_tn(const OzakiA& a, const double* Q, int64_t ldq, int64_t ell, double* Z, int64_t ldz, void* work,
                     cudaStream_t st, bool presliced = false);
// Gram of a tall R (a.m x ell) on the digit path: slice R into work (the
// layout ozaki_tn reads), then G = R^T R (ell x ell).
cudaError_t ozaki_slice_thin(const OzakiA& a, const double* R, int64_t ldr, int64_t ell, void* work, cudaStream_t st);
cudaError_t ozaki_gram_thin(const OzakiA& a, int64_t ell, void* work, double* G, int64_t ldg, cudaStream_t st);
// ---- small dense kernels (small_f64.cu) ----------------------------------
// Upper Cholesky R^T R = G (G c x c, symmetric, upper triangle consulted,
// ld = c) and R^{-1}, both c x c column-major with zeros below the diagonal.
// info[0] = 0 ok, else 1 + the failing column (reference rule: pivot <=
// 1e-14 * max initial diagonal, proj/src/dense.cpp:763-786);
// info_d[0] = min_j pivot_j / trace(G) (the CholeskyQR fast-path gate).
cudaError_t chol_inv(const double* G, int64_t c, double* R, double* Rinv, double* work, int* info,
                     double* info_d, cudaStream_t st);
size_t chol_inv_work_bytes(int64_t c);

// One-sided Jacobi SVD of X (mr x c, ld = mr): X = U diag(S) V^T with S
// sorted non-increasing (proj/src/dense.cpp:585-686 semantics: tolerance
// 1e-15, <= 60 sweeps, columns with S <= smax*1e-250 zeroed). U mr x c,
// V c x c. info[0] = 0 ok, 1 no convergence, 2 zero singular values present
// (those U columns are left zero; the caller completes them).
// sorted = true forces the per-column kernel, which re-orders the columns by
// norm before every sweep exactly as the reference does (dense.cpp:597-618):
// required for graded / ill-conditioned X (a spectrum spanning many decades),
// where unsorted cyclic sweeps can exceed the sweep cap; the block kernel
// (cluster-wide, no per-sweep ordering) serves the well-conditioned l x l
// factors of CholeskyQR2.
cudaError_t jacobi_svd(const double* X, int64_t mr, int64_t c, double* U, double* S, double* V, double* work,
                       int* info, int* sweeps_out, cudaStream_t st, bool sorted = false);
size_t jacobi_work_bytes(int64_t mr, int64_t c);
// Two independent same-shape problems in one launch (one cluster each).
struct JacobiProblem {
  const double* X;
  double* U;
  double* S;
  double* V;
  double* work;  // jacobi_work_bytes(mr, c)
  int* info;
  int* sweeps;
};
cudaError_t jacobi_svd_pair(const JacobiProblem& a, const JacobiProblem& b, int64_t mr, int64_t c, cudaStream_t st);

// y = sum of squares of x[0..n) into *out (fixed-order two-level reduction).
cudaError_t sumsq(const double* x, int64_t n, double* partials, double* out, cudaStream_t st);

// ---- Gram-Schmidt fallback for rank-deficient orth (orth_f64.cu) ---------
// Reference orth semantics (proj/src/dense.cpp:402-431): classical
// Gram-Schmidt applied twice per column, dropping columns whose residual is
// <= drop. Q receives kept columns (ld = m); *r_dev the kept count.
// Optional in-place sum across ranks of a device buffer (NCCL in the
// distributed context; fn == nullptr on one GPU).
struct DeviceAllreduce {
  void* ctx;
  cudaError_t (*fn)(void* ctx, double* buf, int64_t count, cudaStream_t st);
};

size_t gs_orth_work_doubles(int64_t m, int64_t c);
cudaError_t gs_orth(const double* X, int64_t m, int64_t c, int64_t ldx, double* Q, int64_t ldq, int64_t* r_dev,
                    double* work, const DeviceAllreduce& ar, cudaStream_t st);

// ---- column-pivoted QR / interpolative decomposition (cpqr.cu) -----------
// In place on W (m x n, ld, m <= 512): cpqr with CpqrStop::rank(kmax) and the
// reference pivot / recompute / halt rules; perm (n) device, *stopped (device)
// = stopped rank, *recomputes (device) counts exact norm recomputes.
size_t cpqr_work_bytes(int64_t n, int grid, int m);
cudaError_t cpqr_rank(double* W, int64_t ld, int m, int64_t n, int kmax, double halt, int64_t* perm, void* work,
                      int* stopped, int* recomputes, int num_sms, cudaStream_t st);
cudaError_t trinv_upper(const double* R, int64_t ldr, int k, double* Rinv, cudaStream_t st);
cudaError_t assemble_z(const int64_t* perm, int ke, int64_t n, const double* T, double* Z, cudaStream_t st);

// Stream-ordered device allocation from the calling context's memory pools
// (installed for the duration of every C-ABI call: temporaries under 256 MiB
// from a small-block pool, larger ones from a large-block pool, so small
// temporaries never carve up the blocks the digit planes reuse call after
// call); the device's default pool outside a call.
cudaError_t ws_alloc(void** p, size_t bytes, cudaStream_t st);

// *dst += *src (one thread; keeps scalar bookkeeping on the device).
cudaError_t add_scalar(double* dst, const double* src, cudaStream_t st);

// Copy into a buffer that is next read by a DMA engine only (non-temporal stores when the CPU has AVX2).
void host_stream_copy(void* dst, const void* src, size_t bytes);
}  // namespace rfgpu
