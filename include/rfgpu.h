/*
 * rfgpu — C ABI of the B200-native randomized range finder.
 *
 * This is the drop-in boundary for the reference's hot path (namespace
 * randfact in /root/reference/proj/include/randfact/): every entry point below
 * names the reference interface it replaces. Plain pointers and sizes only;
 * matrices are column-major (the reference DenseMatrix layout,
 * proj/include/randfact/dense.hpp:12-24); indices are int64 (randfact::idx,
 * proj/include/randfact/common.hpp:9). Host buffers are caller-owned.
 *
 * Status codes mirror the reference exception tree
 * (proj/include/randfact/common.hpp:11-44) and the CLI exit families
 * (proj/src/cli.cpp:459-471):
 *   RFGPU_OK 0, RFGPU_EPARAM 3 (ParameterError), RFGPU_ENUMERICAL 4
 *   (NumericalError), RFGPU_ECONVERGENCE 5 (ConvergenceError), RFGPU_ENOTPD 6
 *   (NotPositiveDefiniteError), RFGPU_ECUDA 7 (device / NCCL failure),
 *   RFGPU_ESTREAM 8 (StreamContractError), RFGPU_ENOMEM 9.
 * rfgpu_last_error() returns the message of the last failure on the calling
 * thread.
 *
 * Randomness: every algorithm takes the sketch G as an input, bit-identical
 * to the reference generator (rfgpu_gaussian reproduces
 * randfact::gaussian(seed, tag, m, n), proj/src/sketch.cpp:56-62).
 *
 * Multi-GPU: a context created with rfgpu_ctx_create_dist() owns an NCCL
 * communicator; matrices uploaded to it are the caller's ROW SHARD of A.
 * Row-local outputs (Q, U, the tall sketch Y) are returned for the local rows
 * only; replicated outputs (B, V, D, residual) are identical on every rank.
 *
 * One context is not re-entrant: calls on the same context must be
 * serialised by the caller (the C++ drop-in does this with a mutex).
 */
#ifndef RFGPU_H
#define RFGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RFGPU_OK 0
#define RFGPU_EPARAM 3
#define RFGPU_ENUMERICAL 4
#define RFGPU_ECONVERGENCE 5
#define RFGPU_ENOTPD 6
#define RFGPU_ECUDA 7
#define RFGPU_ESTREAM 8
#define RFGPU_ENOMEM 9

typedef struct rfgpu_ctx rfgpu_ctx;
typedef struct rfgpu_matrix rfgpu_matrix;

const char* rfgpu_last_error(void);
int rfgpu_version(void);

/* ---- generator (host) ---------------------------------------------------
 * randfact::gaussian (proj/src/sketch.cpp:56-62, proj/src/rng.cpp:12-56):
 * counter SplitMix64 keyed by mix(seed ^ fnv1a64(tag)), Box-Muller with the
 * sin variate cached. Writes the m x n column-major matrix; multithreaded
 * (element-seekable), bitwise identical to the reference on the same libm. */
int rfgpu_gaussian(uint64_t seed, const char* tag, int64_t m, int64_t n, double* out);
/* Elements [e0, e0+count) of the same column-major stream. */
int rfgpu_gaussian_range(uint64_t seed, const char* tag, int64_t e0, int64_t count, double* out);

/* ---- contexts ------------------------------------------------------------ */
int rfgpu_ctx_create(int device, rfgpu_ctx** out);
/* NCCL unique id for rfgpu_ctx_create_dist (rank 0 creates, all ranks pass
 * the same bytes). id must hold 128 bytes. */
int rfgpu_nccl_unique_id(void* id, size_t id_bytes);
int rfgpu_ctx_create_dist(int device, int rank, int world, const void* nccl_id, size_t id_bytes,
                          rfgpu_ctx** out);
/* One-GPU check of the NCCL transport behind rfgpu_ctx_create_dist (same bindings): a one-rank communicator
 * from a fresh id, ncclAllReduce (sum, double) of `count` values in place on the device, the result back in
 * out[0..count) (one rank: equal to the input). No reference counterpart. */
int rfgpu_nccl_selftest(int device, const double* values, int64_t count, double* out);
/* Host-staged reduction backend: the sums over ranks (the same points where
 * the NCCL context allreduces) go through sum(user, buf, count), which must
 * replace buf[0..count) (pinned host memory) by its elementwise sum over all
 * ranks and return 0 (non-zero fails the call with RFGPU_ECUDA). For hosts
 * without NCCL and for several ranks sharing one GPU (NCCL cannot place two
 * ranks on one device): the test suite runs the row-sharded schedule this way
 * with a torch.distributed gloo callback. No reference counterpart (the
 * reference is single-process). */
typedef int (*rfgpu_host_sum_fn)(void* user, double* buf, int64_t count);
int rfgpu_ctx_create_hostsum(int device, int rank, int world, rfgpu_host_sum_fn sum, void* user, rfgpu_ctx** out);
int rfgpu_ctx_destroy(rfgpu_ctx* ctx);
/* Returns every cached device block of the context to the driver: the
 * stream-ordered pools (trimmed to zero) and the host-call A buffer. The next
 * call re-allocates. */
int rfgpu_ctx_release_memory(rfgpu_ctx* ctx);
/* Device bytes the context currently holds (pool reservations + A cache). */
int64_t rfgpu_ctx_pool_bytes(rfgpu_ctx* ctx);
int rfgpu_ctx_rank(const rfgpu_ctx* ctx);
int rfgpu_ctx_world(const rfgpu_ctx* ctx);
/* Blocks until all work issued on the context's stream is done. */
int rfgpu_ctx_synchronize(rfgpu_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) for callers that time on it. */
void* rfgpu_ctx_stream(rfgpu_ctx* ctx);

/* Per-kernel CUDA-event timing (off by default). name: "gemm_nn",
 * "gemm_tn", "orth", "small_svd", "cpqr", "sketch_f32", ... Returns the
 * number of timed launches and their summed duration since the last reset. */
int rfgpu_profile_enable(rfgpu_ctx* ctx, int on);
int rfgpu_profile_reset(rfgpu_ctx* ctx);
int rfgpu_profile_read(rfgpu_ctx* ctx, const char* name, int64_t* launches, double* total_ms);
/* Number of rfgpu kernel launches issued since the last reset. */
int64_t rfgpu_launch_count(rfgpu_ctx* ctx);

/* ---- device matrices ------------------------------------------------------
 * A (this rank's rows) as a device-resident handle. upload copies from host
 * (column-major, lda >= m); wrap_device adopts an existing device buffer
 * without copying (caller keeps it alive). */
int rfgpu_matrix_upload(rfgpu_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda, rfgpu_matrix** out);
int rfgpu_matrix_wrap_device(rfgpu_ctx* ctx, const double* a_dev, int64_t m, int64_t n, int64_t lda,
                             rfgpu_matrix** out);
int rfgpu_matrix_upload_f32(rfgpu_ctx* ctx, const float* a, int64_t m, int64_t n, int64_t lda, rfgpu_matrix** out);
int rfgpu_matrix_wrap_device_f32(rfgpu_ctx* ctx, const float* a_dev, int64_t m, int64_t n, int64_t lda,
                                 rfgpu_matrix** out);
int rfgpu_matrix_free(rfgpu_matrix* h);
int rfgpu_matrix_shape(const rfgpu_matrix* h, int64_t* m_local, int64_t* n, int64_t* m_global, int64_t* row0);

/* ---- products (randfact::multiply, proj/src/dense.cpp:155-187) ----------
 * C = A * X (NN, C m_local x ncols) or C = A^T * X (TN, X m_local x ncols,
 * C n x ncols, summed over ranks). Host buffers. */
int rfgpu_multiply(rfgpu_ctx* ctx, const rfgpu_matrix* a, int trans, const double* x, int64_t ncols, double* c);

/* ---- range finder ----------------------------------------------------------
 * randfact::power_range / basic_range (proj/include/randfact/rangefinder.hpp:
 * 50,55; proj/src/rangefinder.cpp:56-80) including finish_with_projection
 * (:24-30). G is n x ell (ell = k + p) from rfgpu_gaussian(seed, "range.G").
 * Outputs: Q (m_local x ell_out, caller allocates m_local*ell), B (ell_out x n,
 * caller allocates ell*n), *resid = ||A - Q B||_F by down-dating
 * (frob_residual, :45-54), *ell_out = kept columns (orth may drop). Any of
 * Q/B/resid may be NULL.
 * Device-path limit (all sketching entry points): ell = k + p <= 736, else
 * RFGPU_EPARAM (the reference has no such bound). */
int rfgpu_range_finder(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* g, int64_t ell, int64_t q, int reorth,
                       double* Q, double* B, double* resid, int64_t* ell_out);

/* randfact::rsvd (proj/include/randfact/lowrank.hpp:15-16;
 * proj/src/lowrank.cpp:74-96). U m_local x r, D r, V n x r with
 * r = keep_oversamples ? ell' : min(k, ell'); caller allocates for r = ell. */
int rfgpu_rsvd(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* g, int64_t k, int64_t ell, int64_t q,
               int keep_oversamples, int reorth, double* U, double* D, double* V, int64_t* rank_out);

/* Host-matrix variant: the value-semantics drop-in rsvd(const DenseMatrix& a,
 * ...) (lowrank.hpp:15-16). A (m_local x n, column-major, leading dim lda) is
 * read from host memory: it is copied into a device buffer cached on the
 * context in row panels whose H2D copies overlap the first pass (pinned host
 * memory gives full copy bandwidth; pageable works, slower). The caller's
 * buffer is no longer read once the call returns. Outputs as rfgpu_rsvd. */
int rfgpu_rsvd_host(rfgpu_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda, const double* g, int64_t k,
                    int64_t ell, int64_t q, int keep_oversamples, int reorth, double* U, double* D, double* V,
                    int64_t* rank_out);

/* Device-pointer variant (inputs and outputs in device memory; no host
 * copies): the path bench.py times for the device-resident metric. */
int rfgpu_rsvd_device(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* g_dev, int64_t k, int64_t ell,
                      int64_t q, int keep_oversamples, int reorth, double* U_dev, double* D_dev, double* V_dev,
                      int64_t* rank_out);

/* ---- interpolative decompositions -----------------------------------------
 * Row sketch Y = G * A (ell x n) for randfact::randomized_cur
 * (proj/src/lowrank.cpp:351-352); G is ell x m_global from
 * rfgpu_gaussian(seed, "cur.G"); each rank passes the FULL G. Host buffers. */
int rfgpu_row_sketch(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* g, int64_t ell, double* Y);
int rfgpu_row_sketch_device(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* g_dev, int64_t ell, double* Y_dev);

/* Column ID core (col_id_core, proj/src/lowrank.cpp:51-70 = cpqr with rank
 * stop, dense.cpp:453-552, + solve_upper, dense.cpp:788-804) of Y (m x n):
 * Js (k), Z (k x n) with Z(:, Js) = I, *rank_out = min(k, stopped rank),
 * *truncated = rank_out < k. Pivot order matches the reference exactly
 * (first index attaining the maximum down-dated norm; recompute and halt
 * rules as in the reference). */
int rfgpu_col_id(rfgpu_ctx* ctx, const double* Y, int64_t m, int64_t n, int64_t k, int64_t* Js, double* Z,
                 int64_t* rank_out, int* truncated);
int rfgpu_col_id_device(rfgpu_ctx* ctx, const double* Y_dev, int64_t m, int64_t n, int64_t k, int64_t* Js,
                        double* Z_dev, int64_t* rank_out, int* truncated);

/* randfact::randomized_id (proj/src/lowrank.cpp:312-329): tall sketch
 * Y = (A A^T)^q A G (G n x ell from rfgpu_gaussian(seed, "rid.G")), row ID
 * from col_id_core(Y^T, k). Is (k), X (m x rank, ld m). Single GPU. */
int rfgpu_randomized_id(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* g, int64_t k, int64_t ell, int64_t q,
                        int64_t* Is, double* X, int64_t* rank_out, int* truncated);

/* randfact::randomized_cur (proj/src/lowrank.cpp:348-372): G ell x m from
 * rfgpu_gaussian(seed, "cur.G"); column ID of G A, row ID of A(:, Js),
 * U (kc x kr, ld kc) by the reference's SVD least squares (1e-12 cutoff),
 * cond numbers of C and R, warning = either > 1e8. Single GPU. */
int rfgpu_randomized_cur(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* g, int64_t k, int64_t ell, int64_t q,
                         int64_t* Js, int64_t* Is, double* U, double* cond_c, double* cond_r, int* warning,
                         int64_t* kc_out, int64_t* kr_out);

/* ---- single pass (FP32) ---------------------------------------------------
 * Dual sketch of randfact::single_pass_svd (proj/src/lowrank.cpp:170-176):
 * one read of A (fp32 handle) -> Yc = A Gc (m_local x ell),
 * Yr = A^T Gr (n x ell, summed over ranks). Gc n x ell, Gr m_local x ell. */
int rfgpu_dual_sketch_f32(rfgpu_ctx* ctx, const rfgpu_matrix* a32, const float* gc, const float* gr, int64_t ell,
                          float* yc, float* yr);

/* randfact::svd_dense for tall input (proj/src/dense.cpp:585-701 semantics:
 * D non-increasing, U columns normalised): CholeskyQR2 + one-sided Jacobi on
 * the cols x cols factor (cluster of up to 16 CTAs), or Jacobi on M when
 * CholeskyQR is not accepted. rows >= cols; *sweeps = Jacobi sweeps used. */
int rfgpu_svd(rfgpu_ctx* ctx, const double* M, int64_t rows, int64_t cols, double* U, double* S, double* V,
              int* sweeps);

/* randfact::frob_residual (proj/src/rangefinder.cpp:45-54; the residual of
 * finish_with_projection): *resid = sqrt(max(0, a_frob^2 - ||B||_F^2)),
 * ||B||_F summed on the device over the count entries of B (host buffer).
 * RFGPU_ENUMERICAL when ||B||_F > a_frob (1 + 1e-8) (basis orthonormality was
 * lost upstream); RFGPU_EPARAM when a_frob is negative or NaN. */
int rfgpu_frob_residual(rfgpu_ctx* ctx, double a_frob, const double* B, int64_t count, double* resid);

/* Error of a low-rank factorization A ~ L R recomputed on the device, for the
 * randfact/1 reports (the CLI's error block, proj/src/cli.cpp:191-206):
 * *frob_abs = ||A - L R||_F (L m x k, R k x n, host, column-major; the
 * product is formed in 256-column blocks and subtracted in a fused
 * sum-of-squares pass); probe_norms[i] = ||(A - L R) g_i|| for the nprobes
 * columns g_i of probes (n x nprobes host; the CLI passes
 * gaussian(seed ^ 0x9e3779b9, "specnorm", n, 10), the reference's probe
 * stream, diagnostics.cpp:75-96). k may be 0 (L R = 0). */
int rfgpu_lowrank_error(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* L, const double* R, int64_t k,
                        const double* probes, int64_t nprobes, double* frob_abs, double* probe_norms);

/* ---- single pass (randfact::single_pass_svd, proj/src/lowrank.cpp:160-220)
 * Streaming form (MatrixStream, proj/include/randfact/stream.hpp:13-41):
 * begin with Gc = gaussian(seed, "spsvd.Gc", n, ell) and
 * Gr = gaussian(seed, "spsvd.Gr", m, ell); push every column block once, in
 * order (ESTREAM otherwise); finish solves the core on the device and frees
 * the state (U m x r, D r, V n x r, r = min(k, ell)). */
typedef struct rfgpu_single_pass rfgpu_single_pass;
int rfgpu_single_pass_begin(rfgpu_ctx* ctx, int64_t m, int64_t n, int64_t ell, const double* gc, const double* gr,
                            rfgpu_single_pass** out);
int rfgpu_single_pass_push(rfgpu_single_pass* sp, int64_t col0, const double* block, int64_t ncols);
int rfgpu_single_pass_finish(rfgpu_single_pass* sp, int64_t k, double* U, double* D, double* V, int64_t* rank_out);
int rfgpu_single_pass_abort(rfgpu_single_pass* sp);
/* One-shot on a device-resident A (fp64 or fp32 handle; an fp32 matrix is
 * widened chunk by chunk, every entry read once). Gc, Gr, U, D, V device. */
int rfgpu_single_pass_svd_device(rfgpu_ctx* ctx, const rfgpu_matrix* a, const double* gc_dev, const double* gr_dev,
                                 int64_t k, int64_t ell, double* U_dev, double* D_dev, double* V_dev,
                                 int64_t* rank_out);

#ifdef __cplusplus
}
#endif

#endif /* RFGPU_H */
