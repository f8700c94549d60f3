// Small dense FP64 kernels for the l x l side of the range finder.
//
//  * chol_inv    Cholesky + triangular inverse of the l x l Gram matrix for
//                CholeskyQR2 (replaces orth's MGS, proj/src/dense.cpp:402-431,
//                on well-conditioned sketches; R bitwise follows the
//                reference cholesky recurrence, proj/src/dense.cpp:763-786).
//  * jacobi_svd  one-sided (Hestenes) Jacobi SVD with the reference's rotation
//                formula, skip tolerance and sweep cap (proj/src/dense.cpp:
//                585-686), parallelised with a round-robin pair ordering. The
//                rows of X and V are split across a thread-block cluster of
//                up to 8 CTAs; each round exchanges only the 3 partial inner
//                products per column pair through distributed shared memory.
//  * sumsq       fixed-order sum of squares (frob_norm, dense.cpp:232-236).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "rfgpu_internal.h"

namespace cg = cooperative_groups;

namespace rfgpu {

namespace {

constexpr int kSmallThreads = 1024;
constexpr int kMaxSmallFactor = 736;  // the blocked triangular inverse's block column in shared memory (cpqr.cu)

// ------------------------------------------------------------ chol_inv ---
// One CTA, the packed upper triangle P (column-packed: (i, j) at
// j(j+1)/2 + i, i <= j) in shared memory (c <= 236).
// Outer-product Cholesky on the UNSCALED rows: step j subtracts
// P(j,i) P(j,col) / P(j,j) from every trailing entry (i, col), j < i <= col.
// Row j is final after step j - 1 and only rows > j are written in step j,
// so one barrier per step suffices; the pivot row is read from a contiguous
// copy (rowb, double-buffered by step parity: the lanes that update row j + 1
// in step j also write it there). Afterwards R(j, :) = P(j, :) / sqrt(P(j,j)).
// The pivot test is the reference rule (pivot <= 1e-14 max initial diagonal,
// proj/src/dense.cpp:763-786) plus the CholeskyQR gate statistic
// min_j pivot_j / trace(G). rdiag receives 1 / R(j,j) for trinv_smem_kernel.

__global__ void __launch_bounds__(kSmallThreads, 1)
    chol_kernel(const double* __restrict__ G, int c, double* __restrict__ R, double* __restrict__ rdiag, int* info,
                double* info_d) {
  extern __shared__ double sm[];
  double* rowb = sm;        // [2][c] pivot rows (unscaled)
  double* P = sm + 2 * c;   // packed upper triangle: column col starts at col (col + 1) / 2
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  __shared__ double s_floor, s_trace, s_minratio;

  for (int j = warp; j < c; j += nwarps)
    for (int i = lane; i <= j; i += 32) P[j * (j + 1) / 2 + i] = G[static_cast<int64_t>(j) * c + i];
  for (int j = tid; j < c; j += blockDim.x) rowb[j] = G[static_cast<int64_t>(j) * c];  // row 0
  if (warp == 0) {
    double mx = 0.0, tr = 0.0;
    for (int j = lane; j < c; j += 32) {
      const double g = G[static_cast<int64_t>(j) * c + j];
      mx = fmax(mx, fabs(g));
      tr += g;
    }
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      tr += __shfl_xor_sync(0xffffffffu, tr, o);
    }
    if (lane == 0) {
      s_floor = 1e-14 * mx;
      s_trace = tr;
      s_minratio = INFINITY;
    }
  }
  __syncthreads();
  const double floor = s_floor, trace = s_trace;
  int fail = 0;
  for (int j = 0; j < c; ++j) {
    const double* rj = rowb + (j & 1) * c;
    double* rn = rowb + ((j + 1) & 1) * c;
    const double d = rj[j];
    if (d <= floor || !(d > 0.0)) {  // every thread sees the same pivot
      fail = j + 1;
      break;
    }
    if (tid == 0) s_minratio = fmin(s_minratio, trace > 0.0 ? d / trace : 0.0);
    const double inv_d = 1.0 / d;
    const int i0 = j + 1 + lane;
    const double r0 = i0 < c ? rj[i0] : 0.0;  // this lane's first pivot-row element (same for every column)
    for (int col = j + 1 + warp; col < c; col += nwarps) {
      double* pc = P + col * (col + 1) / 2;
      const double f = rj[col] * inv_d;
      if (i0 <= col) {  // lane 0 holds row j + 1: publish it as the next pivot row
        const double v = fma(-r0, f, pc[i0]);
        pc[i0] = v;
        if (lane == 0) rn[col] = v;
      }
      int i = i0 + 32;
      for (; i + 32 <= col; i += 64) {
        const double a0 = rj[i], a1 = rj[i + 32], p0 = pc[i], p1 = pc[i + 32];
        pc[i] = fma(-a0, f, p0);
        pc[i + 32] = fma(-a1, f, p1);
      }
      if (i <= col) pc[i] = fma(-rj[i], f, pc[i]);
    }
    __syncthreads();
  }
  if (tid == 0) {
    info[0] = fail;
    info_d[0] = s_minratio;
  }
  if (fail) return;
  double* rs = rowb;  // sqrt of the pivots (the row buffers are free now)
  for (int j = tid; j < c; j += blockDim.x) {
    const double r = sqrt(P[j * (j + 1) / 2 + j]);
    rs[j] = r;
    rdiag[j] = 1.0 / r;
  }
  __syncthreads();
  for (int j = warp; j < c; j += nwarps) {
    const double* pj = P + j * (j + 1) / 2;
    for (int i = lane; i < c; i += 32)
      R[static_cast<int64_t>(j) * c + i] = i < j ? pj[i] / rs[i] : (i == j ? rs[j] : 0.0);
  }
}

// The same factorization with the matrix in REGISTERS (c <= 128): the per-step update of chol_kernel moves
// three doubles through shared memory per entry (c^3 / 2 in all: at l = 110 that is 5 MB through 128 B/clk,
// as long as the arithmetic), so here the 32 x 32 thread grid owns the entries 2-D cyclically (thread (ti, tj):
// rows ti + 32 a, columns tj + 32 b) and only the pivot row goes through shared memory (the contiguous
// double-buffered copy, published by the threads that own row j + 1). Same operations on every entry in the
// same order as chol_kernel: bitwise the same R, rdiag and gate statistics.
template <int T>
__global__ void __launch_bounds__(kSmallThreads, 1)
    chol_reg_kernel(const double* __restrict__ G, int c, double* __restrict__ R, double* __restrict__ rdiag, int* info,
                    double* info_d) {
  extern __shared__ double sm[];
  double* rowb = sm;          // [2][c] pivot rows (unscaled)
  double* piv = sm + 2 * c;   // [c] pivots
  const int tid = threadIdx.x, ti = tid & 31, tj = tid >> 5;
  __shared__ double s_floor, s_trace, s_minratio;
  double e[T][T];
#pragma unroll
  for (int b = 0; b < T; ++b)
#pragma unroll
    for (int a = 0; a < T; ++a) {
      const int i = ti + 32 * a, col = tj + 32 * b;
      e[a][b] = (i <= col && col < c) ? G[static_cast<int64_t>(col) * c + i] : 0.0;
      if (i == 0 && col < c) rowb[col] = e[a][b];  // row 0
    }
  if (tj == 0) {
    double mx = 0.0, tr = 0.0;
    for (int j = ti; j < c; j += 32) {
      const double g = G[static_cast<int64_t>(j) * c + j];
      mx = fmax(mx, fabs(g));
      tr += g;
    }
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      tr += __shfl_xor_sync(0xffffffffu, tr, o);
    }
    if (ti == 0) {
      s_floor = 1e-14 * mx;
      s_trace = tr;
      s_minratio = INFINITY;
    }
  }
  __syncthreads();
  const double floor = s_floor, trace = s_trace;
  int fail = 0;
  for (int j = 0; j < c; ++j) {
    const double* rj = rowb + (j & 1) * c;
    double* rn = rowb + ((j + 1) & 1) * c;
    const double d = rj[j];
    if (d <= floor || !(d > 0.0)) {  // every thread sees the same pivot
      fail = j + 1;
      break;
    }
    if (tid == 0) {
      s_minratio = fmin(s_minratio, trace > 0.0 ? d / trace : 0.0);
      piv[j] = d;
    }
    const double inv_d = 1.0 / d;
#pragma unroll
    for (int b = 0; b < T; ++b) {
      const int col = tj + 32 * b;
      if (col > j && col < c) {
        const double f = rj[col] * inv_d;
#pragma unroll
        for (int a = 0; a < T; ++a) {
          const int i = ti + 32 * a;
          if (i > j && i <= col) {
            const double v = fma(-rj[i], f, e[a][b]);
            e[a][b] = v;
            if (i == j + 1) rn[col] = v;  // the next pivot row
          }
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    info[0] = fail;
    info_d[0] = s_minratio;
  }
  if (fail) return;
  double* rs = rowb;  // sqrt of the pivots (the row buffers are free now)
  for (int j = tid; j < c; j += blockDim.x) {
    const double r = sqrt(piv[j]);
    rs[j] = r;
    rdiag[j] = 1.0 / r;
  }
  __syncthreads();
#pragma unroll
  for (int b = 0; b < T; ++b)
#pragma unroll
    for (int a = 0; a < T; ++a) {
      const int i = ti + 32 * a, col = tj + 32 * b;
      if (i < c && col < c) R[static_cast<int64_t>(col) * c + i] = i < col ? e[a][b] / rs[i] : (i == col ? rs[i] : 0.0);
    }
}

// R^{-1} of the upper-triangular c x c R (c <= 236): each CTA stages the packed
// upper triangle in shared memory, one warp per column j: back substitution
// R x = e_j in axpy form, x over the lanes' registers (S slots), the pivots
// multiplied by the precomputed 1 / R(i,i). Measured at l = 220: chol_kernel
// 344 us + this 50 us, against 376 + 257 us for the three-barrier kernel and
// the global-memory trinv_upper.
template <int S>
__global__ void __launch_bounds__(kSmallThreads, 1)
    trinv_smem_kernel(const double* __restrict__ R, int c, const double* __restrict__ rdiag, double* __restrict__ Rinv) {
  extern __shared__ double P[];  // packed upper triangle
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int j = warp; j < c; j += nwarps)
    for (int i = lane; i <= j; i += 32) P[j * (j + 1) / 2 + i] = R[static_cast<int64_t>(j) * c + i];
  __syncthreads();
  const int j = blockIdx.x * nwarps + warp;
  if (j >= c) return;
  double x[S];
#pragma unroll
  for (int s = 0; s < S; ++s) x[s] = (lane + 32 * s == j) ? 1.0 : 0.0;
  // rows i = j .. 0 in slot-major order: the slot si = i / 32 is a compile-time
  // register index, so each step is shuffle + multiply + (si + 1) FMAs
#pragma unroll
  for (int si = S - 1; si >= 0; --si) {
    if (32 * si > j) continue;
    for (int ii = min(31, j - 32 * si); ii >= 0; --ii) {
      const int i = 32 * si + ii;
      const double* pi = P + i * (i + 1) / 2;  // column i of R
      const double xi = __shfl_sync(0xffffffffu, x[si], ii) * rdiag[i];
#pragma unroll
      for (int s = 0; s < si; ++s) x[s] = fma(-xi, pi[lane + 32 * s], x[s]);
      if (lane == ii) x[si] = xi;
      else if (lane < ii) x[si] = fma(-xi, pi[lane + 32 * si], x[si]);
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int r = lane + 32 * s;
    if (r < c) Rinv[static_cast<int64_t>(j) * c + r] = r <= j ? x[s] : 0.0;
  }
}

// ----------------------------------------------------------- jacobi_svd ---
// Round-robin parallel one-sided Jacobi. The rows of X (mr x c) and V (c x c)
// are split over the P CTAs of a cluster; inside a CTA the 32 warps form
// G pair-groups x H row-groups: lane k of a warp owns column pair
// 32*g + k of the round, the warp owns a row slice. Per round:
//   A. partial (app, aqq, apq) over the warp's rows      -> red[h][k]
//   B. row-group reduction (fixed order), pushed to every CTA's pbuf[q][k]
//   C. one warp per pair-group sums the P CTA partials (fixed order) and
//      computes the rotation (reference formula, dense.cpp:624-644)
//   D. every warp rotates its row slice of X and V.
// Decisions are bitwise identical in all CTAs (same sums, same order).
struct JacobiParams {
  const double* X;
  int64_t mr;  // rows of X
  int c;       // columns
  double* U;
  double* S;
  double* V;
  double* gX;  // global staging when X/V rows do not fit in shared memory
  double* gV;
  double* gS;  // per-CTA staging for the physical column permutation of each sweep
  int RX, RV;  // rows of X / V owned per CTA
  int LDX, LDV;
  int bcast;  // 1: every CTA receives every partial (one hop); 0: owner CTA per pair (two hops, less smem)
  long long* trace;  // optional: clock64 at the phase boundaries of sweep 0 (CTA 0, thread 0)
  int* info;
  int* sweeps_out;
};

__device__ __forceinline__ void pair_of(int r, int k, int cc, int* a, int* b) {
  // circle-method round-robin on cc (even) logical positions
  const int n = cc - 1;
  int x, y;
  if (k == 0) {
    x = 0;
    y = 1 + r;  // r < n
  } else {
    int t = r + k;
    if (t >= n) t -= n;
    x = 1 + t;
    t = r - k;
    if (t < 0) t += n;
    y = 1 + t;
  }
  *a = min(x, y);
  *b = max(x, y);
}

template <bool SMEM>
// Two independent problems of the same shape may share a launch: cluster 0
// solves p0, cluster 1 solves p1 (the single-pass core's Yc / Yr and P / W^T
// pairs), so their latency-bound rounds overlap.
__global__ void __launch_bounds__(kSmallThreads, 1) jacobi_svd_kernel(const JacobiParams p0, const JacobiParams p1) {
  cg::cluster_group cluster = cg::this_cluster();
  const int P = static_cast<int>(cluster.num_blocks());
  const JacobiParams& p = (static_cast<int>(blockIdx.x) / P == 0) ? p0 : p1;
  const int q = static_cast<int>(cluster.block_rank());
  const int c = p.c, cc = c + (c & 1), npairs = cc / 2;
  const int RX = p.RX, RV = p.RV, LDX = p.LDX, LDV = p.LDV;
  const int64_t r0x = static_cast<int64_t>(q) * RX;
  const int64_t rem_x = p.mr - r0x;
  const int nrx = rem_x <= 0 ? 0 : static_cast<int>(rem_x < RX ? rem_x : RX);
  const int r0v = q * RV;
  const int nrv = max(0, min(RV, c - r0v));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int G = (npairs + 31) / 32;
  const int H = nwarps / G;  // row groups (>= 1 since npairs <= 1024)
  const int g = warp % G, h = warp / G;
  const bool active = h < H;
  const int k = g * 32 + lane;  // pair owned by this lane
  const int rhx = (nrx + H - 1) / H, rhv = (nrv + H - 1) / H;
  const int x0 = min(nrx, h * rhx), x1 = min(nrx, x0 + rhx);
  const int v0 = min(nrv, h * rhv), v1 = min(nrv, v0 + rhv);
  const bool bc = p.bcast != 0 || P == 1;
  // Exchange layout. Partials are staged per destination in `outb` and shipped
  // with ONE bulk shared->shared copy per destination CTA per round (TMA
  // engine, transaction bytes on the receiver's mbarrier).
  //   bc (one hop): every CTA receives every pair's partial; params computed
  //                 locally.  block = npairs partials.
  //   owner:        pair k's partials go to CTA k % P (block = its owned pairs),
  //                 which broadcasts (cs, sn) back as one bulk copy.
  const int npo = bc ? npairs : (npairs + P - 1) / P;  // pairs per destination block
  const int blk3 = (npo * 3 + 1) & ~1;                 // doubles per partial block (16B multiple)
  auto owned_by = [&](int d) { return bc ? npairs : (npairs - d + P - 1) / P; };

  extern __shared__ double sm[];
  double* Xs;
  double* Vs;
  double* rest;
  if (SMEM) {
    Xs = sm;
    Vs = sm + static_cast<size_t>(c) * LDX;
    rest = Vs + static_cast<size_t>(c) * LDV;
  } else {
    Xs = p.gX + static_cast<size_t>(q) * c * LDX;
    Vs = p.gV + static_cast<size_t>(q) * c * LDV;
    rest = sm;
  }
  const int np3 = npairs * 3;
  uint64_t* bars = reinterpret_cast<uint64_t*>(rest);  // [0..1] partial inbox, [2..3] params
  double* params = rest + 4;                           // [2][P][npo][2] by owner (bc: [2][npairs][2])
  // staging buffers are double-buffered by round parity: a bulk copy of
  // round r is known to have landed everywhere only after round r+1's waits
  double* pout = params + 4 * P * npo;                 // [2][npo][2] this owner's params (owner mode)
  double* outb = pout + 4 * npo;                       // [2][P][blk3] staged partials per destination
  double* inbox = outb + 2 * P * blk3;                 // [2][P][blk3]
  double* red = inbox + 2 * P * blk3;                  // [H][npairs][3], aliased by nrmp [P][cc]
  const int red_sz = max(H * np3, P * cc);
  double* nrmp = red;
  double* nrm = red + red_sz;                          // [cc]
  int* perm = reinterpret_cast<int*>(nrm + cc);        // [cc]
  __shared__ int s_rotated, s_conv;

  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  uint32_t uses0 = 0u, uses1 = 0u;
  for (int e = tid; e < c * RX; e += blockDim.x) {
    const int col = e / RX, r = e % RX;
    Xs[static_cast<size_t>(col) * LDX + r] = (r < nrx) ? p.X[static_cast<int64_t>(col) * p.mr + r0x + r] : 0.0;
  }
  for (int e = tid; e < c * RV; e += blockDim.x) {
    const int col = e / RV, r = e % RV;
    Vs[static_cast<size_t>(col) * LDV + r] = (r < nrv && r0v + r == col) ? 1.0 : 0.0;
  }
  cluster.sync();  // barriers initialised cluster-wide before any remote copy

  // Column norms over the owned rows, exchanged across the cluster; nrm[j]
  // receives the total in fixed rank order.
  auto norms = [&]() {
    for (int col = warp; col < c; col += nwarps) {
      double s = 0.0;
      const double* x = Xs + static_cast<size_t>(col) * LDX;
      for (int r = lane; r < nrx; r += 32) s = fma(x[r], x[r], s);
      s = warp_sum(s);
      if (lane < P) cluster.map_shared_rank(nrmp, lane)[q * cc + col] = s;
    }
    cluster.sync();
    for (int j = tid; j < c; j += blockDim.x) {
      double t = 0.0;
      for (int d = 0; d < P; ++d) t += nrmp[d * cc + j];
      nrm[j] = t;
    }
    __syncthreads();
  };
  auto sort_desc = [&](const double* key) {
    for (int j = tid; j < c; j += blockDim.x) {
      const double kj = key[j];
      int rank = 0;
      for (int i = 0; i < c; ++i) {
        const double ki = key[i];
        rank += (ki > kj || (ki == kj && i < j)) ? 1 : 0;
      }
      perm[rank] = j;
    }
    if (tid == 0 && (c & 1)) perm[c] = -1;  // phantom column
    __syncthreads();
  };
  // Physically reorder the columns of X and V by perm (through global
  // staging), so that a round's pairs are consecutive columns: lanes then hit
  // distinct shared-memory banks (odd leading dimensions).
  auto permute_cols = [&]() {
    double* sx = p.gS + static_cast<size_t>(q) * c * (LDX + LDV);
    double* sv = sx + static_cast<size_t>(c) * LDX;
    for (int e = tid; e < c * LDX; e += blockDim.x) sx[e] = Xs[e];
    for (int e = tid; e < c * LDV; e += blockDim.x) sv[e] = Vs[e];
    __syncthreads();
    for (int e = tid; e < c * nrx; e += blockDim.x) {
      const int col = e / nrx, r = e - col * nrx;
      Xs[static_cast<size_t>(col) * LDX + r] = sx[static_cast<size_t>(perm[col]) * LDX + r];
    }
    for (int e = tid; e < c * nrv; e += blockDim.x) {
      const int col = e / nrv, r = e - col * nrv;
      Vs[static_cast<size_t>(col) * LDV + r] = sv[static_cast<size_t>(perm[col]) * LDV + r];
    }
    __syncthreads();
  };

  const int kd = bc ? 0 : k % P;   // destination block of pair k
  const int kl = bc ? k : k / P;   // slot of pair k inside its block
  int sweep = 0, parity = 0;
#ifdef RFGPU_JACOBI_TRACE
  long long tacc[14] = {0}, tlast = 0;  // per-slot clocks of sweep 0, CTA 0, thread 0
#endif
  if (tid == 0) s_conv = (c <= 1);
  __syncthreads();
  while (!s_conv && sweep < 60) {
    norms();
    sort_desc(nrm);
    permute_cols();
    if (tid == 0) s_rotated = 0;
    __syncthreads();
#ifdef RFGPU_JACOBI_TRACE
    const bool tracing = p.trace && sweep == 0 && q == 0 && tid == 0;
#define RF_TRACE(slot)                                                     \
  if (tracing) {                                                           \
    const long long now = clock64();                                       \
    if (rd >= 1 && rd < 31 && (slot) > 0) tacc[(slot)] += now - tlast;     \
    if ((slot) == 0 && rd >= 2 && rd < 32) tacc[0] += now - tlast;         \
    tlast = now;                                                           \
  }
#else
#define RF_TRACE(slot)
#endif
    for (int rd = 0; rd < cc - 1; ++rd) {
      RF_TRACE(0)
      int cp = -1, cq = -1;
      if (active && k < npairs) {
        int a, b;
        pair_of(rd, k, cc, &a, &b);
        cp = a < c ? a : -1;
        cq = b < c ? b : -1;
      }
      const bool valid = cp >= 0 && cq >= 0;
      const uint32_t ph = (parity ? uses1 : uses0) & 1u;
      if (P > 1 && tid == blockDim.x - 32) {  // a lane off the reduction warps' critical path
        uint32_t bytes = 0;  // partial blocks from every CTA
        for (int d = 0; d < P; ++d) bytes += static_cast<uint32_t>(((owned_by(q) * 3 + 1) & ~1) * 8);
        mbar_arrive_expect_tx(&bars[parity], bytes);
        if (!bc) mbar_arrive_expect_tx(&bars[2 + parity], static_cast<uint32_t>(npairs * 16));
      }
      RF_TRACE(1)
      // A. partial inner products over this warp's rows
      if (active && k < npairs) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        if (valid) {
          const double* __restrict__ xp = Xs + static_cast<size_t>(cp) * LDX;
          const double* __restrict__ xq = Xs + static_cast<size_t>(cq) * LDX;
          // 4 rows in flight: the loads of a group issue back to back
          double bpp = 0.0, bqq = 0.0, bpq = 0.0;
          int r = x0;
          for (; r + 4 <= x1; r += 4) {
            const double u0 = xp[r], u1 = xp[r + 1], u2 = xp[r + 2], u3 = xp[r + 3];
            const double v0 = xq[r], v1 = xq[r + 1], v2 = xq[r + 2], v3 = xq[r + 3];
            app = fma(u0, u0, app);
            aqq = fma(v0, v0, aqq);
            apq = fma(u0, v0, apq);
            bpp = fma(u1, u1, bpp);
            bqq = fma(v1, v1, bqq);
            bpq = fma(u1, v1, bpq);
            app = fma(u2, u2, app);
            aqq = fma(v2, v2, aqq);
            apq = fma(u2, v2, apq);
            bpp = fma(u3, u3, bpp);
            bqq = fma(v3, v3, bqq);
            bpq = fma(u3, v3, bpq);
          }
          for (; r < x1; ++r) {
            const double u = xp[r], v = xq[r];
            app = fma(u, u, app);
            aqq = fma(v, v, aqq);
            apq = fma(u, v, apq);
          }
          app += bpp;
          aqq += bqq;
          apq += bpq;
        }
        RF_TRACE(2)
        double* d = red + (h * npairs + k) * 3;
        d[0] = app;
        d[1] = aqq;
        d[2] = apq;
      }
      RF_TRACE(3)
      __syncthreads();
      RF_TRACE(4)
      // B. CTA partial (fixed row-group order), staged per destination block
      double* ib = inbox + parity * P * blk3;
      double* pr = params + parity * 2 * P * npo;
      if (h == 0 && k < npairs) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll 4
        for (int hh = 0; hh < H; ++hh) {
          const double* s = red + (hh * npairs + k) * 3;
          app += s[0];
          aqq += s[1];
          apq += s[2];
        }
        double* slot = (P > 1 ? outb + (parity * P + kd) * blk3 : ib) + kl * 3;
        slot[0] = app;
        slot[1] = aqq;
        slot[2] = apq;
        if (P > 1) fence_proxy_async_smem();
      }
      RF_TRACE(5)
      __syncthreads();
      RF_TRACE(6)
      if (P > 1 && tid < P) {  // lane d ships block d to CTA d (bc: the same full block to all)
        const int dd = tid;
        const double* src = outb + (parity * P + (bc ? 0 : dd)) * blk3;
        const uint32_t bytes = static_cast<uint32_t>(((owned_by(dd) * 3 + 1) & ~1) * 8);
        bulk_s2s_cluster(mapa_u32(smem_u32(ib + q * blk3), dd), src, bytes, mapa_u32(smem_u32(&bars[parity]), dd));
      }
      RF_TRACE(7)
      if (P > 1 && h == 0) mbar_wait(&bars[parity], ph);
      RF_TRACE(8)
      // C. rotation parameters (reference formula, dense.cpp:624-644)
      if (h == 0 && k < npairs && (bc || kd == q)) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int d = 0; d < P; ++d) {
          const double* s = ib + d * blk3 + kl * 3;
          app += s[0];
          aqq += s[1];
          apq += s[2];
        }
        double cs = 1.0, sn = 2.0;
        if (valid && app != 0.0 && aqq != 0.0 && !(fabs(apq) <= 1e-15 * sqrt(app * aqq))) {
          const double zeta = (aqq - app) / (2.0 * apq);
          const double t = (zeta < 0.0 ? -1.0 : 1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          cs = rsqrt(1.0 + t * t);
          sn = cs * t;
        }
        double* dst = bc ? pr + 2 * k : pout + parity * 2 * npo + 2 * kl;
        dst[0] = cs;
        dst[1] = sn;
        if (!bc) fence_proxy_async_smem();
      }
      RF_TRACE(9)
      __syncthreads();
      RF_TRACE(10)
      if (!bc) {
        if (tid < P) {
          const uint32_t bytes = static_cast<uint32_t>(owned_by(q) * 16);
          bulk_s2s_cluster(mapa_u32(smem_u32(pr + q * 2 * npo), tid), pout + parity * 2 * npo, bytes,
                           mapa_u32(smem_u32(&bars[2 + parity]), tid));
        }
        if (active) mbar_wait(&bars[2 + parity], ph);
      }
      if (parity) ++uses1;
      else ++uses0;
      RF_TRACE(11)
      // D. rotate this warp's rows of X and V
      if (active && k < npairs && valid) {
        const double* prm = bc ? pr + 2 * k : pr + kd * 2 * npo + 2 * kl;
        const double cs = prm[0], sn = prm[1];
        if (sn != 2.0) {
          if (h == 0) s_rotated = 1;
          // columns cp != cq never alias: 4 rows of loads in flight per group
          auto rotate = [&](double* __restrict__ a, double* __restrict__ b, int r0, int r1) {
            int r = r0;
            for (; r + 4 <= r1; r += 4) {
              const double u0 = a[r], u1 = a[r + 1], u2 = a[r + 2], u3 = a[r + 3];
              const double w0 = b[r], w1 = b[r + 1], w2 = b[r + 2], w3 = b[r + 3];
              a[r] = cs * u0 - sn * w0;
              a[r + 1] = cs * u1 - sn * w1;
              a[r + 2] = cs * u2 - sn * w2;
              a[r + 3] = cs * u3 - sn * w3;
              b[r] = sn * u0 + cs * w0;
              b[r + 1] = sn * u1 + cs * w1;
              b[r + 2] = sn * u2 + cs * w2;
              b[r + 3] = sn * u3 + cs * w3;
            }
            for (; r < r1; ++r) {
              const double u = a[r], w = b[r];
              a[r] = cs * u - sn * w;
              b[r] = sn * u + cs * w;
            }
          };
          rotate(Xs + static_cast<size_t>(cp) * LDX, Xs + static_cast<size_t>(cq) * LDX, x0, x1);
          rotate(Vs + static_cast<size_t>(cp) * LDV, Vs + static_cast<size_t>(cq) * LDV, v0, v1);
        }
      }
      RF_TRACE(12)
      __syncthreads();
      RF_TRACE(13)
      parity ^= 1;
    }
#ifdef RFGPU_JACOBI_TRACE
    if (tracing)
      for (int i = 0; i < 14; ++i) p.trace[i] = tacc[i];
#endif
    ++sweep;
    if (tid == 0) s_conv = !s_rotated;
    __syncthreads();
  }
  const bool converged = s_conv;

  // final singular values, stable descending order
  norms();
  double* sig = params;  // 4 * P * npo >= 2 * npairs >= c doubles
  for (int j = tid; j < c; j += blockDim.x) sig[j] = sqrt(nrm[j]);
  __syncthreads();
  sort_desc(sig);
  const double smax = c > 0 ? sig[perm[0]] : 0.0;
  int zero_cols = 0;
  for (int j = 0; j < c; ++j) {
    const int src = perm[j];
    const double s = sig[src];
    const bool ok = s > 0.0 && s > smax * 1e-250;
    if (!ok) zero_cols = 1;
    if (q == 0 && tid == 0) p.S[j] = ok ? s : 0.0;
    const double* x = Xs + static_cast<size_t>(src) * LDX;
    for (int r = tid; r < nrx; r += blockDim.x) p.U[static_cast<int64_t>(j) * p.mr + r0x + r] = ok ? x[r] / s : 0.0;
    const double* v = Vs + static_cast<size_t>(src) * LDV;
    for (int r = tid; r < nrv; r += blockDim.x) p.V[static_cast<int64_t>(j) * c + r0v + r] = v[r];
  }
  if (q == 0 && tid == 0) {
    p.info[0] = converged ? (zero_cols ? 2 : 0) : 1;
    if (p.sweeps_out) p.sweeps_out[0] = sweep;
  }
  cluster.sync();  // keep DSMEM alive until every CTA is done with remote writes
}

// ------------------------------------------------------ block Jacobi (BOSJ) ---
// One-sided block Jacobi for the small (l x l) factors, l <= ~440: the c
// columns are cut into nb = 2P blocks of kBJB, and the P CTAs of a cluster
// run the circle-method tournament over blocks. In a block round CTA q loads
// its two blocks (X and V columns, all rows) from the global working copies
// into shared memory, runs one full inner sweep over those 2 kBJB columns
// (2 kBJB - 1 rounds of kBJB disjoint pairs, 64 threads per pair; reference
// rotation formula and skip tolerance, dense.cpp:624-644), and writes them
// back; a cluster barrier separates block rounds. Every column pair meets
// once per block sweep, all of a round's work is CTA-local, and there are
// nb - 1 cluster barriers per sweep instead of c - 1 exchanges.
// Converged when a block sweep meets no pair above 1e-14 relative (kJacobiDone); <= 60 sweeps. The final
// columns are sorted by norm (stable, descending) exactly as jacobi_svd_kernel.
// Block width B = 8 (more CTAs, fewer pairs per CTA per inner round) when the
// tournament fits a 16-CTA cluster, else 12, else 16; one warp per pair (32 B
// threads). Measured at l = 220: B = 8 7.5 ms, B = 16 9.0 ms, the per-column
// cluster kernel 11.4 ms (9-10 sweeps each).

constexpr double kJacobiDone = 1e-14;
constexpr int kBJRegs = 14;    // register-resident cross rounds: rows and columns up to 32 * 14 = 448 ...
constexpr int kBJRegsMin = 1;  // ... and every smaller size (the register count is a template argument: exact fit)

struct BJParams {
  const double* X;  // mr x c input
  int mr, c, nb;
  int cross_only;   // later block rounds visit only the cross pairs
  double* U;
  double* S;
  double* V;
  double* Xg;  // mr x (nb kBJB) working copy
  double* Vg;  // c x (nb kBJB)
  int* info;
  int* sweeps_out;
};

template <int kBJB>
__global__ void __launch_bounds__(32 * kBJB, 1) bjacobi_kernel(const BJParams p0, const BJParams p1) {
  constexpr int kBJThreads = 32 * kBJB;
  cg::cluster_group cluster = cg::this_cluster();
  const int P = static_cast<int>(cluster.num_blocks());
  const BJParams& p = (static_cast<int>(blockIdx.x) / P == 0) ? p0 : p1;
  const int q = static_cast<int>(cluster.block_rank());
  const int mr = p.mr, c = p.c, nb = p.nb, W = nb * kBJB;  // W columns incl. zero padding
  const bool bj_cross_only = p.cross_only != 0;
  const int LX = mr + (mr & 1), LV = c + (c & 1);  // even: every column 16-byte aligned for the bulk copies
  extern __shared__ double sm[];
  double* Xs = sm;                    // [2 kBJB][LX]
  double* Vs = Xs + 2 * kBJB * LX;    // [2 kBJB][LV]
  __shared__ int s_tot[3];            // rotations per sweep (CTA 0's copy is the cluster total), by sweep % 3
  __shared__ int s_rot;
  __shared__ __align__(8) uint64_t s_bar;  // block loads: transaction bytes of the bulk copies
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // working copies with even leading dimensions LX / LV (padding rows zero)
  for (int j = q; j < W; j += P) {
    for (int i = tid; i < LX; i += kBJThreads)
      p.Xg[static_cast<int64_t>(j) * LX + i] = (j < c && i < mr) ? p.X[static_cast<int64_t>(j) * mr + i] : 0.0;
    for (int i = tid; i < LV; i += kBJThreads) p.Vg[static_cast<int64_t>(j) * LV + i] = (i == j && j < c) ? 1.0 : 0.0;
  }
  if (tid == 0) {
    s_tot[0] = s_tot[1] = s_tot[2] = 0;
    mbar_init(&s_bar, 1);
    mbar_fence_init();
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");  // generic writes -> the bulk copies' reads
  cluster.sync();
  uint32_t bar_phase = 0;

  int sweep = 0;
  bool conv = c <= 1;
  while (!conv && sweep < 60) {
    if (q == 0 && tid == 0) s_tot[(sweep + 1) % 3] = 0;  // read two sweeps ago: every CTA is past it
    if (tid == 0) s_rot = 0;
    for (int r = 0; r < nb - 1; ++r) {
      int bi, bj;
      pair_of(r, q, nb, &bi, &bj);
      auto gcol = [&](int t) { return t < kBJB ? bi * kBJB + t : bj * kBJB + t - kBJB; };
      // both blocks (X and V columns) into shared memory: one bulk copy per column on the TMA engine
      // (issued by the lanes of warp 0, one column each: 4 B copies from one thread cost ~1.5 us per round)
      if (warp == 0) {
        if (lane == 0) mbar_arrive_expect_tx(&s_bar, static_cast<uint32_t>(sizeof(double) * 2 * kBJB * (LX + LV)));
        __syncwarp();
        for (int t = lane; t < 2 * kBJB; t += 32) {
          bulk_g2s(Xs + t * LX, p.Xg + static_cast<int64_t>(gcol(t)) * LX, sizeof(double) * LX, &s_bar);
          bulk_g2s(Vs + t * LV, p.Vg + static_cast<int64_t>(gcol(t)) * LV, sizeof(double) * LV, &s_bar);
        }
      }
      mbar_wait(&s_bar, bar_phase);
      bar_phase ^= 1;
      // The first block round of a sweep runs a full inner sweep over the 2B
      // columns (every intra-block pair); later ones only the B x B cross
      // pairs (B rounds: column w of the first block with column (w + s) mod B
      // of the second), so each column pair is visited once per sweep.
      const bool full = r == 0 || !bj_cross_only;
      // Cross rounds with the warp's own column in REGISTERS: in the B cross rounds of a block round warp w
      // always holds column w of the first block, so its X and V entries (rows lane, lane + 32, ...) are
      // loaded once, rotated in registers and written back once; only the partner column goes through
      // shared memory every round. The inner rounds are bound by shared-memory bandwidth (measured at
      // l = 330: 24.2 of the 29.6 us of a block round, 317 KB per round through 128 B/clk): this cuts a
      // round's traffic from 6 mr + 4 c to 2 mr + 2 c doubles per pair. Same operations in the same order:
      // bitwise the shared-memory path, which tall inputs (rows or columns above 32 kBJRegs) keep. The register
      // count per lane is a template argument (2 .. 14): with 14 for every size l = 60 ran 0.93 ms against 0.80
      // ms in shared memory, with the exact count 0.63 ms.
      const int kneed = (max(mr, c) + 31) / 32;  // entries per lane of a column
      auto cross_in_registers = [&](auto k_c) {
        constexpr int K = decltype(k_c)::value;
        const int u = warp;
        double* xus = Xs + u * LX;
        double* vus = Vs + u * LV;
        double xu[K], vu[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int i = lane + 32 * k;
          xu[k] = i < mr ? xus[i] : 0.0;
          vu[k] = i < c ? vus[i] : 0.0;
        }
        for (int ir = 0; ir < kBJB; ++ir) {
          const int v = kBJB + (warp + ir) % kBJB;
          double* xv = Xs + v * LX;
          double xvr[K];
          double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const int i = lane + 32 * k;
            if (i < mr) {
              const double a = xu[k], b = xv[i];
              xvr[k] = b;
              app = fma(a, a, app);
              aqq = fma(b, b, aqq);
              apq = fma(a, b, apq);
            } else {
              xvr[k] = 0.0;
            }
          }
          app = warp_sum(app);
          aqq = warp_sum(aqq);
          apq = warp_sum(apq);
          if (app != 0.0 && aqq != 0.0 && !(apq * apq <= 1e-30 * (app * aqq))) {
            const double zeta = (aqq - app) / (2.0 * apq);
            const double t = (zeta < 0.0 ? -1.0 : 1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double cs = rsqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const int i = lane + 32 * k;
              if (i < mr) {
                const double a = xu[k], b = xvr[k];
                xu[k] = cs * a - sn * b;
                xv[i] = sn * a + cs * b;
              }
            }
            double* vv = Vs + v * LV;
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const int i = lane + 32 * k;
              if (i < c) {
                const double a = vu[k], b = vv[i];
                vu[k] = cs * a - sn * b;
                vv[i] = sn * a + cs * b;
              }
            }
            if (lane == 0 && !(apq * apq <= kJacobiDone * kJacobiDone * (app * aqq))) s_rot = 1;
          }
          __syncthreads();
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int i = lane + 32 * k;
          if (i < mr) xus[i] = xu[k];
          if (i < c) vus[i] = vu[k];
        }
        __syncthreads();
      };
      const bool in_regs = !full && kneed <= kBJRegs && kneed >= kBJRegsMin;
      if (in_regs) {
        if (kneed <= 2) cross_in_registers(std::integral_constant<int, 2>{});
        else if (kneed <= 3) cross_in_registers(std::integral_constant<int, 3>{});
        else if (kneed <= 5) cross_in_registers(std::integral_constant<int, 5>{});
        else if (kneed <= 7) cross_in_registers(std::integral_constant<int, 7>{});
        else if (kneed <= 9) cross_in_registers(std::integral_constant<int, 9>{});
        else if (kneed <= 11) cross_in_registers(std::integral_constant<int, 11>{});
        else cross_in_registers(std::integral_constant<int, kBJRegs>{});
      }
      const int nir = in_regs ? 0 : (full ? 2 * kBJB - 1 : kBJB);
      for (int ir = 0; ir < nir; ++ir) {
        int u, v;
        if (full) {
          pair_of(ir, warp, 2 * kBJB, &u, &v);
        } else {
          u = warp;
          v = kBJB + (warp + ir) % kBJB;
        }
        double* xu = Xs + u * LX;
        double* xv = Xs + v * LX;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int i = lane; i < mr; i += 32) {
          const double a = xu[i], b = xv[i];
          app = fma(a, a, app);
          aqq = fma(b, b, aqq);
          apq = fma(a, b, apq);
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        // skip rule |apq| <= 1e-15 sqrt(app aqq) (dense.cpp:631), squared: no sqrt on the round's chain
        if (app != 0.0 && aqq != 0.0 && !(apq * apq <= 1e-30 * (app * aqq))) {
          const double zeta = (aqq - app) / (2.0 * apq);
          const double t = (zeta < 0.0 ? -1.0 : 1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = rsqrt(1.0 + t * t), sn = cs * t;
          for (int i = lane; i < mr; i += 32) {
            const double a = xu[i], b = xv[i];
            xu[i] = cs * a - sn * b;
            xv[i] = sn * a + cs * b;
          }
          double* vu = Vs + u * LV;
          double* vv = Vs + v * LV;
          for (int i = lane; i < c; i += 32) {
            const double a = vu[i], b = vv[i];
            vu[i] = cs * a - sn * b;
            vv[i] = sn * a + cs * b;
          }
          // The sweeps end once a whole sweep met no pair above kJacobiDone (relative |apq|): rotations of
          // pairs between the reference's skip tolerance (1e-15) and 1e-14 are still applied, but they are at
          // the rounding level of apq itself (eps sqrt(rows)) and would otherwise cost two or three more
          // sweeps of "noise chasing" before one happens to apply none.
          if (lane == 0 && !(apq * apq <= kJacobiDone * kJacobiDone * (app * aqq))) s_rot = 1;
        }
        __syncthreads();
      }
      // write both blocks back with bulk shared->global copies (all rotations are done: the
      // barrier at the end of the last inner round)
      if (warp == 0) {  // one column per lane; every lane commits and waits for its own bulk group
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int t = lane; t < 2 * kBJB; t += 32) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                           p.Xg + static_cast<int64_t>(gcol(t)) * LX),
                       "r"(smem_u32(Xs + t * LX)), "r"(static_cast<uint32_t>(sizeof(double) * LX))
                       : "memory");
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                           p.Vg + static_cast<int64_t>(gcol(t)) * LV),
                       "r"(smem_u32(Vs + t * LV)), "r"(static_cast<uint32_t>(sizeof(double) * LV))
                       : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      cluster.sync();  // block round done everywhere: the working copies are consistent
    }
    if (tid == 0 && s_rot) atomicAdd(cluster.map_shared_rank(&s_tot[sweep % 3], 0), 1);
    cluster.sync();
    conv = *cluster.map_shared_rank(&s_tot[sweep % 3], 0) == 0;
    ++sweep;
  }

  // final singular values (column norms), stable descending order; CTA 0
  if (q == 0) {
    double* nrm = Xs;                             // [W] (shared memory is free now)
    int* perm = reinterpret_cast<int*>(Xs + W);   // [c]
    for (int j = warp; j < c; j += kBJThreads / 32) {
      const double* x = p.Xg + static_cast<int64_t>(j) * LX;
      double s2 = 0.0;
      for (int i = lane; i < mr; i += 32) s2 = fma(x[i], x[i], s2);
      s2 = warp_sum(s2);
      if (lane == 0) nrm[j] = sqrt(s2);
    }
    __syncthreads();
    for (int j = tid; j < c; j += kBJThreads) {
      const double kj = nrm[j];
      int rank = 0;
      for (int i = 0; i < c; ++i) {
        const double ki = nrm[i];
        rank += (ki > kj || (ki == kj && i < j)) ? 1 : 0;
      }
      perm[rank] = j;
    }
    __syncthreads();
    const double smax = c > 0 ? nrm[perm[0]] : 0.0;
    int zero_cols = 0;
    for (int j = 0; j < c; ++j) {
      const int src = perm[j];
      const double sv = nrm[src];
      const bool ok = sv > 0.0 && sv > smax * 1e-250;
      if (!ok) zero_cols = 1;
      if (tid == 0) p.S[j] = ok ? sv : 0.0;
      const double* x = p.Xg + static_cast<int64_t>(src) * LX;
      for (int i = tid; i < mr; i += kBJThreads) p.U[static_cast<int64_t>(j) * mr + i] = ok ? x[i] / sv : 0.0;
      const double* vv = p.Vg + static_cast<int64_t>(src) * LV;
      for (int i = tid; i < c; i += kBJThreads) p.V[static_cast<int64_t>(j) * c + i] = vv[i];
    }
    if (tid == 0) {
      p.info[0] = conv ? (zero_cols ? 2 : 0) : 1;
      if (p.sweeps_out) p.sweeps_out[0] = sweep;
    }
  }
  cluster.sync();
}

// One-sided Jacobi for narrow problems (c < 32 columns, X and V both in one
// CTA's shared memory): the reference algorithm (dense.cpp:585-686: columns
// re-ordered by descending norm before every sweep, rotation formula, skip
// rule |apq| <= 1e-15 sqrt(app aqq), <= 60 sweeps, D non-increasing) with the
// pairs of a sweep in circle-method rounds, one warp per pair and one CTA
// barrier per round: no cluster barriers, no global round trips. The sort is
// an index permutation (`ord`), never a data move. One problem per CTA
// (blockIdx.x picks p0 / p1).
struct J1Params {
  const double* X;
  int mr, c;
  double *U, *S, *V;
  int* info;
  int* sweeps_out;
};

__global__ void __launch_bounds__(1024, 1) jacobi1_kernel(const J1Params p0, const J1Params p1) {
  const J1Params& p = blockIdx.x == 0 ? p0 : p1;
  const int mr = p.mr, c = p.c, cc = c + (c & 1);  // cc: even count of positions (last one virtual if c odd)
  extern __shared__ double sm[];
  double* X = sm;                      // [c][mr]
  double* V = X + static_cast<size_t>(c) * mr;  // [c][c]
  double* nrm = V + static_cast<size_t>(c) * c;  // [c]
  int* ord = reinterpret_cast<int*>(nrm + c);   // [cc] position -> column
  __shared__ int s_rot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int e = tid; e < c * mr; e += blockDim.x) X[e] = p.X[e];
  for (int e = tid; e < c * c; e += blockDim.x) V[e] = (e % c == e / c) ? 1.0 : 0.0;
  if (tid < cc) ord[tid] = tid;
  __syncthreads();
  auto norms = [&]() {
    for (int j = warp; j < c; j += nwarps) {
      const double* x = X + static_cast<size_t>(j) * mr;
      double s2 = 0.0;
      for (int i = lane; i < mr; i += 32) s2 = fma(x[i], x[i], s2);
      s2 = warp_sum(s2);
      if (lane == 0) nrm[j] = s2;
    }
    __syncthreads();
  };
  // stable descending rank sort of the columns by nrm into ord (positions >= c stay virtual)
  auto sort_cols = [&]() {
    for (int j = tid; j < c; j += blockDim.x) {
      const double kj = nrm[j];
      int rank = 0;
      for (int i = 0; i < c; ++i) {
        const double ki = nrm[i];
        rank += (ki > kj || (ki == kj && i < j)) ? 1 : 0;
      }
      ord[rank] = j;
    }
    if (tid == 0 && cc > c) ord[c] = c;  // the virtual column
    __syncthreads();
  };
  int sweep = 0;
  bool conv = c <= 1;
  while (!conv && sweep < 60) {
    norms();
    sort_cols();
    if (tid == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < cc - 1; ++r) {
      for (int k = warp; k < cc / 2; k += nwarps) {
        int a, b;
        pair_of(r, k, cc, &a, &b);
        const int u = ord[a], v = ord[b];
        if (u >= c || v >= c) continue;
        double* xu = X + static_cast<size_t>(u) * mr;
        double* xv = X + static_cast<size_t>(v) * mr;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int i = lane; i < mr; i += 32) {
          const double x = xu[i], y = xv[i];
          app = fma(x, x, app);
          aqq = fma(y, y, aqq);
          apq = fma(x, y, apq);
        }
        app = warp_sum(app);
        aqq = warp_sum(aqq);
        apq = warp_sum(apq);
        // (u, v) are (p, q) of the reference in sorted position order: a < b
        if (app != 0.0 && aqq != 0.0 && !(apq * apq <= 1e-30 * (app * aqq))) {
          const double zeta = (aqq - app) / (2.0 * apq);
          const double t = (zeta < 0.0 ? -1.0 : 1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
          for (int i = lane; i < mr; i += 32) {
            const double x = xu[i], y = xv[i];
            xu[i] = cs * x - sn * y;
            xv[i] = sn * x + cs * y;
          }
          double* vu = V + static_cast<size_t>(u) * c;
          double* vv = V + static_cast<size_t>(v) * c;
          for (int i = lane; i < c; i += 32) {
            const double x = vu[i], y = vv[i];
            vu[i] = cs * x - sn * y;
            vv[i] = sn * x + cs * y;
          }
          if (lane == 0) s_rot = 1;
        }
      }
      __syncthreads();
    }
    conv = s_rot == 0;
    ++sweep;
    __syncthreads();
  }
  // singular values (column norms) in stable descending order, U = X / s, V permuted
  norms();
  for (int j = tid; j < c; j += blockDim.x) nrm[j] = sqrt(nrm[j]);
  __syncthreads();
  sort_cols();
  const double smax = c > 0 ? nrm[ord[0]] : 0.0;
  bool zero_cols = false;
  for (int j = 0; j < c; ++j) {
    const int src = ord[j];
    const double sv = nrm[src];
    const bool ok = sv > 0.0 && sv > smax * 1e-250;
    zero_cols |= !ok;
    if (tid == 0) p.S[j] = ok ? sv : 0.0;
    const double* x = X + static_cast<size_t>(src) * mr;
    for (int i = tid; i < mr; i += blockDim.x) p.U[static_cast<int64_t>(j) * mr + i] = ok ? x[i] / sv : 0.0;
    const double* vv = V + static_cast<size_t>(src) * c;
    for (int i = tid; i < c; i += blockDim.x) p.V[static_cast<int64_t>(j) * c + i] = vv[i];
  }
  if (tid == 0) {
    p.info[0] = conv ? (zero_cols ? 2 : 0) : 1;
    if (p.sweeps_out) p.sweeps_out[0] = sweep;
  }
}

size_t jacobi1_smem(int64_t mr, int64_t c) {
  return sizeof(double) * static_cast<size_t>(c) * (mr + c + 1) + sizeof(int) * static_cast<size_t>(c + 2);
}

// Block Jacobi applies when the two blocks' rows fit in shared memory and the
// tournament fits one cluster (<= 16 CTAs); RFGPU_JACOBI_BLOCK=0 disables it.
struct BJLayout {
  bool ok;
  int B, P, nb;
  size_t smem, work;  // bytes
};
BJLayout bj_layout(int64_t mr, int64_t c) {
  BJLayout L{};
  const char* e = std::getenv("RFGPU_JACOBI_BLOCK");
  if ((e && e[0] == '0') || c < 32 || mr > 1024) return L;
  for (int B : {8, 12, 16}) {
    if (e && std::atoi(e) > 1 && std::atoi(e) != B) continue;  // RFGPU_JACOBI_BLOCK=8/16 pins the width
    const int64_t blocks = (c + B - 1) / B;
    L.B = B;
    L.nb = static_cast<int>(blocks + (blocks & 1));
    L.P = L.nb / 2;
    L.smem = sizeof(double) * 2 * B * ((mr + (mr & 1)) + (c + (c & 1))) + 256;
    L.work = sizeof(double) * static_cast<size_t>(L.nb) * B * ((mr + (mr & 1)) + (c + (c & 1)));
    L.ok = L.P <= 16 && L.smem <= 220 * 1024;
    if (L.ok) return L;
  }
  L.ok = false;
  return L;
}

__global__ void sumsq_partial_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[32];
  double s = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride)
    s = fma(x[i], x[i], s);
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

struct JacobiLayout {
  int P, RX, RV, LDX, LDV, threads;
  bool smem;
  bool bcast;
  size_t bytes;
};

inline int pad_ld(int r) { return r + ((r % 2 == 0) ? 1 : 0); }  // odd leading dimension

JacobiLayout jacobi_layout(int64_t mr, int64_t c) {
  const int64_t cc = c + (c & 1), npairs = cc / 2;
  const int64_t G = (npairs + 31) / 32;
  // Row groups per pair: enough warps to keep ~8 rows each. More groups make
  // the rows/warp loop shorter but the serial per-pair reduction over groups
  // longer; both sit on every round's critical path.
  constexpr int rpw = 8;  // (measured best at l = 60 ... 330)
  auto groups = [&](int64_t rows) { return std::max<int64_t>(1, std::min<int64_t>(32 / G, (rows + rpw - 1) / rpw)); };
  auto extra = [&](int P, bool bcast) {
    const int64_t H = groups((mr + P - 1) / P);
    const int64_t npo = bcast ? npairs : (npairs + P - 1) / P;
    const int64_t blk3 = (npo * 3 + 1) & ~int64_t(1);
    return sizeof(double) * (4 + 4 * P * npo + 4 * npo + 4 * P * blk3 + std::max<int64_t>(H * npairs * 3, P * cc) +
                             cc) +
           sizeof(int) * cc + 64;
  };
  constexpr size_t kMax = 224 * 1024;
  // Smallest cluster that leaves at most `target` rows of X per CTA: the
  // per-round shared-memory traffic of a CTA is proportional to its rows.
  constexpr int target = 32;
  int P0 = 1;
  while (P0 < 16 && (mr + P0 - 1) / P0 > target) P0 *= 2;
  for (bool bcast : {true, false}) {
    for (int P : {1, 2, 4, 8, 16}) {
      if (P < P0) continue;
      const int RX = static_cast<int>((mr + P - 1) / P), RV = static_cast<int>((c + P - 1) / P);
      const int LDX = pad_ld(RX), LDV = pad_ld(RV);
      const size_t b = sizeof(double) * static_cast<size_t>(c) * (LDX + LDV) + extra(P, bcast);
      if (b <= kMax) return {P, RX, RV, LDX, LDV, static_cast<int>(32 * G * groups(RX)), true, bcast, b};
    }
  }
  const int P = 8;
  const int RX = static_cast<int>((mr + P - 1) / P), RV = static_cast<int>((c + P - 1) / P);
  return {P, RX, RV, pad_ld(RX), pad_ld(RV), static_cast<int>(32 * G * groups(RX)), false, false, extra(P, false)};
}

}  // namespace

size_t chol_inv_work_bytes(int64_t c) { return sizeof(double) * (2 * c + c * (c + 1) / 2); }
namespace {
size_t chol_smem_bytes(int64_t c) { return sizeof(double) * (2 * c + c * (c + 1) / 2); }
}  // namespace

namespace {
// ---- blocked Cholesky for l > 256 (the packed triangle no longer fits in
// one CTA's shared memory): right-looking with kCB-wide panels, R doubling as
// the working copy of G (32-wide panels). Per panel: the diagonal block is factored in shared
// memory by one CTA (reference pivot rule, dense.cpp:763-786) and inverted;
// the block row R(k, k1:) = R_kk^-T G(k, k1:) and the trailing update
// G(k1:, k1:) -= R(k, k1:)^T R(k, k1:) run over many CTAs.
constexpr int kCB = 32;

__global__ void cholb_prep(const double* __restrict__ G, int c, double* __restrict__ R, double* __restrict__ stat,
                           int* info, double* info_d) {
  const int64_t cc = static_cast<int64_t>(c) * c;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < cc;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / c, i = e - j * c;
    R[e] = i <= j ? G[e] : 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double mx = 0.0, tr = 0.0;
    for (int j = 0; j < c; ++j) {
      const double g = G[static_cast<int64_t>(j) * c + j];
      mx = fmax(mx, fabs(g));
      tr += g;
    }
    stat[0] = 1e-14 * mx;
    stat[1] = tr;
    info[0] = 0;
    info_d[0] = INFINITY;
  }
}

__global__ void __launch_bounds__(256) cholb_diag(double* __restrict__ R, int c, int k0, int k1,
                                                  const double* __restrict__ stat, double* __restrict__ Dinv, int* info,
                                                  double* info_d) {
  if (info[0]) return;
  __shared__ double A[kCB][kCB + 1];  // A[col][row]
  __shared__ double X[kCB][kCB + 1];  // inverse, X[col][row]
  __shared__ int s_fail;
  __shared__ double s_min;
  const int b = k1 - k0, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int j = e / b, i = e - j * b;
    A[j][i] = i <= j ? R[static_cast<int64_t>(k0 + j) * c + k0 + i] : 0.0;
  }
  if (tid == 0) {
    s_fail = 0;
    s_min = info_d[0];
  }
  __syncthreads();
  const double floor = stat[0], trace = stat[1];
  // factor the diagonal block: every thread reads the pivot, row j is scaled
  // by warp 0, the trailing columns are updated by the 8 warps (column col by
  // warp col % 8, lane = row), two barriers per step
  for (int j = 0; j < b; ++j) {
    const double d = A[j][j];
    if (d <= floor || !(d > 0.0)) {  // every thread sees the same pivot
      if (tid == 0) s_fail = k0 + j + 1;
      break;
    }
    const double cjj = sqrt(d);
    if (warp == 0) {
      if (lane == 0) s_min = fmin(s_min, trace > 0.0 ? d / trace : 0.0);
      if (lane > j && lane < b) A[lane][j] /= cjj;  // row j of R: column `lane`
    }
    __syncthreads();
    if (tid == 0) A[j][j] = cjj;
    for (int col = j + 1 + warp; col < b; col += 8) {
      const double rc = A[col][j];
      if (lane > j && lane <= col) A[col][lane] = fma(-A[lane][j], rc, A[col][lane]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0) {
      info[0] = s_fail;
      info_d[0] = s_min;
    }
    return;
  }
  // R_kk^{-1} (upper), one warp per column j: back substitution with x over
  // the lanes (lane r holds x_r), one shuffle per step
  __shared__ double rdg[kCB];
  if (tid < b) rdg[tid] = 1.0 / A[tid][tid];
  __syncthreads();
  for (int j = warp; j < b; j += 8) {
    double x = (lane == j) ? 1.0 : 0.0;
    for (int i = j; i >= 0; --i) {
      const double xi = __shfl_sync(0xffffffffu, x, i) * rdg[i];
      if (lane == i) x = xi;
      else if (lane < i) x = fma(-xi, A[i][lane], x);
    }
    X[j][lane] = lane <= j ? x : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int j = e / b, i = e - j * b;
    R[static_cast<int64_t>(k0 + j) * c + k0 + i] = i <= j ? A[j][i] : 0.0;
    Dinv[j * kCB + i] = X[j][i];
  }
  if (tid == 0) info_d[0] = s_min;
}

// R(k0:k1, j) = R_kk^-T W(k0:k1, j) for 32 columns j per CTA.
__global__ void __launch_bounds__(256) cholb_panel(double* __restrict__ R, int c, int k0, int k1,
                                                   const double* __restrict__ Dinv, const int* info) {
  if (info[0]) return;
  __shared__ double D[kCB][kCB + 1];   // D[col][row] = Dinv
  __shared__ double W[32][kCB + 1];    // W[col][row]
  const int b = k1 - k0, tid = threadIdx.x;
  const int j0 = k1 + blockIdx.x * 32, nj = min(32, c - j0);
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int j = e / b, i = e - j * b;
    D[j][i] = Dinv[j * kCB + i];
  }
  for (int e = tid; e < b * nj; e += blockDim.x) {
    const int jj = e / b, i = e - jj * b;
    W[jj][i] = R[static_cast<int64_t>(j0 + jj) * c + k0 + i];
  }
  __syncthreads();
  for (int e = tid; e < b * nj; e += blockDim.x) {
    const int jj = e / b, i = e - jj * b;
    // (Dinv^T W)(i, jj) = sum_t Dinv(t, i) W(t, jj), Dinv upper: t <= i
    double acc = 0.0;
    for (int t = 0; t <= i; ++t) acc = fma(D[i][t], W[jj][t], acc);
    R[static_cast<int64_t>(j0 + jj) * c + k0 + i] = acc;
  }
}

// W(i, j) -= sum_t R(t, i) R(t, j), t in the panel, for k1 <= i <= j: 32 x 32 tiles.
__global__ void __launch_bounds__(256) cholb_update(double* __restrict__ R, int c, int k0, int k1, int ntile,
                                                    const int* info) {
  if (info[0]) return;
  // upper-triangular tile index -> (ti, tj), ti <= tj
  int t = blockIdx.x, ti = 0;
  while (t >= ntile - ti) {
    t -= ntile - ti;
    ++ti;
  }
  const int tj = ti + t;
  __shared__ double Xi[32][kCB + 1], Xj[32][kCB + 1];  // [col][t]
  const int b = k1 - k0, tid = threadIdx.x;
  const int i0 = k1 + ti * 32, j0 = k1 + tj * 32;
  const int ni = min(32, c - i0), nj = min(32, c - j0);
  for (int e = tid; e < b * 32; e += blockDim.x) {
    const int col = e / b, r = e - col * b;
    Xi[col][r] = col < ni ? R[static_cast<int64_t>(i0 + col) * c + k0 + r] : 0.0;
    Xj[col][r] = col < nj ? R[static_cast<int64_t>(j0 + col) * c + k0 + r] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int jj = e >> 5, ii = e & 31;
    const int i = i0 + ii, j = j0 + jj;
    if (ii < ni && jj < nj && i <= j) {
      double acc = 0.0;
      for (int r = 0; r < b; ++r) acc = fma(Xi[ii][r], Xj[jj][r], acc);
      R[static_cast<int64_t>(j) * c + i] -= acc;
    }
  }
}

cudaError_t chol_blocked(const double* G, int c, double* R, double* work, int* info, double* info_d, cudaStream_t st) {
  double* stat = work;          // floor, trace
  double* Dinv = work + 16;     // kCB x kCB
  cholb_prep<<<static_cast<unsigned>(std::min<int64_t>((static_cast<int64_t>(c) * c + 255) / 256, 592)), 256, 0, st>>>(
      G, c, R, stat, info, info_d);
  count_launch();
  for (int k0 = 0; k0 < c; k0 += kCB) {
    const int k1 = std::min(c, k0 + kCB);
    cholb_diag<<<1, 256, 0, st>>>(R, c, k0, k1, stat, Dinv, info, info_d);
    count_launch();
    if (k1 < c) {
      cholb_panel<<<static_cast<unsigned>((c - k1 + 31) / 32), 256, 0, st>>>(R, c, k0, k1, Dinv, info);
      const int ntile = (c - k1 + 31) / 32;
      cholb_update<<<static_cast<unsigned>(ntile * (ntile + 1) / 2), 256, 0, st>>>(R, c, k0, k1, ntile, info);
      count_launch(2);
    }
  }
  return cudaGetLastError();
}
}  // namespace

cudaError_t chol_inv(const double* G, int64_t c, double* R, double* Rinv, double* work, int* info,
                     double* info_d, cudaStream_t st) {
  if (c <= 0) return cudaSuccess;
  if (c > kMaxSmallFactor) return cudaErrorInvalidValue;  // callers check (rfgpu_max_sketch_width)
  const size_t smem = chol_smem_bytes(c);
  const int ci = static_cast<int>(c);
  if (smem <= 224 * 1024 && c <= 256) {
    static std::atomic<uint64_t> cfg{0};
    if (attr_pending(cfg)) {
      for (const void* fn : {reinterpret_cast<const void*>(chol_kernel), reinterpret_cast<const void*>(trinv_smem_kernel<8>)}) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
        if (e != cudaSuccess) return e;
      }
      attr_done(cfg);
    }
    double* rdiag = work;  // c doubles
    // (256 / 512 threads for l <= 64 / 128 measured slower: config 1's 8 Choleskys 0.33 -> 0.44 ms)
    const size_t rsm = sizeof(double) * 3 * c;
    if (ci <= 32)
      chol_reg_kernel<1><<<1, kSmallThreads, rsm, st>>>(G, ci, R, rdiag, info, info_d);
    else if (ci <= 64)
      chol_reg_kernel<2><<<1, kSmallThreads, rsm, st>>>(G, ci, R, rdiag, info, info_d);
    else if (ci <= 96)
      chol_reg_kernel<3><<<1, kSmallThreads, rsm, st>>>(G, ci, R, rdiag, info, info_d);
    else if (ci <= 128)
      chol_reg_kernel<4><<<1, kSmallThreads, rsm, st>>>(G, ci, R, rdiag, info, info_d);
    else
      chol_kernel<<<1, kSmallThreads, smem, st>>>(G, ci, R, rdiag, info, info_d);
    trinv_smem_kernel<8><<<(ci + 31) / 32, kSmallThreads, sizeof(double) * c * (c + 1) / 2, st>>>(R, ci, rdiag, Rinv);
    count_launch(2);
    return cudaGetLastError();
  }
  cudaError_t e = chol_blocked(G, ci, R, work, info, info_d, st);
  if (e != cudaSuccess) return e;
  return trinv_upper(R, c, ci, Rinv, st);
}

size_t jacobi_work_bytes(int64_t mr, int64_t c) {
  const JacobiLayout L = jacobi_layout(mr, c);
  const size_t stage = sizeof(double) * static_cast<size_t>(L.P) * c * (L.LDX + L.LDV);
  const BJLayout B = bj_layout(mr, c);
  return std::max(L.smem ? stage : 2 * stage, B.ok ? B.work : size_t(0));
}

namespace {
// One launch for 1 or 2 same-shape problems (one cluster each).
cudaError_t bjacobi_launch(const JacobiProblem* pr, int count, int64_t mr, int64_t c, const BJLayout& B,
                           cudaStream_t st) {
  BJParams ps[2];
  for (int i = 0; i < count; ++i) {
    ps[i] = BJParams{pr[i].X, static_cast<int>(mr), static_cast<int>(c), B.nb, /*cross_only=*/1,
                     pr[i].U, pr[i].S, pr[i].V,
                     pr[i].work, pr[i].work + static_cast<size_t>(B.nb) * B.B * (mr + (mr & 1)), pr[i].info,
                     pr[i].sweeps};
  }
  if (count == 1) ps[1] = ps[0];
  static std::atomic<uint64_t> cfg_done{0};
  if (attr_pending(cfg_done)) {
    for (const void* fn : {reinterpret_cast<const void*>(bjacobi_kernel<8>), reinterpret_cast<const void*>(bjacobi_kernel<12>),
                           reinterpret_cast<const void*>(bjacobi_kernel<16>)}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    attr_done(cfg_done);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(B.P * count);
  cfg.blockDim = dim3(32 * B.B);
  cfg.dynamicSmemBytes = B.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = B.P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = B.B == 8    ? cudaLaunchKernelEx(&cfg, bjacobi_kernel<8>, ps[0], ps[1])
                  : B.B == 12 ? cudaLaunchKernelEx(&cfg, bjacobi_kernel<12>, ps[0], ps[1])
                              : cudaLaunchKernelEx(&cfg, bjacobi_kernel<16>, ps[0], ps[1]);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t jacobi_launch(const JacobiProblem* pr, int count, int64_t mr, int64_t c, cudaStream_t st,
                          bool sorted = false) {
  if (c <= 0 || mr <= 0) return cudaSuccess;
  // narrow problems (c < 32, below the block kernel's range): the single-CTA kernel. (Measured for
  // 32 <= c <= 128 too, but there the cluster block kernel is faster: l = 60 0.81 vs 0.62 ms, l = 110 3.4 vs
  // 1.2 ms — a round's rotation chain costs the same, and the block kernel's CTAs are smaller.)
  if (c < 32 && jacobi1_smem(mr, c) <= 220 * 1024) {
    static std::atomic<uint64_t> j1cfg{0};
    if (attr_pending(j1cfg)) {
      cudaError_t e = cudaFuncSetAttribute(jacobi1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      if (e != cudaSuccess) {
        cudaGetLastError();
        return e;
      }
      attr_done(j1cfg);
    }
    J1Params ps[2];
    for (int i = 0; i < count; ++i)
      ps[i] = J1Params{pr[i].X, static_cast<int>(mr), static_cast<int>(c), pr[i].U, pr[i].S, pr[i].V, pr[i].info,
                       pr[i].sweeps};
    if (count == 1) ps[1] = ps[0];
    const int pairs = static_cast<int>((c + (c & 1)) / 2);
    const int threads = 32 * std::max(1, std::min(32, pairs));
    jacobi1_kernel<<<count, threads, jacobi1_smem(mr, c), st>>>(ps[0], ps[1]);
    count_launch();
    return cudaGetLastError();
  }
  const BJLayout B = bj_layout(mr, c);
  if (B.ok && !sorted) return bjacobi_launch(pr, count, mr, c, B, st);
  const JacobiLayout L = jacobi_layout(mr, c);
  JacobiParams ps[2];
  for (int i = 0; i < count; ++i) {
    JacobiParams& p = ps[i];
    p = JacobiParams{};
    p.X = pr[i].X;
    p.mr = mr;
    p.c = static_cast<int>(c);
    p.U = pr[i].U;
    p.S = pr[i].S;
    p.V = pr[i].V;
    p.RX = L.RX;
    p.RV = L.RV;
    p.LDX = L.LDX;
    p.LDV = L.LDV;
    p.bcast = L.bcast ? 1 : 0;
    p.info = pr[i].info;
    p.sweeps_out = pr[i].sweeps;
#ifdef RFGPU_JACOBI_TRACE
    static long long* trace_buf = nullptr;
    if (!trace_buf) cudaMalloc(&trace_buf, sizeof(long long) * 16);
    p.trace = trace_buf;
#endif
    const size_t stage = static_cast<size_t>(L.P) * c * (L.LDX + L.LDV);
    p.gS = pr[i].work;
    if (!L.smem) {
      p.gX = pr[i].work + stage;
      p.gV = p.gX + static_cast<size_t>(L.P) * c * L.LDX;
    }
  }
  if (count == 1) ps[1] = ps[0];
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(L.P * count);
  cfg.blockDim = dim3(L.threads);
  cfg.dynamicSmemBytes = L.bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = L.P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // kernel attributes once per device, at the device's opt-in shared-memory maximum (the layout never
  // asks for more), so every context on every device launches with them set
  static std::atomic<uint64_t> attr_cfg{0};
  if (attr_pending(attr_cfg)) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    for (const void* fn : {reinterpret_cast<const void*>(jacobi_svd_kernel<true>),
                           reinterpret_cast<const void*>(jacobi_svd_kernel<false>)}) {
      cudaFuncAttributes fa{};
      cudaError_t ea = cudaFuncGetAttributes(&fa, fn);  // dynamic + static shared memory <= the opt-in maximum
      if (ea == cudaSuccess)
        ea = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  optin - static_cast<int>(fa.sharedSizeBytes));
      if (ea == cudaSuccess) ea = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (ea != cudaSuccess) {
        cudaGetLastError();
        return ea;
      }
    }
    attr_done(attr_cfg);
  }
  cudaError_t e = L.smem ? cudaLaunchKernelEx(&cfg, jacobi_svd_kernel<true>, ps[0], ps[1])
                         : cudaLaunchKernelEx(&cfg, jacobi_svd_kernel<false>, ps[0], ps[1]);
  count_launch();
  if (e != cudaSuccess) return e;
#ifdef RFGPU_JACOBI_TRACE
  {
    long long h[14];
    cudaStreamSynchronize(st);
    cudaMemcpy(h, ps[0].trace, sizeof(h), cudaMemcpyDeviceToHost);
    std::fprintf(stderr, "[rfgpu] jacobi c=%lld P=%d bcast=%d slots (clk/round):", static_cast<long long>(c), L.P,
                 static_cast<int>(L.bcast));
    for (int k = 1; k < 14; ++k) std::fprintf(stderr, " %d:%.0f", k, static_cast<double>(h[k]) / 30);
    std::fprintf(stderr, " next:%.0f\n", static_cast<double>(h[0]) / 30);
  }
#endif
  return cudaGetLastError();
}
}  // namespace

cudaError_t jacobi_svd(const double* X, int64_t mr, int64_t c, double* U, double* S, double* V, double* work,
                       int* info, int* sweeps_out, cudaStream_t st, bool sorted) {
  const JacobiProblem p{X, U, S, V, work, info, sweeps_out};
  return jacobi_launch(&p, 1, mr, c, st, sorted);
}

cudaError_t jacobi_svd_pair(const JacobiProblem& a, const JacobiProblem& b, int64_t mr, int64_t c, cudaStream_t st) {
  const JacobiProblem p[2] = {a, b};
  return jacobi_launch(p, 2, mr, c, st);
}

cudaError_t sumsq(const double* x, int64_t n, double* partials, double* out, cudaStream_t st) {
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(592, (n + 1023) / 1024)));
  sumsq_partial_kernel<<<blocks, 1024, 0, st>>>(x, n, partials);
    count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return sum_array(partials, blocks, out, st);
}

}  // namespace rfgpu
