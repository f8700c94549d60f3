// Column-pivoted Householder QR with the reference's greedy pivot rule, and
// the interpolative-decomposition pieces built on it.
//
//  * cpqr_rank   cpqr(Y, CpqrStop::rank(k)) of proj/src/dense.cpp:453-552:
//                pivot = FIRST column attaining the largest down-dated norm
//                (strict > scan from best = -1), exact recompute when the
//                winner fell below 1e-8 of its original norm, halt when
//                sqrt(best) < 1e-14 ||Y||_F, non-negative R diagonal
//                (make_reflector, dense.cpp:328-357). One persistent
//                cooperative kernel; each CTA owns a contiguous block of
//                columns, two grid barriers per step (argmax, then swap +
//                reflector application), the ell x n sketch stays in L2.
//  * trinv_upper R^{-1} of an upper-triangular k x k factor (warp per column).
//  * assemble_z  Z(:, Js) = I, Z(:, perm(k:)) = T (col_id_core, lowrank.cpp:51-70).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "rfgpu_internal.h"

namespace cg = cooperative_groups;

namespace rfgpu {

namespace {

constexpr int kCpqrThreads = 384;
constexpr int kMaxRows = 512;  // sketch height (k + p) supported by the kernel

struct CpqrParams {
  double* W;  // m x n, column-major, ld
  int64_t ld;
  int m;
  int64_t n;
  int kmax;           // rank stop
  double halt;        // 1e-14 ||Y||_F
  double* norms2;     // [n]
  double* norms0;     // [n]
  int64_t* perm;      // [n]
  // per-step staging (double-buffered by step parity): every CTA publishes
  // its local winner (value, index, perm, norm0, the column itself); the
  // owner of slot r publishes column r. Readers never touch W columns that
  // their owners are rewriting in the same phase.
  double* part_val;   // [2][grid]
  int64_t* part_idx;  // [2][grid]
  int64_t* part_perm; // [2][grid]
  double* part_n0;    // [2][grid]
  double* stage_col;  // [2][grid][m]
  double* stage_r;    // [2][m + 4]: column r, then perm, norms2, norms0
  int* stopped;       // [1] stopped rank
  int* recomputes;    // [1]
};

__device__ __forceinline__ void better(double& bv, int64_t& bi, double v, int64_t i) {
  // "first index attaining the maximum": strictly larger value, or equal value
  // at a smaller index (a total order, so the combine order does not matter).
  if (v > bv || (v == bv && i < bi)) {
    bv = v;
    bi = i;
  }
}

template <int S>
__global__ void __launch_bounds__(kCpqrThreads, 1) cpqr_kernel(const CpqrParams p) {
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int64_t cpb = (p.n + G - 1) / G;
  const int64_t c0 = lmin(p.n, b * cpb), c1 = lmin(p.n, c0 + cpb);
  const int m = p.m;
  const int rmax = static_cast<int>(lmin(lmin(m, p.n), p.kmax));

  __shared__ double colP[kMaxRows], colR[kMaxRows], tail[kMaxRows];
  __shared__ double s_val[32];
  __shared__ int64_t s_idx[32];
  __shared__ double s_beta, s_result, s_best, s_n2r, s_n0r, s_n0p;
  __shared__ int64_t s_piv, s_perm_piv, s_perm_r;
  __shared__ int s_stop, s_recompute;

  auto owner = [&](int64_t c) { return static_cast<int>(c / cpb); };

  // Local winner over owned columns c >= r; published with a copy of the
  // winning column into buffer `buf`. Slot r's owner also stages column r.
  auto publish = [&](int r, int buf) {
    double bv = -1.0;
    int64_t bi = r;
    for (int64_t c = lmax(c0, r) + tid; c < c1; c += blockDim.x) {
      const double v = p.norms2[c];
      if (v > bv) {
        bv = v;
        bi = c;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      better(bv, bi, ov, oi);
    }
    if (lane == 0) {
      s_val[warp] = bv;
      s_idx[warp] = bi;
    }
    __syncthreads();
    if (warp == 0) {
      double v = -1.0;
      int64_t i = r;
      for (int w = lane; w < nwarps; w += 32) better(v, i, s_val[w], s_idx[w]);
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
        better(v, i, ov, oi);
      }
      if (lane == 0) {
        s_val[0] = v;
        s_idx[0] = i;
      }
    }
    __syncthreads();
    const int64_t wi = s_idx[0];
    if (tid == 0) {
      p.part_val[buf * G + b] = s_val[0];
      p.part_idx[buf * G + b] = wi;
      const bool mine = wi >= c0 && wi < c1;
      p.part_perm[buf * G + b] = mine ? p.perm[wi] : -1;
      p.part_n0[buf * G + b] = mine ? p.norms0[wi] : 0.0;
    }
    if (wi >= c0 && wi < c1) {
      const double* src = p.W + wi * p.ld;
      double* dst = p.stage_col + (static_cast<int64_t>(buf) * G + b) * m;
      for (int i = tid; i < m; i += blockDim.x) dst[i] = src[i];
    }
    if (r < p.n && r >= c0 && r < c1) {
      const double* src = p.W + static_cast<int64_t>(r) * p.ld;
      double* dst = p.stage_r + static_cast<int64_t>(buf) * (m + 4);
      for (int i = tid; i < m; i += blockDim.x) dst[i] = src[i];
      if (tid == 0) {
        dst[m] = static_cast<double>(p.perm[r]);
        dst[m + 1] = p.norms2[r];
        dst[m + 2] = p.norms0[r];
      }
    }
  };
  auto global_winner = [&](int r, int buf) {
    if (warp == 0) {
      double v = -1.0;
      int64_t i = r;
      for (int g = lane; g < G; g += 32) better(v, i, __ldcg(p.part_val + buf * G + g), __ldcg(p.part_idx + buf * G + g));
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
        better(v, i, ov, oi);
      }
      if (lane == 0) {
        s_best = v;
        s_piv = i;
        const int w = owner(i);
        s_n0p = __ldcg(p.part_n0 + buf * G + w);
        s_perm_piv = __ldcg(p.part_perm + buf * G + w);
      }
    }
    __syncthreads();
  };

  // initial norms (dense.cpp:466-471) and identity permutation
  for (int64_t c = c0 + warp; c < c1; c += nwarps) {
    const double* col = p.W + c * p.ld;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s = fma(col[i], col[i], s);
    s = warp_sum(s);
    if (lane == 0) {
      p.norms2[c] = s;
      p.norms0[c] = s;
      p.perm[c] = c;
    }
  }
  __syncthreads();
  if (rmax > 0) publish(0, 0);
  grid.sync();

  constexpr int SMAX = S;
  int r = 0;
  for (; r < rmax; ++r) {
    const int buf = r & 1;
    global_winner(r, buf);
    if (tid == 0) s_recompute = (s_best <= 0.0 || s_best < 1e-8 * s_n0p) ? 1 : 0;
    __syncthreads();
    if (s_recompute) {
      // exact recompute of the trailing norms (dense.cpp:503-518)
      if (b == 0 && tid == 0) atomicAdd(p.recomputes, 1);
      grid.sync();  // everyone has read the stale winners
      for (int64_t c = lmax(c0, r) + warp; c < c1; c += nwarps) {
        const double* col = p.W + c * p.ld;
        double s = 0.0;
        for (int i = r + lane; i < m; i += 32) s = fma(col[i], col[i], s);
        s = warp_sum(s);
        if (lane == 0) p.norms2[c] = s;
      }
      __syncthreads();
      publish(r, buf);
      grid.sync();
      global_winner(r, buf);
    }
    if (tid == 0) s_stop = sqrt(fmax(0.0, s_best)) < p.halt ? 1 : 0;  // numerically exhausted
    __syncthreads();
    if (s_stop) break;
    const int64_t piv = s_piv;
    {
      const double* sp = p.stage_col + (static_cast<int64_t>(buf) * G + owner(piv)) * m;
      const double* sr = p.stage_r + static_cast<int64_t>(buf) * (m + 4);
      for (int i = tid; i < m; i += blockDim.x) {
        colP[i] = __ldcg(sp + i);
        colR[i] = __ldcg(sr + i);
      }
      if (tid == 0) {
        s_perm_r = static_cast<int64_t>(__ldcg(sr + m));
        s_n2r = __ldcg(sr + m + 1);
        s_n0r = __ldcg(sr + m + 2);
      }
    }
    __syncthreads();
    // reflector for x = colP[r:m) (make_reflector, dense.cpp:328-357)
    {
      double sg = 0.0;
      for (int i = r + 1 + tid; i < m; i += blockDim.x) sg = fma(colP[i], colP[i], sg);
      __shared__ double red[32];
      const double sigma = block_sum(sg, red);
      const double alpha = colP[r];
      double beta, result, v0 = 1.0;
      if (sigma == 0.0) {
        beta = alpha >= 0.0 ? 0.0 : 2.0;
        result = fabs(alpha);
      } else {
        const double mu = sqrt(alpha * alpha + sigma);
        v0 = (alpha <= 0.0) ? alpha - mu : -sigma / (alpha + mu);
        beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
        result = mu;
      }
      for (int i = r + 1 + tid; i < m; i += blockDim.x) tail[i] = sigma == 0.0 ? 0.0 : colP[i] / v0;
      if (tid == 0) {
        s_beta = beta;
        s_result = result;
      }
    }
    __syncthreads();
    const double beta = s_beta;
    // apply (I - beta v v^T), v = [1; tail], to owned columns c >= r with the swap
    auto slow_column = [&](int64_t c) {
      double* col = p.W + c * p.ld;
      if (c == r) {
        for (int i = lane; i < m; i += 32) col[i] = (i < r) ? colP[i] : (i == r ? s_result : 0.0);
        if (lane == 0) {
          p.perm[r] = s_perm_piv;
          p.norms2[r] = s_best;
          p.norms0[r] = s_n0p;
        }
        return;
      }
      // c == piv: slot piv receives the old column r
      double dot = 0.0;
      for (int i = r + 1 + lane; i < m; i += 32) dot = fma(tail[i], colR[i], dot);
      dot = warp_sum(dot) + colR[r];
      const double bd = beta * dot;
      for (int i = lane; i < m; i += 32) {
        double v = colR[i];
        if (beta != 0.0) {
          if (i == r) v -= bd;
          else if (i > r) v -= bd * tail[i];
        }
        col[i] = v;
      }
      __syncwarp();
      if (lane == 0) {
        const double wr = col[r];
        p.perm[c] = s_perm_r;
        p.norms0[c] = s_n0r;
        p.norms2[c] = s_n2r - wr * wr;  // down-date (dense.cpp:531-533)
      }
    };
    const int lr = r & 31;
    // Reflector in registers: t[s] = v_i for row i = lane + 32 s (v_r = 1,
    // rows above r zero), so the dot and the update are plain FMAs.
    double t[SMAX];
#pragma unroll
    for (int s = 0; s < SMAX; ++s) {
      const int i = lane + 32 * s;
      t[s] = (i < r || i >= m) ? 0.0 : (i == r ? 1.0 : tail[i]);
    }
    const int sfirst = r >> 5;  // slots entirely above row r are skipped (warp-uniform)
    const int64_t cstart = lmax(c0, r);
    constexpr int NC = SMAX <= 8 ? 4 : (SMAX <= 12 ? 3 : 2);  // columns per warp in flight
    for (int64_t cb = cstart + NC * warp; cb < c1; cb += NC * nwarps) {
      bool special = false;
#pragma unroll
      for (int u = 0; u < NC; ++u) special |= (cb + u < c1) && (cb + u == r || cb + u == piv);
      if (special) {
        for (int u = 0; u < NC; ++u) {
          const int64_t c = cb + u;
          if (c >= c1) break;
          if (c == r || c == piv) {
            slow_column(c);
            continue;
          }
          double* col = p.W + c * p.ld;  // ordinary column next to a special one
          double dot = 0.0;
          for (int i = r + 1 + lane; i < m; i += 32) dot = fma(tail[i], col[i], dot);
          dot = warp_sum(dot) + col[r];
          const double bd = beta * dot;
          if (beta != 0.0)
            for (int i = r + lane; i < m; i += 32) col[i] = (i == r) ? col[i] - bd : col[i] - bd * tail[i];
          __syncwarp();
          if (lane == 0) {
            const double wr = col[r];
            p.norms2[c] -= wr * wr;
          }
        }
        continue;
      }
      double x[NC][SMAX];
      double* pc[NC];
      bool live[NC];
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        live[u] = cb + u < c1;
        pc[u] = p.W + (live[u] ? cb + u : cb) * p.ld;
      }
#pragma unroll
      for (int s = 0; s < SMAX; ++s) {
        const int i = lane + 32 * s;
        const bool in = s >= sfirst && i >= r && i < m;
#pragma unroll
        for (int u = 0; u < NC; ++u) x[u][s] = in ? pc[u][i] : 0.0;
      }
      double d[NC], xr[NC], n2[NC];
#pragma unroll
      for (int u = 0; u < NC; ++u) {
        d[u] = 0.0;
        xr[u] = 0.0;
        n2[u] = (lane == lr && live[u]) ? p.norms2[cb + u] : 0.0;  // prefetched with the column loads
      }
#pragma unroll
      for (int s = 0; s < SMAX; ++s) {
        if (s < sfirst) continue;
#pragma unroll
        for (int u = 0; u < NC; ++u) d[u] = fma(t[s], x[u][s], d[u]);
      }
#pragma unroll
      for (int u = 0; u < NC; ++u) d[u] = warp_sum(d[u]) * beta;
      if (beta != 0.0) {
#pragma unroll
        for (int s = 0; s < SMAX; ++s) {
          if (s < sfirst) continue;
          const int i = lane + 32 * s;
          const bool in = i >= r && i < m;
#pragma unroll
          for (int u = 0; u < NC; ++u) {
            x[u][s] = fma(-d[u], t[s], x[u][s]);
            if (in && live[u]) pc[u][i] = x[u][s];
          }
        }
      }
      // down-date with the new row-r entries (owned by lane r & 31, slot r >> 5)
#pragma unroll
      for (int s = 0; s < SMAX; ++s)
        if (s == sfirst)
#pragma unroll
          for (int u = 0; u < NC; ++u) xr[u] = x[u][s];
      if (lane == lr) {
#pragma unroll
        for (int u = 0; u < NC; ++u)
          if (live[u]) p.norms2[cb + u] = n2[u] - xr[u] * xr[u];
      }
    }
    __syncthreads();
    if (r + 1 < rmax) publish(r + 1, buf ^ 1);
    grid.sync();
  }
  if (b == 0 && tid == 0) p.stopped[0] = r;
}

// R^{-1} of the leading k x k upper triangle of R (ld ldr): warp per column,
// back substitution R x = e_j in axpy form, x in the lanes' registers.
template <int S>
__global__ void trinv_upper_kernel(const double* __restrict__ R, int64_t ldr, int k, double* __restrict__ Rinv) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= k) return;
  double x[S];
#pragma unroll
  for (int s = 0; s < S; ++s) x[s] = (lane + 32 * s == j) ? 1.0 : 0.0;
  for (int i = j; i >= 0; --i) {
    const int si = i >> 5;
    double v = 0.0;
#pragma unroll
    for (int s = 0; s < S; ++s)
      if (s == si) v = x[s];
    const double* ri = R + static_cast<int64_t>(i) * ldr;
    const double xi = __shfl_sync(0xffffffffu, v, i & 31) / ri[i];
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int r = lane + 32 * s;
      if (r == i) x[s] = xi;
      else if (r < i) x[s] = fma(-xi, ri[r], x[s]);
    }
  }
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const int r = lane + 32 * s;
    if (r < k) Rinv[static_cast<int64_t>(j) * k + r] = r <= j ? x[s] : 0.0;
  }
}

// Blocked R^{-1} (k > 64): 32 x 32 diagonal blocks D_I = R_II^{-1} first (one
// CTA each, warp-parallel back substitution per column with precomputed
// reciprocal pivots), then one CTA per block column J:
//   X_JJ = D_J,  X_IJ = -D_I sum_{K=I+1..J} R_IK X_KJ  for I = J-1 .. 0,
// the X_KJ blocks of the column held in shared memory. Every dependency chain
// is 32 steps long instead of k (the per-column trinv_upper_kernel reads R
// from global memory in a k-step chain).
constexpr int kTB = 32;

__global__ void __launch_bounds__(256) trinv_diag_kernel(const double* __restrict__ R, int64_t ldr, int k,
                                                         double* __restrict__ Dinv) {
  __shared__ double A[kTB][kTB + 1];  // A[col][row]
  __shared__ double rd[kTB];
  const int I = blockIdx.x, i0 = I * kTB, bw = min(kTB, k - i0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < kTB * kTB; e += blockDim.x) {
    const int c = e / kTB, r = e % kTB;
    A[c][r] = (c < bw && r <= c) ? R[static_cast<int64_t>(i0 + c) * ldr + i0 + r] : 0.0;
  }
  __syncthreads();
  if (tid < kTB) rd[tid] = tid < bw ? 1.0 / A[tid][tid] : 0.0;
  __syncthreads();
  for (int j = warp; j < kTB; j += 8) {
    double x = (lane == j && j < bw) ? 1.0 : 0.0;
    if (j < bw)
      for (int i = j; i >= 0; --i) {
        const double xi = __shfl_sync(0xffffffffu, x, i) * rd[i];
        if (lane == i) x = xi;
        else if (lane < i) x = fma(-xi, A[i][lane], x);
      }
    Dinv[(static_cast<int64_t>(I) * kTB + j) * kTB + lane] = (lane <= j && j < bw) ? x : 0.0;
  }
}

__global__ void __launch_bounds__(256) trinv_blockcol_kernel(const double* __restrict__ R, int64_t ldr, int k,
                                                             const double* __restrict__ Dinv,
                                                             double* __restrict__ Rinv) {
  extern __shared__ double X[];       // [J + 1][kTB][kTB + 1]: X_KJ blocks, [c][r]
  __shared__ double Rt[kTB][kTB + 1];  // R_IK, [c][r]
  __shared__ double S[kTB][kTB + 1];   // partial sum, [c][r]
  const int J = blockIdx.x, j0 = J * kTB;
  const int tid = threadIdx.x;
  const int c = tid & 31, r0 = (tid >> 5) * 4;  // this thread's outputs: rows r0..r0+3 of column c
  auto xb = [&](int K) { return X + static_cast<size_t>(K) * kTB * (kTB + 1); };
  {
    const double* d = Dinv + static_cast<int64_t>(J) * kTB * kTB;
    double* x = xb(J);
    for (int e = tid; e < kTB * kTB; e += blockDim.x) x[(e / kTB) * (kTB + 1) + e % kTB] = d[e];
  }
  __syncthreads();
  for (int I = J - 1; I >= 0; --I) {
    const int i0 = I * kTB;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int K = I + 1; K <= J; ++K) {
      const int kk0 = K * kTB, kw = min(kTB, k - kk0);
      __syncthreads();  // Rt reuse
      for (int e = tid; e < kTB * kTB; e += blockDim.x) {
        const int cc = e / kTB, rr = e % kTB;
        Rt[cc][rr] = cc < kw ? R[static_cast<int64_t>(kk0 + cc) * ldr + i0 + rr] : 0.0;
      }
      __syncthreads();
      const double* x = xb(K);
#pragma unroll 4
      for (int t = 0; t < kTB; ++t) {
        const double b = x[c * (kTB + 1) + t];  // X_KJ(t, c)
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] = fma(Rt[t][r0 + u], b, acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) S[c][r0 + u] = acc[u];
    __syncthreads();
    // X_IJ = -D_I S
    const double* d = Dinv + static_cast<int64_t>(I) * kTB * kTB;  // [col][row]
    double o[4] = {0.0, 0.0, 0.0, 0.0};
    for (int t = 0; t < kTB; ++t) {
      const double b = S[c][t];
#pragma unroll
      for (int u = 0; u < 4; ++u) o[u] = fma(d[t * kTB + r0 + u], b, o[u]);
    }
    double* xi = xb(I);
#pragma unroll
    for (int u = 0; u < 4; ++u) xi[c * (kTB + 1) + r0 + u] = -o[u];
    __syncthreads();
  }
  // column block J of R^{-1}: rows 0 .. j0 + kTB from the X blocks, zeros below
  const int jw = min(kTB, k - j0);
  for (int e = tid; e < jw * k; e += blockDim.x) {
    const int cc = e / k, rr = e % k;
    const int K = rr / kTB;
    Rinv[static_cast<int64_t>(j0 + cc) * k + rr] = K <= J ? xb(K)[cc * (kTB + 1) + rr % kTB] : 0.0;
  }
}

// Z (ke x n): Z(:, perm[j]) = e_j for j < ke, = T(:, j - ke) otherwise.
__global__ void assemble_z_kernel(const int64_t* __restrict__ perm, int ke, int64_t n,
                                  const double* __restrict__ T, double* __restrict__ Z) {
  const int64_t total = n * ke;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / ke;
    const int i = static_cast<int>(e % ke);
    const int64_t col = perm[j];
    Z[col * ke + i] = (j < ke) ? (i == j ? 1.0 : 0.0) : T[(j - ke) * ke + i];
  }
}

}  // namespace

size_t cpqr_work_bytes(int64_t n, int grid, int m) {
  return sizeof(double) * 2 * n + sizeof(int64_t) * n +
         2 * static_cast<size_t>(grid) * (sizeof(double) * 2 + sizeof(int64_t) * 2) +
         sizeof(double) * (2 * static_cast<size_t>(grid) * m + 2 * (m + 4)) + 256;
}

cudaError_t cpqr_rank(double* W, int64_t ld, int m, int64_t n, int kmax, double halt, int64_t* perm, void* work,
                      int* stopped, int* recomputes, int num_sms, cudaStream_t st) {
  if (m > kMaxRows) return cudaErrorInvalidValue;
  const int G = num_sms;
  CpqrParams prm{};
  prm.W = W;
  prm.ld = ld;
  prm.m = m;
  prm.n = n;
  prm.kmax = kmax;
  prm.halt = halt;
  double* w = static_cast<double*>(work);
  prm.norms2 = w;
  prm.norms0 = prm.norms2 + n;
  prm.part_val = prm.norms0 + n;
  prm.part_n0 = prm.part_val + 2 * G;
  prm.stage_col = prm.part_n0 + 2 * G;
  prm.stage_r = prm.stage_col + 2 * static_cast<int64_t>(G) * m;
  prm.part_idx = reinterpret_cast<int64_t*>(prm.stage_r + 2 * (m + 4));
  prm.part_perm = prm.part_idx + 2 * G;
  prm.perm = perm;
  prm.stopped = stopped;
  prm.recomputes = recomputes;
  void* args[] = {&prm};
  void* fn;
  if (m <= 128) fn = reinterpret_cast<void*>(cpqr_kernel<4>);
  else if (m <= 256) fn = reinterpret_cast<void*>(cpqr_kernel<8>);
  else if (m <= 384) fn = reinterpret_cast<void*>(cpqr_kernel<12>);
  else fn = reinterpret_cast<void*>(cpqr_kernel<16>);
  cudaError_t e = cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kCpqrThreads), args, 0, st);
  count_launch();
  return e;
}

cudaError_t trinv_upper(const double* R, int64_t ldr, int k, double* Rinv, cudaStream_t st) {
  if (k <= 0) return cudaSuccess;
  const int nb = (k + kTB - 1) / kTB;
  const size_t smem = sizeof(double) * nb * kTB * (kTB + 1);
  // the blocked kernel holds one block column in shared memory (k <= 736); the per-column kernel keeps a
  // column in 11 registers per lane (k <= 352)
  if (k > 352 && smem > 200 * 1024) return cudaErrorInvalidValue;
  if (k > 64 && smem <= 200 * 1024) {
    static std::atomic<uint64_t> cfg{0};
    if (attr_pending(cfg)) {
      cudaError_t e = cudaFuncSetAttribute(trinv_blockcol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      if (e != cudaSuccess) return e;
      attr_done(cfg);
    }
    double* dinv = nullptr;
    cudaError_t e = ws_alloc(reinterpret_cast<void**>(&dinv), sizeof(double) * nb * kTB * kTB, st);
    if (e != cudaSuccess) return e;
    trinv_diag_kernel<<<nb, 256, 0, st>>>(R, ldr, k, dinv);
    trinv_blockcol_kernel<<<nb, 256, smem, st>>>(R, ldr, k, dinv, Rinv);
    count_launch(2);
    e = cudaGetLastError();
    cudaFreeAsync(dinv, st);
    return e;
  }
  const int warps = 8;
  trinv_upper_kernel<11><<<(k + warps - 1) / warps, warps * 32, 0, st>>>(R, ldr, k, Rinv);
  count_launch();
  return cudaGetLastError();
}

cudaError_t assemble_z(const int64_t* perm, int ke, int64_t n, const double* T, double* Z, cudaStream_t st) {
  if (ke <= 0 || n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n * ke + 255) / 256, 148 * 8);
  assemble_z_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(perm, ke, n, T, Z);
  count_launch();
  return cudaGetLastError();
}

}  // namespace rfgpu
