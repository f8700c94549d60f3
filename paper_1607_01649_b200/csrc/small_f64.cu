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

#include "common.cuh"
#include "rfgpu_internal.h"

namespace cg = cooperative_groups;

namespace rfgpu {

namespace {

constexpr int kSmallThreads = 1024;

// ------------------------------------------------------------ chol_inv ---
// Augmented elimination on M = [G | I] (c x 2c, row-major, W = 2c): row j is
// scaled by 1/sqrt(pivot) and eliminated from the trailing rows, so the left
// block becomes R and the right block L^{-1} = R^{-T}.
template <bool SMEM>
__global__ void __launch_bounds__(kSmallThreads, 1)
    chol_inv_kernel(const double* __restrict__ G, int c, double* __restrict__ R, double* __restrict__ Rinv,
                    double* __restrict__ work, int* info, double* info_d) {
  extern __shared__ double sm[];
  double* M = SMEM ? sm : work;
  const int W = 2 * c;
  const int tid = threadIdx.x, nthr = blockDim.x;
  __shared__ double s_floor, s_trace, s_minratio, s_cjj;
  __shared__ int s_fail;
  __shared__ double red[32];

  for (int e = tid; e < c * W; e += nthr) {
    const int i = e / W, col = e % W;
    double v;
    if (col < c) {
      const int a = min(i, col), b = max(i, col);
      v = G[static_cast<int64_t>(b) * c + a];  // upper triangle of G (col-major)
    } else {
      v = (col - c == i) ? 1.0 : 0.0;
    }
    M[e] = v;
  }
  double md = 0.0, tr = 0.0;
  for (int j = tid; j < c; j += nthr) {
    const double g = G[static_cast<int64_t>(j) * c + j];
    md = fmax(md, fabs(g));
  }
  // block max via shuffles
  for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
  if ((tid & 31) == 0) red[tid >> 5] = md;
  __syncthreads();
  if (tid == 0) {
    double mx = 0.0;
    for (int w = 0; w < nthr / 32; ++w) mx = fmax(mx, red[w]);
    for (int j = 0; j < c; ++j) tr += G[static_cast<int64_t>(j) * c + j];
    s_floor = 1e-14 * mx;
    s_trace = tr;
    s_minratio = INFINITY;
    s_fail = 0;
  }
  __syncthreads();

  for (int j = 0; j < c; ++j) {
    if (tid == 0) {
      const double d = M[j * W + j];
      if (d <= s_floor || !(d > 0.0)) {
        s_fail = j + 1;
      } else {
        s_minratio = fmin(s_minratio, s_trace > 0.0 ? d / s_trace : 0.0);
        s_cjj = sqrt(d);
      }
    }
    __syncthreads();
    if (s_fail) break;
    const double cjj = s_cjj;
    // scale row j: left columns > j, right columns c..c+j
    for (int col = j + 1 + tid; col <= c + j; col += nthr) M[j * W + col] = M[j * W + col] / cjj;
    if (tid == 0) M[j * W + j] = cjj;
    __syncthreads();
    // eliminate rows i > j over columns j+1 .. c+j (left part: col >= i only)
    const int rows = c - j - 1, width = c;
    const int total = rows * width;
    for (int e = tid; e < total; e += nthr) {
      const int i = j + 1 + e / width;
      const int col = j + 1 + e % width;
      if (col < c && col < i) continue;
      M[i * W + col] -= M[j * W + i] * M[j * W + col];
    }
    __syncthreads();
  }

  if (tid == 0) {
    info[0] = s_fail;
    info_d[0] = s_minratio;
  }
  if (s_fail) return;
  for (int e = tid; e < c * c; e += nthr) {
    const int col = e / c, i = e % c;  // column-major output index
    R[e] = (i <= col) ? M[i * W + col] : 0.0;
    Rinv[e] = (i <= col) ? M[col * W + c + i] : 0.0;  // Rinv(i, col) = Linv(col, i)
  }
}

// ----------------------------------------------------------- jacobi_svd ---
struct JacobiParams {
  const double* X;
  int64_t mr;  // rows of X
  int c;       // columns
  double* U;
  double* S;
  double* V;
  double* gX;  // global staging (mode without smem residency), [P][c][RX]
  double* gV;  // [P][c][RV]
  int RX, RV;  // rows of X / V owned per CTA
  int* info;
  int* sweeps_out;
};

__device__ __forceinline__ void pair_of(int r, int k, int cc, int* a, int* b) {
  // circle-method round-robin on cc (even) logical positions
  const int n = cc - 1;
  if (k == 0) {
    *a = 0;
    *b = 1 + (r % n);
  } else {
    *a = 1 + (r + k) % n;
    *b = 1 + (r - k + n) % n;
  }
  if (*a > *b) {
    const int t = *a;
    *a = *b;
    *b = t;
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(kSmallThreads, 1) jacobi_svd_kernel(const JacobiParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  const int P = static_cast<int>(cluster.num_blocks());
  const int q = static_cast<int>(cluster.block_rank());
  const int c = p.c, cc = c + (c & 1), npairs = cc / 2;
  const int RX = p.RX, RV = p.RV;
  const int64_t r0x = static_cast<int64_t>(q) * RX;
  const int64_t rem_x = p.mr - r0x;
  const int nrx = rem_x <= 0 ? 0 : static_cast<int>(rem_x < RX ? rem_x : RX);
  const int r0v = q * RV;
  const int nrv = max(0, min(RV, c - r0v));

  extern __shared__ double sm[];
  // layout: [X rows (c*RX)] [V rows (c*RV)] (SMEM only) | partials[2][P][npairs*3] | nrm[P][cc] | perm, cs/sn
  double* Xs;
  double* Vs;
  double* part;
  if (SMEM) {
    Xs = sm;
    Vs = sm + static_cast<size_t>(c) * RX;
    part = Vs + static_cast<size_t>(c) * RV;
  } else {
    Xs = p.gX + static_cast<size_t>(q) * c * RX;
    Vs = p.gV + static_cast<size_t>(q) * c * RV;
    part = sm;
  }
  double* nrmp = part + 2 * P * npairs * 3;        // [P][cc]
  double* csn = nrmp + P * cc;                      // [npairs][2]
  int* perm = reinterpret_cast<int*>(csn + 2 * npairs);  // [cc]
  int* rotflag = perm + cc;                         // [npairs]
  __shared__ int s_rotated, s_conv;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  // load owned rows; V = I
  for (int e = tid; e < c * RX; e += blockDim.x) {
    const int col = e / RX, r = e % RX;
    Xs[e] = (r < nrx) ? p.X[static_cast<int64_t>(col) * p.mr + r0x + r] : 0.0;
  }
  for (int e = tid; e < c * RV; e += blockDim.x) {
    const int col = e / RV, r = e % RV;
    Vs[e] = (r < nrv && r0v + r == col) ? 1.0 : 0.0;
  }
  __syncthreads();

  auto exchange_norms = [&]() {
    // partial squared column norms over owned rows -> every CTA's nrmp[q][*]
    for (int col = warp; col < c; col += nwarps) {
      double s = 0.0;
      const double* x = Xs + static_cast<size_t>(col) * RX;
      for (int r = lane; r < nrx; r += 32) s = fma(x[r], x[r], s);
      s = warp_sum(s);
      if (lane == 0) {
        for (int d = 0; d < P; ++d) cluster.map_shared_rank(nrmp, d)[q * cc + col] = s;
      }
    }
    cluster.sync();
  };
  auto rank_sort = [&]() {
    // stable descending sort by total norm (std::stable_sort with >)
    for (int j = tid; j < c; j += blockDim.x) {
      double nj = 0.0;
      for (int d = 0; d < P; ++d) nj += nrmp[d * cc + j];
      int rank = 0;
      for (int i = 0; i < c; ++i) {
        double ni = 0.0;
        for (int d = 0; d < P; ++d) ni += nrmp[d * cc + i];
        if (ni > nj || (ni == nj && i < j)) ++rank;
      }
      perm[rank] = j;
    }
    if (tid == 0 && (c & 1)) perm[c] = -1;  // phantom
    __syncthreads();
  };

  int sweep = 0;
  if (tid == 0) s_conv = (c <= 1);
  __syncthreads();
  int parity = 0;
  while (!s_conv && sweep < 60) {
    exchange_norms();
    rank_sort();
    if (tid == 0) s_rotated = 0;
    __syncthreads();
    for (int rd = 0; rd < cc - 1; ++rd) {
      double* pbuf = part + parity * P * npairs * 3;
      // 1. partial inner products for every pair of this round
      for (int k = warp; k < npairs; k += nwarps) {
        int a, b;
        pair_of(rd, k, cc, &a, &b);
        const int cp = perm[a], cq = perm[b];
        double app = 0.0, aqq = 0.0, apq = 0.0;
        if (cp >= 0 && cq >= 0) {
          const double* xp = Xs + static_cast<size_t>(cp) * RX;
          const double* xq = Xs + static_cast<size_t>(cq) * RX;
          for (int r = lane; r < nrx; r += 32) {
            const double u = xp[r], v = xq[r];
            app = fma(u, u, app);
            aqq = fma(v, v, aqq);
            apq = fma(u, v, apq);
          }
          app = warp_sum(app);
          aqq = warp_sum(aqq);
          apq = warp_sum(apq);
        }
        if (lane < P) {
          double* dst = cluster.map_shared_rank(pbuf, lane) + (q * npairs + k) * 3;
          dst[0] = app;
          dst[1] = aqq;
          dst[2] = apq;
        }
      }
      cluster.sync();
      // 2. identical rotation decisions in every CTA; rotate owned rows
      for (int k = warp; k < npairs; k += nwarps) {
        int a, b;
        pair_of(rd, k, cc, &a, &b);
        const int cp = perm[a], cq = perm[b];
        if (cp < 0 || cq < 0) continue;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int d = 0; d < P; ++d) {
          const double* s = pbuf + (d * npairs + k) * 3;
          app += s[0];
          aqq += s[1];
          apq += s[2];
        }
        if (app == 0.0 || aqq == 0.0) continue;
        if (fabs(apq) <= 1e-15 * sqrt(app * aqq)) continue;
        const double zeta = (aqq - app) / (2.0 * apq);
        const double t = (zeta < 0.0 ? -1.0 : 1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t);
        const double sn = cs * t;
        if (lane == 0) s_rotated = 1;
        double* xp = Xs + static_cast<size_t>(cp) * RX;
        double* xq = Xs + static_cast<size_t>(cq) * RX;
        for (int r = lane; r < nrx; r += 32) {
          const double u = xp[r], v = xq[r];
          xp[r] = cs * u - sn * v;
          xq[r] = sn * u + cs * v;
        }
        double* vp = Vs + static_cast<size_t>(cp) * RV;
        double* vq = Vs + static_cast<size_t>(cq) * RV;
        for (int r = lane; r < nrv; r += 32) {
          const double u = vp[r], v = vq[r];
          vp[r] = cs * u - sn * v;
          vq[r] = sn * u + cs * v;
        }
      }
      __syncthreads();
      parity ^= 1;
    }
    ++sweep;
    if (tid == 0) s_conv = !s_rotated;
    __syncthreads();
  }
  const bool converged = s_conv;

  // final singular values, stable descending order
  exchange_norms();
  for (int j = tid; j < c; j += blockDim.x) {
    double nj = 0.0;
    for (int d = 0; d < P; ++d) nj += nrmp[d * cc + j];
    nrmp[j] = nj;  // rank-0 slot reused after the sum (all reads of slot d=0 for j done by this thread only)
  }
  __syncthreads();
  // sigma_j = sqrt(total norm); use a separate array to avoid read/write races
  double* sig = csn;  // npairs*2 >= c doubles
  for (int j = tid; j < c; j += blockDim.x) sig[j] = sqrt(nrmp[j]);
  __syncthreads();
  for (int j = tid; j < c; j += blockDim.x) {
    int rank = 0;
    for (int i = 0; i < c; ++i)
      if (sig[i] > sig[j] || (sig[i] == sig[j] && i < j)) ++rank;
    perm[rank] = j;
  }
  __syncthreads();
  const double smax = c > 0 ? sig[perm[0]] : 0.0;
  int zero_cols = 0;
  for (int j = 0; j < c; ++j) {
    const int src = perm[j];
    const double s = sig[src];
    const bool ok = s > 0.0 && s > smax * 1e-250;
    if (!ok) zero_cols = 1;
    if (q == 0 && tid == 0) p.S[j] = ok ? s : 0.0;
    const double* x = Xs + static_cast<size_t>(src) * RX;
    for (int r = tid; r < nrx; r += blockDim.x) p.U[static_cast<int64_t>(j) * p.mr + r0x + r] = ok ? x[r] / s : 0.0;
    const double* v = Vs + static_cast<size_t>(src) * RV;
    for (int r = tid; r < nrv; r += blockDim.x) p.V[static_cast<int64_t>(j) * c + r0v + r] = v[r];
  }
  if (q == 0 && tid == 0) {
    p.info[0] = converged ? (zero_cols ? 2 : 0) : 1;
    if (p.sweeps_out) p.sweeps_out[0] = sweep;
  }
  cluster.sync();  // keep DSMEM alive until every CTA is done with remote writes
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
  int P, RX, RV;
  bool smem;
  size_t bytes;
};

JacobiLayout jacobi_layout(int64_t mr, int64_t c) {
  const int64_t cc = c + (c & 1), npairs = cc / 2;
  auto extra = [&](int P) {
    return sizeof(double) * (2 * P * npairs * 3 + P * cc + 2 * npairs) + sizeof(int) * (cc + npairs) + 64;
  };
  constexpr size_t kMax = 220 * 1024;
  for (int P : {1, 2, 4, 8}) {
    const int RX = static_cast<int>((mr + P - 1) / P), RV = static_cast<int>((c + P - 1) / P);
    const size_t b = sizeof(double) * static_cast<size_t>(c) * (RX + RV) + extra(P);
    if (b <= kMax) return {P, RX, RV, true, b};
  }
  const int P = 8;
  return {P, static_cast<int>((mr + P - 1) / P), static_cast<int>((c + P - 1) / P), false, extra(P)};
}

}  // namespace

size_t chol_inv_work_bytes(int64_t c) { return sizeof(double) * 2 * c * c; }

cudaError_t chol_inv(const double* G, int64_t c, double* R, double* Rinv, double* work, int* info,
                     double* info_d, cudaStream_t st) {
  if (c <= 0) return cudaSuccess;
  const size_t smem = sizeof(double) * 2 * c * c;
  if (smem <= 200 * 1024) {
    static bool cfg = false;
    if (!cfg) {
      cudaError_t e = cudaFuncSetAttribute(chol_inv_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           200 * 1024);
      if (e != cudaSuccess) return e;
      cfg = true;
    }
    chol_inv_kernel<true><<<1, kSmallThreads, smem, st>>>(G, static_cast<int>(c), R, Rinv, work, info, info_d);
    count_launch();
  } else {
    chol_inv_kernel<false><<<1, kSmallThreads, 0, st>>>(G, static_cast<int>(c), R, Rinv, work, info, info_d);
    count_launch();
  }
  return cudaGetLastError();
}

size_t jacobi_work_bytes(int64_t mr, int64_t c) {
  const JacobiLayout L = jacobi_layout(mr, c);
  if (L.smem) return 0;
  return sizeof(double) * static_cast<size_t>(L.P) * c * (L.RX + L.RV);
}

cudaError_t jacobi_svd(const double* X, int64_t mr, int64_t c, double* U, double* S, double* V, double* work,
                       int* info, int* sweeps_out, cudaStream_t st) {
  if (c <= 0 || mr <= 0) return cudaSuccess;
  const JacobiLayout L = jacobi_layout(mr, c);
  JacobiParams p{};
  p.X = X;
  p.mr = mr;
  p.c = static_cast<int>(c);
  p.U = U;
  p.S = S;
  p.V = V;
  p.RX = L.RX;
  p.RV = L.RV;
  p.info = info;
  p.sweeps_out = sweeps_out;
  if (!L.smem) {
    p.gX = work;
    p.gV = work + static_cast<size_t>(L.P) * c * L.RX;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(L.P);
  cfg.blockDim = dim3(kSmallThreads);
  cfg.dynamicSmemBytes = L.bytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = L.P;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  if (L.smem) {
    static size_t c1 = 0;
    if (L.bytes > c1) {
      e = cudaFuncSetAttribute(jacobi_svd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(L.bytes));
      if (e != cudaSuccess) return e;
      c1 = L.bytes;
    }
    e = cudaLaunchKernelEx(&cfg, jacobi_svd_kernel<true>, p);
    count_launch();
  } else {
    static size_t c2 = 0;
    if (L.bytes > c2) {
      e = cudaFuncSetAttribute(jacobi_svd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(L.bytes));
      if (e != cudaSuccess) return e;
      c2 = L.bytes;
    }
    e = cudaLaunchKernelEx(&cfg, jacobi_svd_kernel<false>, p);
    count_launch();
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
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
