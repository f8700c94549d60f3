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
// Packed upper-triangular storage P (column-packed: (i, j) at j(j+1)/2 + i,
// i <= j), in shared memory when it fits (c <= 236), else in global memory.
// Phase 1: right-looking Cholesky in the reference recurrence order
// (dense.cpp:763-786): row j is divided by sqrt(pivot), then each trailing
// entry (i, col), j < i <= col, subtracts R(j,i) R(j,col).
// Phase 2: R^{-1} one warp per column: back substitution R x = e_j in axpy
// form, x distributed over the lanes' registers (S slots per lane).
__device__ __forceinline__ int64_t pk(int i, int j) { return static_cast<int64_t>(j) * (j + 1) / 2 + i; }

template <bool SMEM, int S>
__global__ void __launch_bounds__(kSmallThreads, 1)
    chol_inv_kernel(const double* __restrict__ G, int c, double* __restrict__ R, double* __restrict__ Rinv,
                    double* __restrict__ work, int* info, double* info_d) {
  extern __shared__ double sm[];
  double* base = SMEM ? sm : work;
  double* rowj = base;          // [c]  current pivot row of R
  double* rdiag = base + c;     // [c]  1 / R(j,j)
  double* P = base + 2 * c;     // packed upper triangle
  const int tid = threadIdx.x, nthr = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nthr >> 5;
  __shared__ double s_floor, s_trace, s_minratio;
  __shared__ int s_fail;

  for (int j = warp; j < c; j += nwarps)
    for (int i = lane; i <= j; i += 32) P[pk(i, j)] = G[static_cast<int64_t>(j) * c + i];
  if (tid == 0) {
    double mx = 0.0, tr = 0.0;
    for (int j = 0; j < c; ++j) {
      const double g = G[static_cast<int64_t>(j) * c + j];
      mx = fmax(mx, fabs(g));
      tr += g;
    }
    s_floor = 1e-14 * mx;
    s_trace = tr;
    s_minratio = INFINITY;
    s_fail = 0;
  }
  __syncthreads();

  for (int j = 0; j < c; ++j) {
    if (tid == 0) {
      const double d = P[pk(j, j)];
      if (d <= s_floor || !(d > 0.0)) {
        s_fail = j + 1;
      } else {
        s_minratio = fmin(s_minratio, s_trace > 0.0 ? d / s_trace : 0.0);
        const double cjj = sqrt(d);
        P[pk(j, j)] = cjj;
        rowj[j] = cjj;
        rdiag[j] = 1.0 / cjj;
      }
    }
    __syncthreads();
    if (s_fail) break;
    const double cjj = rowj[j];
    for (int col = j + 1 + tid; col < c; col += nthr) {
      const double v = P[pk(j, col)] / cjj;
      P[pk(j, col)] = v;
      rowj[col] = v;
    }
    __syncthreads();
    for (int col = j + 1 + warp; col < c; col += nwarps) {
      const double rc = rowj[col];
      double* pc = P + pk(0, col);
      for (int i = j + 1 + lane; i <= col; i += 32) pc[i] -= rowj[i] * rc;
    }
    __syncthreads();
  }
  if (tid == 0) {
    info[0] = s_fail;
    info_d[0] = s_minratio;
  }
  if (s_fail) return;

  for (int j = warp; j < c; j += nwarps)
    for (int i = lane; i < c; i += 32) R[static_cast<int64_t>(j) * c + i] = i <= j ? P[pk(i, j)] : 0.0;

  // R^{-1} is formed by trinv_upper (many CTAs, one warp per column).
  (void)Rinv;
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
  int RX, RV;  // rows of X / V owned per CTA
  int LDX, LDV;
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
__global__ void __launch_bounds__(kSmallThreads, 1) jacobi_svd_kernel(const JacobiParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  const int P = static_cast<int>(cluster.num_blocks());
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
  const int npo = (npairs + P - 1) / P;            // pairs per owner CTA
  const int owned = (npairs - q + P - 1) / P;      // pairs owned by this CTA (k % P == q)

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
  double* params = rest + 4;                           // [2][npairs][2] (cs, sn; sn = 2 => skip)
  double* inbox = params + 4 * npairs;                 // [2][P][npo][3]
  double* red = inbox + 2 * P * npo * 3;               // [H][npairs][3], aliased by nrmp [P][cc]
  const int red_sz = max(H * np3, P * cc);
  double* nrmp = red;
  double* nrm = red + red_sz;                          // [cc]
  int* perm = reinterpret_cast<int*>(nrm + cc);        // [cc]
  __shared__ int s_rotated, s_conv;

  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  uint32_t uses[2] = {0u, 0u};
  for (int e = tid; e < c * RX; e += blockDim.x) {
    const int col = e / RX, r = e % RX;
    Xs[static_cast<size_t>(col) * LDX + r] = (r < nrx) ? p.X[static_cast<int64_t>(col) * p.mr + r0x + r] : 0.0;
  }
  for (int e = tid; e < c * RV; e += blockDim.x) {
    const int col = e / RV, r = e % RV;
    Vs[static_cast<size_t>(col) * LDV + r] = (r < nrv && r0v + r == col) ? 1.0 : 0.0;
  }
  cluster.sync();  // barriers initialised cluster-wide before any st.async

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

  int sweep = 0, parity = 0;
  if (tid == 0) s_conv = (c <= 1);
  __syncthreads();
  while (!s_conv && sweep < 60) {
    norms();
    sort_desc(nrm);
    if (tid == 0) s_rotated = 0;
    __syncthreads();
    for (int rd = 0; rd < cc - 1; ++rd) {
      int cp = -1, cq = -1;
      if (active && k < npairs) {
        int a, b;
        pair_of(rd, k, cc, &a, &b);
        cp = perm[a];
        cq = perm[b];
      }
      const bool valid = cp >= 0 && cq >= 0;
      if (P > 1 && tid == 0) {
        mbar_arrive_expect_tx(&bars[parity], static_cast<uint32_t>(P * owned * 24));
        mbar_arrive_expect_tx(&bars[2 + parity], static_cast<uint32_t>(npairs * 16));
      }
      // A. partial inner products over this warp's rows
      if (active && k < npairs) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        if (valid) {
          const double* xp = Xs + static_cast<size_t>(cp) * LDX;
          const double* xq = Xs + static_cast<size_t>(cq) * LDX;
          for (int r = x0; r < x1; ++r) {
            const double u = xp[r], v = xq[r];
            app = fma(u, u, app);
            aqq = fma(v, v, aqq);
            apq = fma(u, v, apq);
          }
        }
        double* d = red + (h * npairs + k) * 3;
        d[0] = app;
        d[1] = aqq;
        d[2] = apq;
      }
      __syncthreads();
      // B. CTA partial -> the pair's owner CTA (k mod P)
      double* ib = inbox + parity * P * npo * 3;
      double* pr = params + parity * npairs * 2;
      if (h == 0 && k < npairs) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int hh = 0; hh < H; ++hh) {
          const double* s = red + (hh * npairs + k) * 3;
          app += s[0];
          aqq += s[1];
          apq += s[2];
        }
        double* slot = ib + (q * npo + k / P) * 3;
        if (P > 1) {
          const uint32_t o = static_cast<uint32_t>(k % P);
          const uint32_t ra = mapa_u32(smem_u32(slot), o), rb = mapa_u32(smem_u32(&bars[parity]), o);
          st_async_f64(ra, app, rb);
          st_async_f64(ra + 8, aqq, rb);
          st_async_f64(ra + 16, apq, rb);
        } else {
          slot[0] = app;
          slot[1] = aqq;
          slot[2] = apq;
        }
      }
      if (P == 1) __syncthreads();
      else if (h == 0) mbar_wait(&bars[parity], uses[parity] & 1u);
      // C. owners: rotation parameters (reference formula), broadcast to all
      if (h == 0 && k < npairs && k % P == q) {
        double app = 0.0, aqq = 0.0, apq = 0.0;
        for (int d = 0; d < P; ++d) {
          const double* s = ib + (d * npo + k / P) * 3;
          app += s[0];
          aqq += s[1];
          apq += s[2];
        }
        double cs = 1.0, sn = 2.0;
        if (valid && app != 0.0 && aqq != 0.0 && !(fabs(apq) <= 1e-15 * sqrt(app * aqq))) {
          const double zeta = (aqq - app) / (2.0 * apq);
          const double t = (zeta < 0.0 ? -1.0 : 1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          cs = 1.0 / sqrt(1.0 + t * t);
          sn = cs * t;
        }
        if (P > 1) {
          const uint32_t la = smem_u32(pr + 2 * k), lb = smem_u32(&bars[2 + parity]);
          for (int d = 0; d < P; ++d) st_async_v2(mapa_u32(la, d), cs, sn, mapa_u32(lb, d));
        } else {
          pr[2 * k] = cs;
          pr[2 * k + 1] = sn;
        }
      }
      if (P == 1) __syncthreads();
      else if (active) mbar_wait(&bars[2 + parity], uses[parity] & 1u);
      uses[parity] += 1u;
      // D. rotate this warp's rows of X and V
      if (active && k < npairs && valid) {
        const double cs = pr[2 * k], sn = pr[2 * k + 1];
        if (sn != 2.0) {
          if (h == 0) s_rotated = 1;
          double* xp = Xs + static_cast<size_t>(cp) * LDX;
          double* xq = Xs + static_cast<size_t>(cq) * LDX;
          for (int r = x0; r < x1; ++r) {
            const double u = xp[r], v = xq[r];
            xp[r] = cs * u - sn * v;
            xq[r] = sn * u + cs * v;
          }
          double* vp = Vs + static_cast<size_t>(cp) * LDV;
          double* vq = Vs + static_cast<size_t>(cq) * LDV;
          for (int r = v0; r < v1; ++r) {
            const double u = vp[r], v = vq[r];
            vp[r] = cs * u - sn * v;
            vq[r] = sn * u + cs * v;
          }
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
  norms();
  double* sig = red + P * cc;  // free after norms(): red_sz >= P*cc, use params-sized scratch instead
  sig = params;                // 4*npairs >= c doubles
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
  int P, RX, RV, LDX, LDV;
  bool smem;
  size_t bytes;
};

inline int pad_ld(int r) { return r + ((r % 2 == 0) ? 1 : 0); }  // odd leading dimension

JacobiLayout jacobi_layout(int64_t mr, int64_t c) {
  const int64_t cc = c + (c & 1), npairs = cc / 2;
  const int64_t G = (npairs + 31) / 32, H = 32 / G;
  auto extra = [&](int P) {
    const int64_t npo = (npairs + P - 1) / P;
    return sizeof(double) * (4 + 4 * npairs + 2 * P * npo * 3 + std::max<int64_t>(H * npairs * 3, P * cc) + cc) +
           sizeof(int) * cc + 64;
  };
  constexpr size_t kMax = 224 * 1024;
  for (int P : {1, 2, 4, 8, 16}) {
    const int RX = static_cast<int>((mr + P - 1) / P), RV = static_cast<int>((c + P - 1) / P);
    const int LDX = pad_ld(RX), LDV = pad_ld(RV);
    const size_t b = sizeof(double) * static_cast<size_t>(c) * (LDX + LDV) + extra(P);
    if (b <= kMax) return {P, RX, RV, LDX, LDV, true, b};
  }
  const int P = 8;
  const int RX = static_cast<int>((mr + P - 1) / P), RV = static_cast<int>((c + P - 1) / P);
  return {P, RX, RV, pad_ld(RX), pad_ld(RV), false, extra(P)};
}

}  // namespace

size_t chol_inv_work_bytes(int64_t c) { return sizeof(double) * (2 * c + c * (c + 1) / 2); }

cudaError_t chol_inv(const double* G, int64_t c, double* R, double* Rinv, double* work, int* info,
                     double* info_d, cudaStream_t st) {
  if (c <= 0) return cudaSuccess;
  if (c > 352) return cudaErrorInvalidValue;
  const size_t smem = chol_inv_work_bytes(c);
  const int ci = static_cast<int>(c);
  if (smem <= 224 * 1024 && c <= 256) {
    static bool cfg = false;
    if (!cfg) {
      cudaError_t e = cudaFuncSetAttribute(chol_inv_kernel<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           224 * 1024);
      if (e != cudaSuccess) return e;
      cfg = true;
    }
    chol_inv_kernel<true, 8><<<1, kSmallThreads, smem, st>>>(G, ci, R, Rinv, work, info, info_d);
    count_launch();
  } else {
    chol_inv_kernel<false, 11><<<1, kSmallThreads, 0, st>>>(G, ci, R, Rinv, work, info, info_d);
    count_launch();
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return trinv_upper(R, c, ci, Rinv, st);
}

size_t jacobi_work_bytes(int64_t mr, int64_t c) {
  const JacobiLayout L = jacobi_layout(mr, c);
  if (L.smem) return 0;
  return sizeof(double) * static_cast<size_t>(L.P) * c * (L.LDX + L.LDV);
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
  p.LDX = L.LDX;
  p.LDV = L.LDV;
  p.info = info;
  p.sweeps_out = sweeps_out;
  if (!L.smem) {
    p.gX = work;
    p.gV = work + static_cast<size_t>(L.P) * c * L.LDX;
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
      e = cudaFuncSetAttribute(jacobi_svd_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
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
