// Tall-skinny FP64 GEMMs on the sm_100a FP64 tensor pipe (SASS DMMA.8x8x4).
//
// These replace the reference's `multiply` kernels on the hot path
// (proj/src/dense.cpp:102-126): every pass over A in power_range / rsvd /
// randomized_id / randomized_cur (proj/src/rangefinder.cpp:68-78,
// proj/src/lowrank.cpp:92,320,352) is one launch of
//
//   NN:  C(M x N) = A(M x K) * B(K x N)      A col-major (lda >= M)
//   TN:  C(M x N) = A(K x M)^T * B(K x N)    A col-major (lda >= K)
//
// with N = l = k + p small (<= a few hundred) and M or K huge. A streams
// from HBM exactly once per pass: the N dimension is split into at most
// ceil(N/128) CTA columns whose CTAs are scheduled adjacently (n-tile is the
// fastest-varying block index) so sibling reads of the same A block hit L2.
// The thin operand B is staged per K-tile from L2.
//
// CTA tile 128 x (16*NT), 8 warps as 4 (M) x 2 (N), warp tile 32 x 8*NT,
// BK = 32, 3-stage cp.async ring. Shared-memory rows are padded to
// ld = 4 (mod 16) doubles so the 8x4 / 4x8 fragment loads are conflict-free.
// Split-K writes per-split partials to a workspace; rf_reduce_splits sums
// them in a fixed order (deterministic, no atomics).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "rfgpu_internal.h"

namespace rfgpu {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;
constexpr int STAGES = 3;
constexpr int NTHREADS = 256;
constexpr int LDA_NN = BM + 4;  // sA[k][m]
constexpr int LDK = BK + 4;     // sA[m][k] (TN) and sB[n][k]

template <bool TRANS>
constexpr int a_stage_elems() { return TRANS ? BM * LDK : BK * LDA_NN; }

template <int NT>
constexpr int b_stage_elems() { return 16 * NT * LDK; }

template <bool TRANS, int NT>
constexpr size_t smem_bytes() {
  return sizeof(double) * STAGES * (a_stage_elems<TRANS>() + b_stage_elems<NT>());
}

struct GemmParams {
  int64_t M, N, K;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;  // splits == 1: final output (ldc); else partial workspace [S][N][M]
  int64_t ldc;
  int ntiles;       // CTA columns along N
  int mtiles;
  int splits;
  int64_t ktiles;   // ceil(K / BK)
  double* sumsq;    // optional (NN): per-(mtile,split) sum of squares of A
};

template <bool TRANS, int NT, bool V16>
__device__ __forceinline__ void load_stage(const GemmParams& g, double* sA, double* sB, int64_t m0,
                                           int64_t n0, int64_t k0) {
  const int tid = threadIdx.x;
  constexpr int BN = 16 * NT;
  if constexpr (!TRANS) {
    constexpr int CPC = BM / 2;  // 16-byte chunks per A column
    for (int c = tid; c < BK * CPC; c += NTHREADS) {
      const int kk = c / CPC, mm = (c % CPC) * 2;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      const double* src = g.A;
      int bytes = 0;
      if (gk < g.K && gm < g.M) {
        src = g.A + gk * g.lda + gm;
        bytes = (g.M - gm) >= 2 ? 16 : 8;
      }
      double* dst = sA + kk * LDA_NN + mm;
      if constexpr (V16) {
        cp_async16(dst, src, bytes);
      } else {
        cp_async8(dst, src, bytes >= 8 ? 8 : 0);
        cp_async8(dst + 1, bytes == 16 ? src + 1 : g.A, bytes == 16 ? 8 : 0);
      }
    }
  } else {
    constexpr int CPR = BK / 2;  // chunks per op(A) row (contiguous along k)
    for (int c = tid; c < BM * CPR; c += NTHREADS) {
      const int mm = c / CPR, kk = (c % CPR) * 2;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      const double* src = g.A;
      int bytes = 0;
      if (gm < g.M && gk < g.K) {
        src = g.A + gm * g.lda + gk;
        bytes = (g.K - gk) >= 2 ? 16 : 8;
      }
      double* dst = sA + mm * LDK + kk;
      if constexpr (V16) {
        cp_async16(dst, src, bytes);
      } else {
        cp_async8(dst, src, bytes >= 8 ? 8 : 0);
        cp_async8(dst + 1, bytes == 16 ? src + 1 : g.A, bytes == 16 ? 8 : 0);
      }
    }
  }
  constexpr int CPB = BK / 2;
  for (int c = tid; c < BN * CPB; c += NTHREADS) {
    const int nn = c / CPB, kk = (c % CPB) * 2;
    const int64_t gn = n0 + nn, gk = k0 + kk;
    const double* src = g.B;
    int bytes = 0;
    if (gn < g.N && gk < g.K) {
      src = g.B + gn * g.ldb + gk;
      bytes = (g.K - gk) >= 2 ? 16 : 8;
    }
    double* dst = sB + nn * LDK + kk;
    if constexpr (V16) {
      cp_async16(dst, src, bytes);
    } else {
      cp_async8(dst, src, bytes >= 8 ? 8 : 0);
      cp_async8(dst + 1, bytes == 16 ? src + 1 : g.B, bytes == 16 ? 8 : 0);
    }
  }
}

template <bool TRANS, int NT, bool V16>
__global__ void __launch_bounds__(NTHREADS, 1) gemm_f64_kernel(const GemmParams g) {
  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * a_stage_elems<TRANS>();

  // Block decode: n-tile fastest so CTAs sharing an A block run together.
  const int64_t bid = blockIdx.x;
  const int nt_idx = static_cast<int>(bid % g.ntiles);
  const int64_t rest = bid / g.ntiles;
  const int mt_idx = static_cast<int>(rest % g.mtiles);
  const int split = static_cast<int>(rest / g.mtiles);

  const int64_t m0 = static_cast<int64_t>(mt_idx) * BM;
  const int64_t n0 = static_cast<int64_t>(nt_idx) * 16 * NT;
  const int64_t kt0 = g.ktiles * split / g.splits;
  const int64_t kt1 = g.ktiles * (split + 1) / g.splits;
  const int64_t nkt = kt1 - kt0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int g4 = lane >> 2, t4 = lane & 3;
  const bool do_sumsq = (!TRANS) && g.sumsq != nullptr && nt_idx == 0;

  double acc[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ss = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt)
      load_stage<TRANS, NT, V16>(g, sA + s * a_stage_elems<TRANS>(), sB + s * b_stage_elems<NT>(), m0, n0,
                                 (kt0 + s) * BK);
    cp_async_commit();
  }

  for (int64_t it = 0; it < nkt; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int64_t nxt = it + STAGES - 1;
      if (nxt < nkt) {
        const int st = static_cast<int>(nxt % STAGES);
        load_stage<TRANS, NT, V16>(g, sA + st * a_stage_elems<TRANS>(), sB + st * b_stage_elems<NT>(), m0, n0,
                                   (kt0 + nxt) * BK);
      }
      cp_async_commit();
    }
    const int st = static_cast<int>(it % STAGES);
    const double* a = sA + st * a_stage_elems<TRANS>();
    const double* b = sB + st * b_stage_elems<NT>();

    if (do_sumsq) {
      // Fused ||A||_F^2 (finish_with_projection's frob_norm, rangefinder.cpp:27)
      // from the tile already in shared memory: zero-filled padding adds 0.
#pragma unroll 4
      for (int e = tid; e < BK * BM; e += NTHREADS) {
        const double v = a[(e / BM) * LDA_NN + (e % BM)];
        ss = fma(v, v, ss);
      }
    }

#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double af[4], bf[NT];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int mrow = wm * 32 + i * 8 + g4;
        if constexpr (!TRANS) af[i] = a[(ks * 4 + t4) * LDA_NN + mrow];
        else af[i] = a[mrow * LDK + ks * 4 + t4];
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = b[(wn * NT * 8 + j * 8 + g4) * LDK + ks * 4 + t4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  double* out;
  int64_t ldo;
  if (g.splits == 1) {
    out = g.C;
    ldo = g.ldc;
  } else {
    out = g.C + static_cast<int64_t>(split) * g.M * g.N;
    ldo = g.M;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t m = m0 + wm * 32 + i * 8 + g4;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const int64_t n = n0 + wn * NT * 8 + j * 8 + 2 * t4;
      if (n < g.N) out[n * ldo + m] = acc[i][j][0];
      if (n + 1 < g.N) out[(n + 1) * ldo + m] = acc[i][j][1];
    }
  }

  if (do_sumsq) {
    __shared__ double red[NTHREADS / 32];
    const double tot = block_sum(ss, red);
    if (tid == 0) g.sumsq[static_cast<int64_t>(split) * g.mtiles + mt_idx] = tot;
  }
}

// C(m, n) = sum_{s < S} part[s][n][m], fixed order.
__global__ void reduce_splits_kernel(const double* __restrict__ part, int64_t M, int64_t N, int S,
                                     double* __restrict__ C, int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < S; ++k) s += part[k * total + e];
    const int64_t n = e / M, m = e % M;
    C[n * ldc + m] = s;
  }
}

// Fixed-order sum of n doubles in one CTA.
__global__ void sum_array_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

template <bool TRANS, int NT, bool V16>
cudaError_t launch_one(const GemmParams& g, int64_t grid, cudaStream_t st) {
  auto kern = gemm_f64_kernel<TRANS, NT, V16>;
  constexpr size_t smem = smem_bytes<TRANS, NT>();
  static bool configured = false;  // per-instantiation, per-process (device 0 properties apply to all B200s)
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = true;
  }
  kern<<<static_cast<unsigned>(grid), NTHREADS, smem, st>>>(g);
    count_launch();
  return cudaGetLastError();
}

template <bool TRANS, bool V16>
cudaError_t dispatch_nt(int NT, const GemmParams& g, int64_t grid, cudaStream_t st) {
  switch (NT) {
    case 1: return launch_one<TRANS, 1, V16>(g, grid, st);
    case 2: return launch_one<TRANS, 2, V16>(g, grid, st);
    case 3: return launch_one<TRANS, 3, V16>(g, grid, st);
    case 4: return launch_one<TRANS, 4, V16>(g, grid, st);
    case 5: return launch_one<TRANS, 5, V16>(g, grid, st);
    case 6: return launch_one<TRANS, 6, V16>(g, grid, st);
    case 7: return launch_one<TRANS, 7, V16>(g, grid, st);
    default: return launch_one<TRANS, 8, V16>(g, grid, st);
  }
}

}  // namespace

GemmPlan plan_gemm(int64_t M, int64_t N, int64_t K, int num_sms, int force_splits) {
  GemmPlan p{};
  p.ntiles = static_cast<int>((N + 127) / 128);
  if (p.ntiles < 1) p.ntiles = 1;
  p.nt = static_cast<int>((N + 16 * p.ntiles - 1) / (16 * p.ntiles));
  p.nt = std::max(1, std::min(8, p.nt));
  p.mtiles = static_cast<int>((M + BM - 1) / BM);
  p.ktiles = (K + BK - 1) / BK;
  const int64_t units = static_cast<int64_t>(p.mtiles) * p.ntiles;
  int best = 1;
  if (force_splits > 0) {
    best = static_cast<int>(std::min<int64_t>(force_splits, std::max<int64_t>(1, p.ktiles)));
  } else if (units < 12 * num_sms && p.ktiles > 1) {
    // Smallest split count whose last wave is >= 90% full, keeping >= 4
    // K-tiles per split; else the best-filling one.
    double best_eff = -1.0;
    const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(p.ktiles / 4, 256));
    for (int64_t s = 1; s <= max_s; ++s) {
      const int64_t work = units * s;
      const int64_t waves = (work + num_sms - 1) / num_sms;
      const double eff = static_cast<double>(work) / static_cast<double>(waves * num_sms);
      if (eff >= 0.9) {
        best = static_cast<int>(s);
        best_eff = eff;
        break;
      }
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        best = static_cast<int>(s);
      }
    }
  }
  p.splits = best;
  return p;
}

cudaError_t gemm_f64(bool trans_a, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc, double* workspace,
                     size_t workspace_bytes, double* sumsq_partials, const GemmPlan& p, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (K <= 0) {
    for (int64_t n = 0; n < N; ++n) {
      cudaError_t e = cudaMemsetAsync(C + n * ldc, 0, sizeof(double) * M, st);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  GemmParams g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = A;
  g.lda = lda;
  g.B = B;
  g.ldb = ldb;
  g.ntiles = p.ntiles;
  g.mtiles = p.mtiles;
  g.splits = p.splits;
  g.ktiles = p.ktiles;
  g.sumsq = sumsq_partials;
  if (p.splits == 1) {
    g.C = C;
    g.ldc = ldc;
  } else {
    if (workspace_bytes < gemm_workspace_bytes(M, N, p)) return cudaErrorInvalidValue;
    g.C = workspace;
    g.ldc = M;
  }
  const bool v16 = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                   (lda % 2 == 0) && (ldb % 2 == 0);
  const int64_t grid = static_cast<int64_t>(p.ntiles) * p.mtiles * p.splits;
  cudaError_t e;
  if (trans_a) e = v16 ? dispatch_nt<true, true>(p.nt, g, grid, st) : dispatch_nt<true, false>(p.nt, g, grid, st);
  else e = v16 ? dispatch_nt<false, true>(p.nt, g, grid, st) : dispatch_nt<false, false>(p.nt, g, grid, st);
  if (e != cudaSuccess) return e;
  if (p.splits > 1) {
    const int64_t total = M * N;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
    reduce_splits_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(workspace, M, N, p.splits, C, ldc);
    count_launch();
    e = cudaGetLastError();
  }
  return e;
}

size_t gemm_workspace_bytes(int64_t M, int64_t N, const GemmPlan& p) {
  return p.splits > 1 ? sizeof(double) * static_cast<size_t>(p.splits) * M * N : 0;
}

cudaError_t sum_array(const double* x, int64_t n, double* out, cudaStream_t st) {
  sum_array_kernel<<<1, 1024, 0, st>>>(x, n, out);
    count_launch();
  return cudaGetLastError();
}

}  // namespace rfgpu
