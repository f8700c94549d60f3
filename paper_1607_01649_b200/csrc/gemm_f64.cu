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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <mutex>

#include "common.cuh"
#include "rfgpu_internal.h"

namespace rfgpu {

namespace {

__host__ __device__ __forceinline__ int64_t i64min(int64_t a, int64_t b) { return a < b ? a : b; }

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
  int sym;          // C symmetric (Gram): only tiles touching the upper triangle
  int tri_b;        // B upper triangular (K == N): n-tile j needs k < (j+1)*BN
  int64_t units;    // work units per split (sym: upper tiles only)
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

// ---------------------------------------------------------------------------
// Warp-specialised variant (the default for 16B-aligned operands): one
// producer warp streams the A and B tiles with bulk async copies on the TMA
// engine (cp.async.bulk, mbarrier transaction counts) into a 3-stage ring;
// eight consumer warps run the DMMA loop and release stages through "empty"
// mbarriers, so the tensor pipe never waits on a CTA-wide barrier. Rows /
// columns beyond M or N are left stale in shared memory (they only feed
// output entries that are never stored); the K tail is masked in registers.
constexpr int NCONS = 8;
// 8 consumer warps (2 warpgroups) + 1 producer warpgroup (warp 8 issues the
// copies, warps 9-11 retire). setmaxnreg moves the producer warpgroup's
// registers to the consumers (232 each) so the 4 x NT x 2 FP64 accumulators
// never spill.
constexpr int WS_THREADS = (NCONS + 4) * 32;

// TN tiles arrive through 2-D tensor TMA with the 128-byte swizzle: per
// stage A is [2 k-halves][128 m][16 k] and B is [2][BN n][16 k], dense.
template <bool TRANS>
constexpr int a_stage_ws() { return TRANS ? 2 * BM * 16 : BK * LDA_NN; }
template <bool TRANS, int NT>
constexpr int b_stage_ws() { return 2 * 16 * NT * 16; }  // [2 k-halves][BN][16], both modes
template <bool TRANS, int NT>
constexpr size_t smem_bytes_ws() {
  return sizeof(double) * STAGES * (a_stage_ws<TRANS>() + b_stage_ws<TRANS, NT>()) + 2 * STAGES * sizeof(uint64_t) +
         1024;  // manual 1024-byte alignment of the swizzled boxes
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void decode_unit(const GemmParams& g, int64_t bid, int bn, int& nt_idx, int& mt_idx,
                                            int& split) {
  if (!g.sym) {
    nt_idx = static_cast<int>(bid % g.ntiles);
    const int64_t rest = bid / g.ntiles;
    mt_idx = static_cast<int>(rest % g.mtiles);
    split = static_cast<int>(rest / g.mtiles);
    return;
  }
  int64_t u = bid % g.units;
  split = static_cast<int>(bid / g.units);
  nt_idx = mt_idx = 0;
  for (int mt = 0; mt < g.mtiles; ++mt)
    for (int nt = 0; nt < g.ntiles; ++nt)
      if (static_cast<int64_t>(mt) * BM < static_cast<int64_t>(nt + 1) * bn) {
        if (u == 0) {
          mt_idx = mt;
          nt_idx = nt;
          return;
        }
        --u;
      }
}

template <bool TRANS, int NT>
__global__ void __launch_bounds__(WS_THREADS, 1)
    gemm_f64_tma_kernel(const GemmParams g, const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB) {
  constexpr int BN = 16 * NT;
  extern __shared__ __align__(128) double smem_ws[];
  double* sA = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smem_ws) + 1023) & ~uintptr_t(1023));
  double* sB = sA + STAGES * a_stage_ws<TRANS>();
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * b_stage_ws<TRANS, NT>());
  uint64_t* empty = full + STAGES;

  int nt_idx, mt_idx, split;
  decode_unit(g, blockIdx.x, BN, nt_idx, mt_idx, split);
  const int64_t m0 = static_cast<int64_t>(mt_idx) * BM;
  const int64_t n0 = static_cast<int64_t>(nt_idx) * BN;
  int64_t kt_lim = g.ktiles;
  if (g.tri_b) kt_lim = i64min(kt_lim, (i64min(g.K, n0 + BN) + BK - 1) / BK);
  int64_t kt0 = g.ktiles * split / g.splits;
  int64_t kt1 = g.ktiles * (split + 1) / g.splits;
  kt1 = min(kt1, kt_lim);
  kt0 = min(kt0, kt1);
  const int64_t nkt = kt1 - kt0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCONS);
    }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp >= NCONS) {
    // ------------------------------------------------ producer warpgroup
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::);
    if (warp != NCONS) return;
    const int64_t rows_m = i64min(BM, g.M - m0);
    const int64_t cols_n = i64min(BN, g.N - n0);
    for (int64_t it = 0; it < nkt; ++it) {
      const int s = static_cast<int>(it % STAGES);
      const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
      mbar_wait(&empty[s], ph ^ 1u);
      const int64_t k0 = (kt0 + it) * BK;
      if constexpr (TRANS) {
        double* a_st = sA + s * a_stage_ws<TRANS>();
        double* b_st = sB + s * b_stage_ws<TRANS, NT>();
        if (lane == 0) {
          mbar_arrive_expect_tx(&full[s], sizeof(double) * (a_stage_ws<TRANS>() + b_stage_ws<TRANS, NT>()));
          tma_load_2d(a_st, &tmA, static_cast<int>(k0), static_cast<int>(m0), &full[s]);
          tma_load_2d(a_st + BM * 16, &tmA, static_cast<int>(k0 + 16), static_cast<int>(m0), &full[s]);
          tma_load_2d(b_st, &tmB, static_cast<int>(k0), static_cast<int>(n0), &full[s]);
          tma_load_2d(b_st + BN * 16, &tmB, static_cast<int>(k0 + 16), static_cast<int>(n0), &full[s]);
        }
        __syncwarp();
        continue;
      }
      const int kv = static_cast<int>(i64min(BK, g.K - k0));
      const uint32_t bytes_k = static_cast<uint32_t>(((kv * 8) + 15) & ~15);
      int na;
      uint32_t bytes_a;
      if constexpr (!TRANS) {
        na = kv;
        bytes_a = static_cast<uint32_t>(((rows_m * 8) + 15) & ~15);
      } else {
        na = static_cast<int>(rows_m);
        bytes_a = bytes_k;
      }
      // B: two swizzled tensor boxes (zero-filled beyond K / N)
      if (lane == 0)
        mbar_arrive_expect_tx(&full[s], na * bytes_a + static_cast<uint32_t>(sizeof(double) * b_stage_ws<TRANS, NT>()));
      __syncwarp();
      double* a_st = sA + s * a_stage_ws<TRANS>();
      double* b_st = sB + s * b_stage_ws<TRANS, NT>();
      for (int c = lane; c < na; c += 32) {
        if constexpr (!TRANS) bulk_g2s(a_st + c * LDA_NN, g.A + (k0 + c) * g.lda + m0, bytes_a, &full[s]);
        else bulk_g2s(a_st + c * LDK, g.A + (m0 + c) * g.lda + k0, bytes_a, &full[s]);
      }
      if (lane == 0) {
        tma_load_2d(b_st, &tmB, static_cast<int>(k0), static_cast<int>(n0), &full[s]);
        tma_load_2d(b_st + BN * 16, &tmB, static_cast<int>(k0 + 16), static_cast<int>(n0), &full[s]);
      }
    }
    return;
  }

  // -------------------------------------------------- consumer warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::);
  const int wm = warp & 3, wn = warp >> 2;
  const int g4 = lane >> 2, t4 = lane & 3;
  const bool do_sumsq = (!TRANS) && g.sumsq != nullptr && nt_idx == 0 && wn == 0;
  double rowmask[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) rowmask[i] = (m0 + wm * 32 + i * 8 + g4 < g.M) ? 1.0 : 0.0;
  // NN: B arrives swizzled; natural k = 4*ks + t4 -> chunk (kk >> 1) ^ (row & 7)
  int bsw[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int kk = 4 * u + t4;
    bsw[u] = (((kk >> 1) ^ g4) << 1) | (kk & 1);
  }

  double acc[4][NT][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ss = 0.0;

  for (int64_t it = 0; it < nkt; ++it) {
    const int s = static_cast<int>(it % STAGES);
    const uint32_t ph = static_cast<uint32_t>((it / STAGES) & 1);
    mbar_wait(&full[s], ph);
    const double* a = sA + s * a_stage_ws<TRANS>();
    const double* b = sB + s * b_stage_ws<TRANS, NT>();
    const int kv = static_cast<int>(i64min(BK, g.K - (kt0 + it) * BK));
    if constexpr (TRANS) {
      // Swizzled [k-half][row][16] tiles; the K tail is zero-filled by TMA.
      // k order inside a step: {2u, 2u+1, 2u+8, 2u+9} so the 16 lanes of a
      // half-warp hit 16 distinct bank pairs under the 128B XOR swizzle.
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        const int kh = ks >> 2, u = ks & 3;
        const int coff = (((u + 4 * (t4 >> 1)) ^ g4) << 1) | (t4 & 1);
        double af[4], bf[NT];
#pragma unroll
        for (int i = 0; i < 4; ++i) af[i] = a[kh * (BM * 16) + (wm * 32 + i * 8 + g4) * 16 + coff];
#pragma unroll
        for (int j = 0; j < NT; ++j) bf[j] = b[kh * (BN * 16) + (wn * NT * 8 + j * 8 + g4) * 16 + coff];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    } else if (kv == BK) {
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
        for (int j = 0; j < NT; ++j) bf[j] = b[(ks >> 2) * (BN * 16) + (wn * NT * 8 + j * 8 + g4) * 16 + bsw[ks & 3]];
        if (do_sumsq) {
#pragma unroll
          for (int i = 0; i < 4; ++i) ss = fma(af[i] * rowmask[i], af[i], ss);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    } else {
      for (int ks = 0; ks < BK / 4; ++ks) {
        const bool kin = ks * 4 + t4 < kv;
        double af[4], bf[NT];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int mrow = wm * 32 + i * 8 + g4;
          double v;
          if constexpr (!TRANS) v = a[(ks * 4 + t4) * LDA_NN + mrow];
          else v = a[mrow * LDK + ks * 4 + t4];
          af[i] = kin ? v : 0.0;
        }
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          bf[j] = b[(ks >> 2) * (BN * 16) + (wn * NT * 8 + j * 8 + g4) * 16 + bsw[ks & 3]];
        }
        if (do_sumsq) {
#pragma unroll
          for (int i = 0; i < 4; ++i) ss = fma(af[i] * rowmask[i], af[i], ss);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

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

  if ((!TRANS) && g.sumsq != nullptr && nt_idx == 0) {
    __shared__ double red[NCONS];
    const double v = warp_sum(ss);
    if (lane == 0) red[warp] = v;
    asm volatile("bar.sync 1, %0;\n" ::"n"(NCONS * 32));
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < NCONS; ++w) tot += red[w];
      g.sumsq[static_cast<int64_t>(split) * g.mtiles + mt_idx] = tot;
    }
  }
}

// C(m, n) = sum_{s < S} part[s][n][m], fixed order.
__global__ void reduce_splits_kernel(const double* __restrict__ part, int64_t M, int64_t N, int S,
                                     double* __restrict__ C, int64_t ldc, int sym) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = e / M, m = e % M;
    if (sym && m > n) continue;
    double s = 0.0;
    for (int k = 0; k < S; ++k) s += part[k * total + e];
    C[n * ldc + m] = s;
    if (sym) C[m * ldc + n] = s;
  }
}

// Lower triangle <- upper triangle (sym GEMM with a direct store).
__global__ void symmetrize_kernel(double* __restrict__ C, int64_t N, int64_t ldc) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < N * N;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = e / N, m = e % N;
    if (m > n) C[n * ldc + m] = C[m * ldc + n];
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
  static std::atomic<uint64_t> configured{0};
  if (attr_pending(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_done(configured);
  }
  kern<<<static_cast<unsigned>(grid), NTHREADS, smem, st>>>(g);
  count_launch();
  return cudaGetLastError();
}

template <bool TRANS, int NT>
cudaError_t launch_tma(const GemmParams& g, const CUtensorMap& ta, const CUtensorMap& tb, int64_t grid,
                       cudaStream_t st) {
  auto kern = gemm_f64_tma_kernel<TRANS, NT>;
  constexpr size_t smem = smem_bytes_ws<TRANS, NT>();
  static std::atomic<uint64_t> configured{0};
  if (attr_pending(configured)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    attr_done(configured);
  }
  kern<<<static_cast<unsigned>(grid), WS_THREADS, smem, st>>>(g, ta, tb);
  count_launch();
  return cudaGetLastError();
}

// mode: 0 cp.async (any alignment), 1 TMA bulk (16B-aligned operands)
template <bool TRANS>
cudaError_t dispatch_nt(int mode, int NT, const GemmParams& g, const CUtensorMap& ta, const CUtensorMap& tb,
                        int64_t grid, cudaStream_t st) {
  if (mode == 1) {
    switch (NT) {
      case 1: return launch_tma<TRANS, 1>(g, ta, tb, grid, st);
      case 2: return launch_tma<TRANS, 2>(g, ta, tb, grid, st);
      case 3: return launch_tma<TRANS, 3>(g, ta, tb, grid, st);
      case 4: return launch_tma<TRANS, 4>(g, ta, tb, grid, st);
      case 5: return launch_tma<TRANS, 5>(g, ta, tb, grid, st);
      case 6: return launch_tma<TRANS, 6>(g, ta, tb, grid, st);
      case 7: return launch_tma<TRANS, 7>(g, ta, tb, grid, st);
      default: return launch_tma<TRANS, 8>(g, ta, tb, grid, st);
    }
  }
  switch (NT) {
    case 1: return launch_one<TRANS, 1, false>(g, grid, st);
    case 2: return launch_one<TRANS, 2, false>(g, grid, st);
    case 3: return launch_one<TRANS, 3, false>(g, grid, st);
    case 4: return launch_one<TRANS, 4, false>(g, grid, st);
    case 5: return launch_one<TRANS, 5, false>(g, grid, st);
    case 6: return launch_one<TRANS, 6, false>(g, grid, st);
    case 7: return launch_one<TRANS, 7, false>(g, grid, st);
    default: return launch_one<TRANS, 8, false>(g, grid, st);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D FP64 tensor map over a column-major (rows x cols, ld) matrix with a
// box of 16 rows (128 bytes, the swizzle span) x box_cols columns.
bool make_tmap(CUtensorMap* tm, const double* base, int64_t rows, int64_t cols, int64_t ld, int box_cols) {
  auto fn = encoder();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  cuuint32_t box[2] = {16u, static_cast<cuuint32_t>(box_cols)};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace

GemmPlan plan_gemm(int64_t M, int64_t N, int64_t K, int num_sms, int force_splits, bool sym) {
  GemmPlan p{};
  p.ntiles = static_cast<int>((N + 127) / 128);
  if (p.ntiles < 1) p.ntiles = 1;
  p.nt = static_cast<int>((N + 16 * p.ntiles - 1) / (16 * p.ntiles));
  p.nt = std::max(1, std::min(8, p.nt));
  p.mtiles = static_cast<int>((M + BM - 1) / BM);
  p.ktiles = (K + BK - 1) / BK;
  p.sym = sym && M == N;
  int64_t units = static_cast<int64_t>(p.mtiles) * p.ntiles;
  if (p.sym) {
    units = 0;
    for (int mt = 0; mt < p.mtiles; ++mt)
      for (int nt = 0; nt < p.ntiles; ++nt)
        if (static_cast<int64_t>(mt) * BM < static_cast<int64_t>(nt + 1) * 16 * p.nt) ++units;
  }
  p.units = units;
  int best = 1;
  if (force_splits > 0) {
    best = static_cast<int>(std::min<int64_t>(force_splits, std::max<int64_t>(1, p.ktiles)));
  } else if (units < 12 * num_sms && p.ktiles > 1) {
    // Split-K count with the fullest last wave, keeping >= 4 K-tiles per
    // split (deterministic fixed-order reduction afterwards). Among counts
    // within 1% of the best wave efficiency, the smallest wins.
    const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(p.ktiles / 4, 256));
    auto eff_of = [&](int64_t s) {
      const int64_t work = units * s;
      const int64_t waves = (work + num_sms - 1) / num_sms;
      return static_cast<double>(work) / static_cast<double>(waves * num_sms) - 0.002 * (waves - 1);
    };
    double best_eff = -1.0;
    for (int64_t s = 1; s <= max_s; ++s) best_eff = std::max(best_eff, eff_of(s));
    for (int64_t s = 1; s <= max_s; ++s)
      if (eff_of(s) >= best_eff - 0.01) {
        best = static_cast<int>(s);
        break;
      }
  }
  p.splits = best;
  return p;
}

cudaError_t gemm_f64(bool trans_a, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                     const double* B, int64_t ldb, double* C, int64_t ldc, double* workspace,
                     size_t workspace_bytes, double* sumsq_partials, const GemmPlan& p, cudaStream_t st,
                     bool tri_b) {
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
  int mode = v16 ? 1 : 0;
  CUtensorMap ta{}, tb{};
  if (mode == 1) {
    const bool dims_ok = K < (int64_t(1) << 31) && M < (int64_t(1) << 31) && N < (int64_t(1) << 31);
    bool ok = dims_ok && make_tmap(&tb, B, K, N, ldb, 16 * p.nt);
    if (ok && trans_a) ok = make_tmap(&ta, A, K, M, lda, BM);
    if (!ok) mode = 0;
  }
  // The cp.async kernel computes every tile; the TMA kernel honours sym/tri_b.
  g.sym = (mode == 1 && p.sym) ? 1 : 0;
  g.tri_b = (mode == 1 && tri_b && K == N) ? 1 : 0;
  g.units = g.sym ? p.units : static_cast<int64_t>(p.ntiles) * p.mtiles;
  const int64_t grid = g.units * p.splits;
  cudaError_t e = trans_a ? dispatch_nt<true>(mode, p.nt, g, ta, tb, grid, st)
                          : dispatch_nt<false>(mode, p.nt, g, ta, tb, grid, st);
  if (e != cudaSuccess) return e;
  if (p.splits > 1) {
    const int64_t total = M * N;
    const int64_t blocks = std::min<int64_t>((total + 255) / 256, 148 * 16);
    reduce_splits_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(workspace, M, N, p.splits, C, ldc,
                                                                          p.sym ? 1 : 0);
    count_launch();
    e = cudaGetLastError();
  } else if (p.sym) {
    const int64_t blocks = std::min<int64_t>((M * N + 255) / 256, 148 * 4);
    symmetrize_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(C, M, ldc);
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
