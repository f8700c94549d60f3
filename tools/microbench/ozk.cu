// Feasibility probe: tcgen05.mma kind::i8 GEMM (int8 x int8 -> int32 in TMEM),
// both operands K-major, TMA 128B-swizzled tiles, warp-specialised
// (TMA warp, MMA warp, 4 epilogue warps). C[m][n] = sum_k A[m][k] * B[n][k].
// Checks a sample of outputs against the CPU and reports TOPS.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int BM = 128, BK = 128, STAGES = 4;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(
          su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          su32(dst)),
      "l"(tm), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t sdesc(const void* p) {
  uint64_t d = 0;
  d |= (static_cast<uint64_t>(su32(p)) >> 4) & 0x3FFF;
  d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO: 8 rows x 128 B
  d |= static_cast<uint64_t>(1) << 46;            // descriptor version (sm100)
  d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
  return d;
}


// Ozaki-shaped: S int8 slices per operand, accumulators grouped by d = s + t
// (t = 0..S-1, s = 0..S-1, s + t <= S - 1: S groups, triangular truncation).
// A slices: [S][M][K], B slices: [S][N][K]; TMEM: S groups x BN columns.
template <int S, int BN, int BKB, int NST>
__global__ void __launch_bounds__(192, 1) ozk(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                              int M, int N, int K, double* C) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int ASZ = S * BM * BKB, BSZ = S * BN * BKB;
  uint8_t* sA = smem;
  uint8_t* sB = sA + NST * ASZ;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + NST * BSZ);
  uint64_t* empty = full + NST;
  uint64_t* done = empty + NST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  constexpr int TCOLS = (S * BN <= 32) ? 32 : (S * BN <= 64) ? 64 : (S * BN <= 128) ? 128 : (S * BN <= 256) ? 256 : 512;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = N / BN;
  const int m0 = (blockIdx.x / ntn) * BM, n0 = (blockIdx.x % ntn) * BN;
  const int nk = K / BKB;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  constexpr uint64_t SW = BKB == 128 ? 2 : (BKB == 64 ? 4 : 6);
  constexpr uint64_t SBO = 8 * BKB;
  auto desc = [&](const void* p) {
    uint64_t d = 0;
    d |= (static_cast<uint64_t>(su32(p)) >> 4) & 0x3FFF;
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(SBO >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= SW << 61;
    return d;
  };
  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NST;
      const uint32_t ph = (kb / NST) & 1;
      mb_wait(&empty[st], ph ^ 1);
      mb_expect(&full[st], ASZ + BSZ);
#pragma unroll
      for (int s = 0; s < S; ++s) {
        tma2d(sA + st * ASZ + s * BM * BKB, &ta, &full[st], kb * BKB, s * M + m0);
        tma2d(sB + st * BSZ + s * BN * BKB, &tb, &full[st], kb * BKB, s * N + n0);
      }
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                           (static_cast<uint32_t>(BM >> 4) << 24);
    for (int kb = 0; kb < nk; ++kb) {
      const int st = kb % NST;
      const uint32_t ph = (kb / NST) & 1;
      mb_wait(&full[st], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kk = 0; kk < BKB / 32; ++kk) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
#pragma unroll
          for (int t = 0; t + s < S; ++t) {
            const uint64_t da = desc(sA + st * ASZ + s * BM * BKB + kk * 32);
            const uint64_t db = desc(sB + st * BSZ + t * BN * BKB + kk * 32);
            const uint32_t acc = (kb | kk | t) ? 1u : 0u;  // first product of a group (t = 0 at s = d) clears
            const uint32_t first = (kb == 0 && kk == 0 && s == 0) ? 0u : 1u;
            (void)acc;
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + (s + t) * BN),
                "l"(da), "l"(db), "r"(idesc), "r"(first));
          }
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&empty[st]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(done))
                 : "memory");
  } else if (warp >= 2) {
    mb_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    for (int c = 0; c < BN; c += 16) {
      double acc[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[j] = 0.0;
#pragma unroll
      for (int g = S - 1; g >= 0; --g) {
        uint32_t r[16];
        const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + g * BN + c;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const double sc = ldexp(1.0, -7 * (g + 2));
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = fma(static_cast<double>(static_cast<int32_t>(r[j])), sc, acc[j]);
      }
      if (row < M)
        for (int j = 0; j < 16; ++j) C[static_cast<size_t>(row) * N + n0 + c + j] = acc[j];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void tmap(CUtensorMap* tm, const void* base, long rows, int K, int box_rows, int bkb) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(bkb), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUtensorMapSwizzle sw = bkb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : (bkb == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
  CUresult r = enc()(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("tmap error %d\n", r);
}

__global__ void fill_i8(int8_t* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    uint32_t h = static_cast<uint32_t>(i) * 2654435761u ^ seed ^ static_cast<uint32_t>(i >> 32) * 40503u;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    p[i] = static_cast<int8_t>(static_cast<int>(h % 255u) - 127);
  }
}

template <int S, int BN, int BKB, int NST>
void run(int M, int N, int K, bool check) {
  std::vector<int8_t> a, b;
  int8_t *da, *db;
  double* dc;
  const size_t na = static_cast<size_t>(S) * M * K, nb = static_cast<size_t>(S) * N * K;
  cudaMalloc(&da, na);
  cudaMalloc(&db, nb);
  cudaMalloc(&dc, sizeof(double) * static_cast<size_t>(M) * N);
  fill_i8<<<1184, 256>>>(da, na, 1u);
  fill_i8<<<1184, 256>>>(db, nb, 7u);
  if (check) {
    a.resize(na);
    b.resize(nb);
    cudaMemcpy(a.data(), da, na, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), db, nb, cudaMemcpyDeviceToHost);
  }
  CUtensorMap ta, tb;
  tmap(&ta, da, static_cast<long>(S) * M, K, BM, BKB);
  tmap(&tb, db, static_cast<long>(S) * N, K, BN, BKB);
  const size_t smem = NST * S * (BM + BN) * BKB + 1024 + 256;
  cudaFuncSetAttribute(ozk<S, BN, BKB, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const int grid = (M / BM) * (N / BN);
  ozk<S, BN, BKB, NST><<<grid, 192, smem>>>(ta, tb, M, N, K, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("launch error: %s\n", cudaGetErrorString(e));
    exit(1);
  }
  int bad = 0;
  if (check) {
    std::vector<double> c(static_cast<size_t>(M) * N);
    cudaMemcpy(c.data(), dc, sizeof(double) * c.size(), cudaMemcpyDeviceToHost);
    for (int t = 0; t < 300; ++t) {
      const int i = (t * 7919) % M, j = (t * 104729) % N;
      double want = 0.0;
      for (int g = S - 1; g >= 0; --g) {
        long long sg = 0;
        for (int s = 0; s <= g; ++s) {
          const int tt = g - s;
          for (int k = 0; k < K; ++k)
            sg += static_cast<long long>(a[(static_cast<size_t>(s) * M + i) * K + k]) * b[(static_cast<size_t>(tt) * N + j) * K + k];
        }
        want += static_cast<double>(sg) * ldexp(1.0, -7 * (g + 2));
      }
      const double got = c[static_cast<size_t>(i) * N + j];
      if (fabs(got - want) > 1e-12 * fabs(want) + 1e-300) {
        if (bad < 5) printf("mismatch (%d,%d): got %.17g want %.17g\n", i, j, got, want);
        ++bad;
      }
    }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 3;
  for (int r = 0; r < reps; ++r) ozk<S, BN, BKB, NST><<<grid, 192, smem>>>(ta, tb, M, N, K, dc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  const double ops = 2.0 * M * N * static_cast<double>(K) * (S * (S + 1) / 2);
  printf("S=%d BN=%d BKB=%d NST=%d M=%d N=%d K=%d: %s, %.3f ms, %.0f int8 TOPS, FP64-equiv %.1f TF/s\n", S, BN, BKB,
         NST, M, N, K, check ? (bad ? "WRONG" : "ok") : "unchecked", ms, ops / ms / 1e9,
         2.0 * M * N * static_cast<double>(K) / ms / 1e9);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dc);
}

int main() {
  run<7, 64, 64, 2>(128 * 148, 64, 1024, true);
  run<7, 64, 64, 2>(128 * 2048, 256, 4096, false);
  run<7, 64, 32, 4>(128 * 2048, 256, 4096, false);
  run<7, 32, 64, 2>(128 * 2048, 256, 4096, false);
  return 0;
}
