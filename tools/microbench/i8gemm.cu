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

template <int BN>
__global__ void __launch_bounds__(192, 1) i8gemm(const __grid_constant__ CUtensorMap ta,
                                                 const __grid_constant__ CUtensorMap tb, int M, int N, int K,
                                                 int32_t* C) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + STAGES * BM * BK;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * BN * BK);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntn = N / BN;
  const int m0 = (blockIdx.x / ntn) * BM, n0 = (blockIdx.x % ntn) * BN;
  const int nk = K / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    mb_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(BN < 32 ? 32 : BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0 && lane == 0) {
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mb_wait(&empty[s], ph ^ 1);
      mb_expect(&full[s], (BM + BN) * BK);
      tma2d(sA + s * BM * BK, &ta, &full[s], kb * BK, m0);
      tma2d(sB + s * BN * BK, &tb, &full[s], kb * BK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                           (static_cast<uint32_t>(BM >> 4) << 24);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mb_wait(&full[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kk = 0; kk < BK / 32; ++kk) {
        const uint64_t da = sdesc(sA + s * BM * BK + kk * 32);
        const uint64_t db = sdesc(sB + s * BN * BK + kk * 32);
        const uint32_t acc = (kb | kk) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       su32(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(done))
                 : "memory");
  } else if (warp >= 2) {
    mb_wait(done, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = m0 + q * 32 + lane;
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      const uint32_t ta_ = tmem + (static_cast<uint32_t>(q * 32) << 16) + c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%"
          "19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
            "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(ta_));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < M)
        for (int j = 0; j < 32; ++j) C[static_cast<size_t>(row) * N + n0 + c + j] = static_cast<int32_t>(r[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN < 32 ? 32 : BN));
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void tmap(CUtensorMap* tm, const void* base, int rows, int K, int box_rows) {
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("tmap error %d\n", r);
}

template <int BN>
void run(int M, int N, int K) {
  std::vector<int8_t> a(static_cast<size_t>(M) * K), b(static_cast<size_t>(N) * K);
  srand(1);
  for (auto& x : a) x = static_cast<int8_t>((rand() % 255) - 127);
  for (auto& x : b) x = static_cast<int8_t>((rand() % 255) - 127);
  int8_t *da, *db;
  int32_t* dc;
  cudaMalloc(&da, a.size());
  cudaMalloc(&db, b.size());
  cudaMalloc(&dc, sizeof(int32_t) * static_cast<size_t>(M) * N);
  cudaMemcpy(da, a.data(), a.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size(), cudaMemcpyHostToDevice);
  CUtensorMap ta, tb;
  tmap(&ta, da, M, K, BM);
  tmap(&tb, db, N, K, BN);
  const size_t smem = STAGES * (BM + BN) * BK + 1024 + 256;
  cudaFuncSetAttribute(i8gemm<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  const int grid = (M / BM) * (N / BN);
  i8gemm<BN><<<grid, 192, smem>>>(ta, tb, M, N, K, dc);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("BN=%d launch error: %s\n", BN, cudaGetErrorString(e));
    exit(1);
  }
  std::vector<int32_t> c(static_cast<size_t>(M) * N);
  cudaMemcpy(c.data(), dc, sizeof(int32_t) * c.size(), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int t = 0; t < 2000; ++t) {
    const int i = (t * 7919) % M, j = (t * 104729) % N;
    int64_t s = 0;
    for (int k = 0; k < K; ++k) s += static_cast<int64_t>(a[static_cast<size_t>(i) * K + k]) * b[static_cast<size_t>(j) * K + k];
    if (s != c[static_cast<size_t>(i) * N + j]) {
      if (bad < 5) printf("mismatch (%d,%d): got %d want %lld\n", i, j, c[static_cast<size_t>(i) * N + j], (long long)s);
      ++bad;
    }
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 5;
  for (int r = 0; r < reps; ++r) i8gemm<BN><<<grid, 192, smem>>>(ta, tb, M, N, K, dc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  printf("BN=%d M=%d N=%d K=%d: %s (%d bad of 2000), %.3f ms, %.1f TOPS\n", BN, M, N, K, bad ? "WRONG" : "ok", bad, ms,
         2.0 * M * N * static_cast<double>(K) / ms / 1e9);
  cudaFree(da);
  cudaFree(db);
  cudaFree(dc);
}

int main() {
  run<64>(128 * 296, 256, 4096);
  run<128>(128 * 296, 256, 4096);
  run<256>(128 * 296, 256, 4096);
  run<256>(128 * 1184, 256, 4096);
  return 0;
}
