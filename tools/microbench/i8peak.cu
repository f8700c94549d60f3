// INT8 dense tensor peak on this B200: tcgen05.mma kind::i8 (M=128, N=256,
// K=32) back to back on shared-memory operands, one issuing thread per CTA,
// one CTA per SM. No global traffic. Reports TOPS (2*M*N*K per MMA).
//   i8peak [pattern|zero|random]
// pattern (default): one operand tile set holding bytes 7 i, re-used by every MMA (the round-1 figure);
// zero: all-zero operands; random: kSets distinct tile sets of hashed bytes, cycled, so that consecutive
// MMAs see different operands the way a streaming GEMM does (operand toggling costs power, and at the
// power cap power is throughput).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
constexpr int kSets = 4;
constexpr int kSetBytes = (128 + 256) * 128;
__global__ void __launch_bounds__(128, 1) peak(int iters, int* sink, int mode) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < kSets * kSetBytes; i += blockDim.x) {
    uint32_t h = (static_cast<uint32_t>(i) + 0x9E3779B9u * (blockIdx.x + 1)) * 2654435761u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    sm[i] = mode == 0 ? static_cast<uint8_t>((i % kSetBytes) * 7) : mode == 1 ? 0 : static_cast<uint8_t>(h >> 11);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  auto desc = [&](const void* p) {
    uint64_t d = (static_cast<uint64_t>(su32(p)) >> 4) & 0x3FFF;
    d |= 1ull << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;
    return d;
  };
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint8_t* set = sm + (mode == 2 ? (it % kSets) * kSetBytes : 0);
        const uint64_t da = desc(set + kk * 32), db = desc(set + 128 * 128 + kk * 32);
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                     "l"(da), "l"(db), "r"(idesc), "r"(it | kk));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (r == 0x12345) sink[0] = 1;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
  }
}
int main(int argc, char** argv) {
  int mode = 0;
  if (argc > 1) mode = argv[1][0] == 'z' ? 1 : argv[1][0] == 'r' ? 2 : 0;
  const char* mname = mode == 0 ? "pattern" : mode == 1 ? "zero" : "random";
  int* sink;
  cudaMalloc(&sink, 4);
  const int smem = kSets * kSetBytes + 1024;
  cudaFuncSetAttribute(peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  peak<<<sms, 128, smem>>>(100, sink, mode);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    peak<<<sms, 128, smem>>>(iters, sink, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double ops = 2.0 * 128 * 256 * 32 * 4.0 * iters * sms;
  printf("[%s] int8 tcgen05 dense peak: %.1f TOPS (%d SMs, %.3f ms, err=%s)\n", mname, ops / best / 1e9, sms, best,
         cudaGetErrorString(cudaGetLastError()));
  // sustained: back to back for ~4 s (the power cap settles), like MEASURED_PEAKS.json's bf16_tflops_sustained
  const int reps = static_cast<int>(4000.0f / best) + 1;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) peak<<<sms, 128, smem>>>(iters, sink, mode);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float total;
  cudaEventElapsedTime(&total, a, b);
  printf("[%s] int8 tcgen05 dense sustained: %.1f TOPS (%d launches back to back, %.1f ms, err=%s)\n",
         mname, ops * reps / total / 1e9, reps, total, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
