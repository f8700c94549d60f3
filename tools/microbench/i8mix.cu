// INT8 tensor throughput on this B200 by MMA shape: tcgen05.mma kind::i8
// (M=128, K=32, N per mode) back to back on shared-memory operands, one
// issuing thread per CTA, one CTA per SM, no global traffic. Modes: N = 256,
// 192, 128, 64, and "mix" = the digit kernel's 10 MMAs per K step (N = 256,
// 192, 256, 128, 256, 64, 256, 192, 128, 64 into TMEM groups s + t).
// Reports TOPS (2*M*N*K per MMA).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void __launch_bounds__(128, 1) peak(int iters, int* sink, int mode) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) sm[i] = static_cast<uint8_t>(i * 7);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
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
    auto mma = [&](int n, int col, int kk, uint32_t acc) {
      const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((static_cast<uint32_t>(n) >> 3) << 17) | ((128u >> 4) << 24);
      const uint64_t da = desc(sm + kk * 32), db = desc(sm + 128 * 128 + kk * 32);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + col),
                   "l"(da), "l"(db), "r"(idesc), "r"(acc));
    };
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = it | kk;
        if (mode == 0) {  // mix: A digit s, B digits t0.., group s + t0 at column 64 (s + t0)
          mma(256, 0, kk, acc); mma(192, 256, kk, acc);
          mma(256, 64, kk, acc); mma(128, 320, kk, acc);
          mma(256, 128, kk, acc); mma(64, 384, kk, acc);
          mma(256, 192, kk, acc); mma(192, 256, kk, acc);
          mma(128, 320, kk, acc); mma(64, 384, kk, acc);
        } else {
          mma(mode, 0, kk, acc);
        }
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
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}
int main(int argc, char** argv) {
  int* sink;
  cudaMalloc(&sink, 4);
  const int smem = (128 + 256) * 128 + 1024;
  cudaFuncSetAttribute(peak, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode : {256, 192, 128, 64, 0}) {
    const int iters = mode == 0 ? 2000 : 20000;
    const double cols = mode == 0 ? 1792.0 : mode;  // N summed over one K step's MMAs
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
    const double ops = 2.0 * 128 * cols * 32 * 4.0 * iters * sms;
    printf("mode %s: burst %.1f TOPS (%.3f ms, err=%s)", mode == 0 ? "mix" : std::to_string(mode).c_str(),
           ops / best / 1e9, best, cudaGetErrorString(cudaGetLastError()));
    const int reps = static_cast<int>(3000.0f / best) + 1;
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) peak<<<sms, 128, smem>>>(iters, sink, mode);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float total;
    cudaEventElapsedTime(&total, a, b);
    printf("  sustained %.1f TOPS (%.0f ms)\n", ops * reps / total / 1e9, total);
  }
  return 0;
}
