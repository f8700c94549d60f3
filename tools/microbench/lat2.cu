// Costs (clk, thread 0 of a 1024-thread CTA) of the mbarrier / proxy primitives.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__global__ void k(long long* t, double* g, int n, int which) {
  __shared__ uint64_t bar[4];
  __shared__ double buf[1024];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar[i])), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  buf[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  if (which == 0) for (int i = 0; i < n; ++i) {
    buf[i & 1023] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  long long t1 = clock64();
  if (which == 1) for (int i = 0; i < n; ++i) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[0])), "r"(0) : "memory");
  }
  long long t2 = clock64();
  if (which == 2) for (int i = 0; i < n; ++i) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[1])), "r"(0) : "memory");
  }
  long long t3 = clock64();
  if (which == 3) for (int i = 0; i < n; ++i) {
    buf[i & 1023] = i;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[2])), "r"(0) : "memory");
  }
  long long t4 = clock64();
  if (which == 4) for (int i = 0; i < n; ++i) {
    g[i] = i;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[3])), "r"(0) : "memory");
  }
  long long t5 = clock64();
  if (which == 5) for (int i = 0; i < n; ++i) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[0])), "r"(256) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sa(buf + 512)), "r"(sa(buf)), "r"(256), "r"(sa(&bar[0])) : "memory");
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(sa(&bar[0])), "r"(i & 1) : "memory");
  }
  long long t6 = clock64();
  t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5;
}
int main() {
  long long* t; double* g; cudaMallocManaged(&t, 8 * 8); cudaMalloc(&g, 8 * 4096);
  const int n = 64;
  long long res[6];
  for (int w = 0; w < 5; ++w) {
    k<<<1, 1024>>>(t, g, n, w); k<<<1, 1024>>>(t, g, n, w);
    cudaError_t e = cudaDeviceSynchronize();
    printf("test %d err=%s\n", w, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    res[w] = t[w];
  }
  for (int w = 0; w < 6; ++w) t[w] = res[w];
  const char* nm[6] = {"sts+fence.proxy.async", "arrive.expect_tx (release)", "arrive.expect_tx.relaxed",
                       "sts+arrive.expect_tx", "stg+arrive.expect_tx", "expect+bulk s2s+wait"};
  for (int i = 0; i < 5; ++i) printf("  %-28s %.1f clk\n", nm[i], double(t[i]) / n);
}
