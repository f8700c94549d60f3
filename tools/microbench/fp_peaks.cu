// FP64/FP32 pipe-peak microbenchmarks for B200 (sm_100a).
// Measures: DFMA (vector FP64), DMMA via mma.sync m8n8k4 f64, DMMA via
// m16n8k16 f64, FFMA (vector FP32). Prints one JSON line per measurement.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_peaks fp_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678f) out[0] = s;
}

template <int ACC>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int ACC>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - threadIdx.x * 1e-4 + i;
  double c[ACC][4];
#pragma unroll
  for (int i = 0; i < ACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 "
                   "{%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <typename K, typename... Args>
float time_kernel(K kern, int grid, int block, int reps, Args... args) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<grid, block>>>(args...);  // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    kern<<<grid, block>>>(args...);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\"}\n", prop.name, sms, prop.major, prop.minor);
  double* dout; float* fout;
  CK(cudaMalloc(&dout, 64)); CK(cudaMalloc(&fout, 64));
  const int reps = 5;
  for (int blocksPerSm : {1, 2, 4}) {
    for (int threads : {256, 512}) {
      int grid = sms * blocksPerSm;
      int iters = 20000;
      float ms = time_kernel(dfma_kernel<8>, grid, threads, reps, dout, iters, 0.999999, 1e-9);
      double flops = 2.0 * 8 * iters * (double)grid * threads;
      printf("{\"op\": \"DFMA\", \"bps\": %d, \"threads\": %d, \"tflops\": %.2f}\n", blocksPerSm, threads, flops / ms / 1e9);
      ms = time_kernel(ffma_kernel<8>, grid, threads, reps, fout, iters * 4, 0.999999f, 1e-9f);
      flops = 2.0 * 8 * iters * 4 * (double)grid * threads;
      printf("{\"op\": \"FFMA\", \"bps\": %d, \"threads\": %d, \"tflops\": %.2f}\n", blocksPerSm, threads, flops / ms / 1e9);
      ms = time_kernel(dmma884_kernel<8>, grid, threads, reps, dout, iters / 2);
      flops = 2.0 * 8 * 8 * 4 * 8 * (iters / 2) * (double)grid * (threads / 32);
      printf("{\"op\": \"DMMA_m8n8k4\", \"bps\": %d, \"threads\": %d, \"tflops\": %.2f}\n", blocksPerSm, threads, flops / ms / 1e9);
      ms = time_kernel(dmma16816_kernel<4>, grid, threads, reps, dout, iters / 16);
      flops = 2.0 * 16 * 8 * 16 * 4 * (iters / 16) * (double)grid * (threads / 32);
      printf("{\"op\": \"DMMA_m16n8k16\", \"bps\": %d, \"threads\": %d, \"tflops\": %.2f}\n", blocksPerSm, threads, flops / ms / 1e9);
    }
  }
  // single-warp-per-SM DMMA latency-ish probe: 1 warp/SM with dependent chain
  {
    int grid = sms;
    float ms = time_kernel(dmma884_kernel<1>, grid, 32, reps, dout, 20000);
    double cyc = ms * 1e-3 * prop.clockRate * 1e3 / 20000;
    printf("{\"op\": \"DMMA_m8n8k4_dep_chain\", \"cycles_per_mma_at_max_clock\": %.1f}\n", cyc);
    ms = time_kernel(dmma884_kernel<8>, grid, 32, reps, dout, 20000);
    cyc = ms * 1e-3 * prop.clockRate * 1e3 / 20000 / 8;
    printf("{\"op\": \"DMMA_m8n8k4_1warp_8acc\", \"cycles_per_mma_at_max_clock\": %.1f}\n", cyc);
    ms = time_kernel(dmma884_kernel<8>, grid, 128, reps, dout, 20000);
    cyc = ms * 1e-3 * prop.clockRate * 1e3 / 20000 / 8;
    printf("{\"op\": \"DMMA_m8n8k4_4warp_8acc\", \"cycles_per_mma_per_warp_at_max_clock\": %.1f}\n", cyc);
  }
  return 0;
}
