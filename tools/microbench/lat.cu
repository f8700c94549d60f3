// Dependent-chain latencies (clk) of the FP64 ops the Jacobi rounds are made of.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* t, double a, double b, int n) {
  __shared__ double s[1024];
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { s[i] = 1.0 + i * 1e-9; idx[i] = (i * 7 + 1) & 1023; }
  __syncthreads();
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x + y;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = y / x;
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x);
  long long t5 = clock64();
  int j = threadIdx.x;
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1);
  long long t7 = clock64();
  __syncthreads();
  long long t8 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t9 = clock64();
  out[threadIdx.x] = x + j;
  if (threadIdx.x == 0) {
    t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; t[5] = t6 - t5; t[6] = t7 - t6;
    t[7] = t9 - t8;
  }
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 8 * 1024); cudaMallocManaged(&t, 8 * 16);
  const char* nm[8] = {"dfma", "dadd", "dsqrt", "ddiv", "drsqrt", "lds(int chase)", "shfl.xor f64 + dadd", "syncthreads"};
  for (int thr : {32, 1024}) {
    const int n = 256;
    lat<<<1, thr>>>(o, t, 1.0000001, 0.999999, n);
    lat<<<1, thr>>>(o, t, 1.0000001, 0.999999, n);
    cudaDeviceSynchronize();
    printf("blockDim %d:\n", thr);
    for (int i = 0; i < 8; ++i) printf("  %-22s %.1f clk\n", nm[i], double(t[i]) / n);
  }
  return 0;
}
