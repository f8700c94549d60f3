// Host copy bandwidth pageable -> pinned (the staging ring's inner loop) and H2D from pinned, GPU box host.
// nvcc -O3 -o hostcopy hostcopy.cu
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
int main() {
  const size_t total = size_t{8} << 30, slot = size_t{512} << 20;
  std::vector<char> src(total);
  std::memset(src.data(), 1, total);
  char* pin = nullptr;
  cudaMallocHost(&pin, slot);
  char* dev = nullptr;
  cudaMalloc(&dev, slot);
  for (int T : {1, 2, 4, 8, 12, 16}) {
    auto t0 = std::chrono::steady_clock::now();
    for (size_t off = 0; off < total; off += slot) {
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          const size_t a = slot * t / T, b = slot * (t + 1) / T;
          std::memcpy(pin + a, src.data() + off + a, b - a);
        });
      for (auto& x : th) x.join();
    }
    double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::printf("pageable->pinned %2d threads: %.1f GB/s\n", T, total / s / 1e9);
  }
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 16; ++i) cudaMemcpy(dev, pin, slot, cudaMemcpyHostToDevice);
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("pinned H2D: %.1f GB/s\n", 16.0 * slot / s / 1e9);
  t0 = std::chrono::steady_clock::now();
  for (size_t off = 0; off < (size_t{4} << 30); off += slot) cudaMemcpy(dev, src.data() + off, slot, cudaMemcpyHostToDevice);
  s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("pageable H2D (driver staging): %.1f GB/s\n", (4.0 * (1 << 30)) / s / 1e9);
  t0 = std::chrono::steady_clock::now();
  cudaHostRegister(src.data(), size_t{4} << 30, cudaHostRegisterDefault);
  s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("cudaHostRegister 4 GiB: %.3f s (%.1f GB/s)\n", s, 4.0 * (1 << 30) / s / 1e9);
  t0 = std::chrono::steady_clock::now();
  for (size_t off = 0; off < (size_t{4} << 30); off += slot) cudaMemcpy(dev, src.data() + off, slot, cudaMemcpyHostToDevice);
  s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("registered H2D: %.1f GB/s\n", (4.0 * (1 << 30)) / s / 1e9);
  t0 = std::chrono::steady_clock::now();
  cudaHostUnregister(src.data());
  s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("cudaHostUnregister: %.3f s\n", s);
  return 0;
}
