// Staging-copy variants on the GPU box host: pageable -> pinned in 512 KB column chunks (what the staging ring
// copies: one column of a 65536-row panel per memcpy), with glibc memcpy and with explicit non-temporal stores,
// alone and while the copy engine reads another pinned buffer (the H2D DMA of the previous slot).
// nvcc -O3 -Xcompiler -mavx2 -o hostcopy_nt hostcopy_nt.cu
#include <cuda_runtime.h>
#include <immintrin.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
static void nt_copy(char* dst, const char* src, size_t n) {
  size_t i = 0;
  while ((reinterpret_cast<uintptr_t>(dst + i) & 31) && i < n) { dst[i] = src[i]; ++i; }
  for (; i + 128 <= n; i += 128) {
    __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}
__attribute__((target("avx512f"))) static void nt_copy512(char* dst, const char* src, size_t n) {
  size_t i = 0;
  while ((reinterpret_cast<uintptr_t>(dst + i) & 63) && i < n) { dst[i] = src[i]; ++i; }
  for (; i + 256 <= n; i += 256) {
    __m512i a = _mm512_loadu_si512(src + i), b = _mm512_loadu_si512(src + i + 64);
    __m512i c = _mm512_loadu_si512(src + i + 128), d = _mm512_loadu_si512(src + i + 192);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i), a);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 64), b);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 128), c);
    _mm512_stream_si512(reinterpret_cast<__m512i*>(dst + i + 192), d);
  }
  for (; i < n; ++i) dst[i] = src[i];
  _mm_sfence();
}
int main() {
  const size_t total = size_t{8} << 30, slot = size_t{128} << 20, chunk = size_t{512} << 10;
  std::vector<char> src(total);
  std::memset(src.data(), 1, total);
  char *pin = nullptr, *pin2 = nullptr, *dev = nullptr;
  cudaMallocHost(&pin, slot);
  cudaMallocHost(&pin2, slot);
  std::memset(pin2, 2, slot);
  cudaMalloc(&dev, slot);
  cudaStream_t cs;
  cudaStreamCreate(&cs);
  const int T = std::min(16u, std::max(1u, std::thread::hardware_concurrency()));
  for (int dma = 0; dma < 2; ++dma)
    for (int mode = 0; mode < (__builtin_cpu_supports("avx512f") ? 3 : 2); ++mode) {
      std::atomic<bool> stop{false};
      std::atomic<long> dma_bytes{0};
      std::thread feeder;
      if (dma) feeder = std::thread([&] {
        while (!stop.load()) {
          cudaMemcpyAsync(dev, pin2, slot, cudaMemcpyHostToDevice, cs);
          cudaStreamSynchronize(cs);
          dma_bytes += static_cast<long>(slot);
        }
      });
      auto t0 = std::chrono::steady_clock::now();
      for (size_t off = 0; off < total; off += slot) {
        std::vector<std::thread> th;
        const size_t nchunks = slot / chunk;
        for (int t = 0; t < T; ++t)
          th.emplace_back([&, t] {
            for (size_t c = nchunks * t / T; c < nchunks * (t + 1) / T; ++c) {
              if (mode == 0) std::memcpy(pin + c * chunk, src.data() + off + c * chunk, chunk);
              else if (mode == 1) nt_copy(pin + c * chunk, src.data() + off + c * chunk, chunk);
              else nt_copy512(pin + c * chunk, src.data() + off + c * chunk, chunk);
            }
          });
        for (auto& x : th) x.join();
      }
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      stop = true;
      if (dma) feeder.join();
      std::printf("%s 512 KB chunks, %d threads, %s: copy %.1f GB/s%s", mode == 0 ? "memcpy " : mode == 1 ? "nt_copy(avx2)" : "nt_copy(avx512)", T,
                  dma ? "with concurrent H2D" : "alone", total / s / 1e9, dma ? "" : "\n");
      if (dma) std::printf(", H2D meanwhile %.1f GB/s\n", dma_bytes.load() / s / 1e9);
    }
  return 0;
}
