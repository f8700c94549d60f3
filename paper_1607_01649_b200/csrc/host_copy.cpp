// Host-side staging copy for the pinned ring (rfgpu_api.cu: host_copy_cols): pageable caller memory into a
// pinned slot that only the copy engine will read. Non-temporal stores: the destination lines are not read
// for ownership and do not evict the source stream from the caches, which matters because the staging copy
// shares the host's memory system with the DMA of the previous slot (tools/microbench/hostcopy_nt.cu).
#include <cstddef>
#include <cstdint>
#include <cstring>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

namespace rfgpu {

#if defined(__x86_64__)
__attribute__((target("avx2"))) static void stream_copy_avx2(char* dst, const char* src, size_t n) {
  size_t i = 0;
  const size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
  if (head) {
    const size_t h = head < n ? head : n;
    std::memcpy(dst, src, h);
    i = h;
  }
  for (; i + 128 <= n; i += 128) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    const __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  if (i < n) std::memcpy(dst + i, src + i, n - i);
  _mm_sfence();
}
#endif

// dst is written once and next read by a DMA engine: stream it past the caches when the CPU can.
void host_stream_copy(void* dst, const void* src, size_t bytes) {
#if defined(__x86_64__)
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2 && bytes >= 4096) {
    stream_copy_avx2(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
    return;
  }
#endif
  std::memcpy(dst, src, bytes);
}

}  // namespace rfgpu
