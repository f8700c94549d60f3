// rfgpu C ABI (include/rfgpu.h) and the device-side orchestration of the
// randomized range finder. One call = one reference entry point:
//
//   rfgpu_range_finder  <- randfact::power_range / basic_range
//                          (proj/src/rangefinder.cpp:56-80, :24-30)
//   rfgpu_rsvd          <- randfact::rsvd (proj/src/lowrank.cpp:74-96)
//   rfgpu_row_sketch    <- the G*A pass of randfact::randomized_cur (:351-352)
//   rfgpu_col_id        <- col_id_core (proj/src/lowrank.cpp:51-70)
//
// Everything between the host copies runs on the context's stream; the only
// host round trips are one status read per orth() (CholeskyQR2 accepted or
// Gram-Schmidt fallback) and the final result copies.
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "rfgpu.h"
#include "rfgpu_internal.h"

namespace rfgpu {

static std::atomic<int64_t> g_launches{0};
int64_t launch_counter() { return g_launches.load(); }
void count_launch(int n) { g_launches.fetch_add(n); }

namespace {

__global__ void add_scalar_kernel(double* dst, const double* src) { *dst += *src; }

__global__ void transpose_kernel(const double* __restrict__ in, int64_t rows, int64_t cols, int64_t ldi,
                                 double* __restrict__ out, int64_t ldo) {
  // out(j, i) = in(i, j); in rows x cols
  __shared__ double tile[32][33];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * 32, j0 = static_cast<int64_t>(blockIdx.y) * 32;
  for (int dj = threadIdx.y; dj < 32; dj += blockDim.y) {
    const int64_t i = i0 + threadIdx.x, j = j0 + dj;
    if (i < rows && j < cols) tile[dj][threadIdx.x] = in[j * ldi + i];
  }
  __syncthreads();
  for (int di = threadIdx.y; di < 32; di += blockDim.y) {
    const int64_t j = j0 + threadIdx.x, i = i0 + di;
    if (i < rows && j < cols) out[i * ldo + j] = tile[threadIdx.x][di];
  }
}

__global__ void gather_cols_kernel(const double* __restrict__ A, int64_t lda, int64_t m, const int64_t* __restrict__ idx,
                                   int64_t k, double* __restrict__ C, int64_t ldc) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < m * k;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / m, i = e % m;
    C[j * ldc + i] = A[idx[j] * lda + i];
  }
}

// R(i, :) = A(idx[i] - row0, :) for global row indices owned by this shard
// (rows row0 .. row0 + m_loc - 1), zero otherwise: summed over ranks this
// assembles A(idx, :) of the row-sharded A.
__global__ void gather_rows_kernel(const double* __restrict__ A, int64_t lda, int64_t n, const int64_t* __restrict__ idx,
                                   int64_t k, double* __restrict__ R, int64_t ldr, int64_t row0, int64_t m_loc) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n * k;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / k, i = e % k;
    const int64_t r = idx[i] - row0;
    R[j * ldr + i] = (r >= 0 && r < m_loc) ? A[j * lda + r] : 0.0;
  }
}

// scale row i of X (r x c, ld r) by inv(s_i) with the least_squares cutoff
// (dense.cpp:825-837): 1/s if s > 1e-12 s_max and s > 0, else 0.
__global__ void lsq_scale_kernel(double* __restrict__ X, int64_t r, int64_t c, const double* __restrict__ S) {
  const double cutoff = (r > 0 ? S[0] : 0.0) * 1e-12;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < r * c;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % r;
    const double d = S[i];
    X[e] *= (d > cutoff && d > 0.0) ? 1.0 / d : 0.0;
  }
}

__global__ void add_inplace_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] += x[i];
}

// X(i, j) /= (a_i^2 + b_j^2): the Sylvester solve in the eigenbases.
__global__ void sylvester_scale_kernel(double* __restrict__ X, int64_t k, const double* __restrict__ a,
                                       const double* __restrict__ b) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < k * k;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % k, j = e / k;
    X[e] /= (a[i] * a[i] + b[j] * b[j]);
  }
}

__global__ void f32_to_f64_kernel(const float* __restrict__ x, int64_t rows, int64_t cols, int64_t ldx,
                                  double* __restrict__ y, int64_t ldy) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < rows * cols;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = e % rows, j = e / rows;
    y[j * ldy + i] = static_cast<double>(x[j * ldx + i]);
  }
}

// Shifted CholeskyQR3: G += shift * trace(G) on the diagonal (one CTA), and the reference-drop-rule statistic
// out[0] = min_j r1(j,j) r2(j,j) r3(j,j) / sqrt(trace(G of X)) from the three Cholesky factors' diagonals.
__global__ void shift_diag_kernel(double* __restrict__ G, int c, double shift, double* __restrict__ trace_out) {
  __shared__ double red[32];
  double t = 0.0;
  for (int j = threadIdx.x; j < c; j += blockDim.x) t += G[static_cast<int64_t>(j) * c + j];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    t = 0.0;
    for (unsigned w = 0; w < (blockDim.x >> 5); ++w) t += red[w];
    red[0] = t;
    trace_out[0] = t;
  }
  __syncthreads();
  const double s = shift * red[0];
  for (int j = threadIdx.x; j < c; j += blockDim.x) G[static_cast<int64_t>(j) * c + j] += s;
}
__global__ void rdiag_min_kernel(const double* __restrict__ R1, const double* __restrict__ R2,
                                 const double* __restrict__ R3, int c, const double* __restrict__ trace,
                                 double* __restrict__ out) {
  __shared__ double red[32];
  double mn = INFINITY;
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    const int64_t d = static_cast<int64_t>(j) * c + j;
    mn = fmin(mn, R1[d] * R2[d] * R3[d]);
  }
  for (int o = 16; o > 0; o >>= 1) mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mn;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (unsigned w = 1; w < (blockDim.x >> 5); ++w) mn = fmin(mn, red[w]);
    out[0] = trace[0] > 0.0 ? mn / sqrt(trace[0]) : 0.0;
  }
}

// Speculative orth: the CholeskyQR2 gate (both factorizations succeeded and min pivot / trace(G) >= gate),
// else bit 0 of *flags. Jacobi: info 1 (no convergence) sets bit 1.
__global__ void orth_gate_kernel(const int* info, const double* info_d, double gate, int* flags) {
  if (info[0] != 0 || info[1] != 0 || !(info_d[0] >= gate)) atomicOr(flags, 1);
}
__global__ void jacobi_gate_kernel(const int* info, int* flags) {
  if (info[0] == 1) atomicOr(flags + 1, 1);
}

// part[blockIdx.x] = sum over this block's share of (A - S)^2 for a rows x cols block (column-major both).
__global__ void diff_sumsq_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ S, int64_t lds,
                                  int64_t rows, int64_t cols, double* __restrict__ part) {
  __shared__ double red[32];
  double acc = 0.0;
  const int64_t total = rows * cols, stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total; e += stride) {
    const int64_t j = e / rows, i = e - j * rows;
    const double d = A[j * lda + i] - S[j * lds + i];
    acc = fma(d, d, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    acc = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
  }
}

__global__ void f64_to_f32_kernel(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = static_cast<float>(x[i]);
}

}  // namespace

cudaError_t add_scalar(double* dst, const double* src, cudaStream_t st) {
  add_scalar_kernel<<<1, 1, 0, st>>>(dst, src);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t transpose(const double* in, int64_t rows, int64_t cols, int64_t ldi, double* out, int64_t ldo,
                             cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  dim3 grid(static_cast<unsigned>((rows + 31) / 32), static_cast<unsigned>((cols + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(in, rows, cols, ldi, out, ldo);
  count_launch();
  return cudaGetLastError();
}

}  // namespace rfgpu

using namespace rfgpu;

// ============================================================ errors =====
namespace {

thread_local std::string t_err;

struct Status {
  int code = RFGPU_OK;
  std::string msg;
  bool ok() const { return code == RFGPU_OK; }
};

Status make_err(int code, const std::string& msg) { return Status{code, msg}; }

int finish(const Status& s) {
  if (!s.ok()) t_err = s.msg;
  return s.code;
}

#define RF_CUDA(expr)                                                                              \
  do {                                                                                             \
    cudaError_t _e = (expr);                                                                       \
    if (_e != cudaSuccess)                                                                         \
      return make_err(RFGPU_ECUDA, std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #expr); \
  } while (0)

#define RF_TRY(expr)            \
  do {                          \
    Status _s = (expr);         \
    if (!_s.ok()) return _s;    \
  } while (0)

// ============================================================ NCCL (dlopen)
// NCCL is loaded lazily so the single-GPU path has no NCCL dependency and so
// an NCCL already loaded in the process (e.g. torch's) is reused.
// ncclUniqueId is a 128-byte struct passed BY VALUE to ncclCommInitRank (on the stack in the x86-64 ABI): the
// binding must declare it as a struct, not as a char array (which would decay to a pointer argument).
struct NcclUniqueId {
  char internal[128];
};
struct Nccl {
  void* h = nullptr;
  int (*getUniqueId)(NcclUniqueId*) = nullptr;
  int (*commInitRank)(void**, int, NcclUniqueId, int) = nullptr;
  int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*commDestroy)(void*) = nullptr;
  const char* (*getErrorString)(int) = nullptr;
  bool load(std::string* why) {
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      *why = "NCCL library not found (libnccl.so.2)";
      return false;
    }
    getUniqueId = reinterpret_cast<decltype(getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    commInitRank = reinterpret_cast<decltype(commInitRank)>(dlsym(h, "ncclCommInitRank"));
    allReduce = reinterpret_cast<decltype(allReduce)>(dlsym(h, "ncclAllReduce"));
    commDestroy = reinterpret_cast<decltype(commDestroy)>(dlsym(h, "ncclCommDestroy"));
    getErrorString = reinterpret_cast<decltype(getErrorString)>(dlsym(h, "ncclGetErrorString"));
    if (!getUniqueId || !commInitRank || !allReduce || !commDestroy || !getErrorString) {
      *why = "NCCL symbols missing";
      return false;
    }
    return true;
  }
};
Nccl g_nccl;
std::mutex g_nccl_mu;
constexpr int kNcclDouble = 8;  // ncclFloat64
constexpr int kNcclSum = 0;     // ncclSum

}  // namespace

// ============================================================ context ====
// Persistent host worker threads for the staging copies (pageable <-> pinned):
// run(n, fn) executes fn(0..n-1) across the workers and the calling thread.
class HostPool {
 public:
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 1 || workers() == 0) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      n_ = n;
      next_.store(0);
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == n_; });
    fn_ = nullptr;
  }
  int workers() {
    std::call_once(once_, [&] {
      const int nt = static_cast<int>(std::max(1u, std::thread::hardware_concurrency())) - 1;
      for (int i = 0; i < std::min(nt, 31); ++i) th_.emplace_back([this] { loop(); });
    });
    return static_cast<int>(th_.size());
  }

 private:
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n_) return;
      (*fn_)(i);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == n_) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        if (!fn_) continue;
      }
      work();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  std::vector<std::thread> th_;
  std::once_flag once_;
  const std::function<void(int)>* fn_ = nullptr;
  std::atomic<int> next_{0};
  int n_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

struct rfgpu_ctx {
  int device = 0, rank = 0, world = 1;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  void* comm = nullptr;
  std::mutex mu;
  // pinned scratch for status reads
  int* h_info = nullptr;
  double* h_d = nullptr;
  int64_t* h_i64 = nullptr;
  // profiling
  bool profile = false;
  struct Pending {
    std::string name;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  std::map<std::string, std::pair<int64_t, double>> prof;
  int64_t launch_base = 0;
  // host-input calls (rfgpu_rsvd_host): H2D copy stream and a reusable
  // device buffer for A, so repeated drop-in calls neither re-allocate nor
  // serialise the upload in front of the first pass
  cudaStream_t copy_stream = nullptr;
  // pinned staging ring for pageable host buffers (host copy threads fill a
  // slot, the copy engine moves it; a slot is refilled once its copy is done)
  HostPool host_pool;
  double* sp_stage_h[2] = {nullptr, nullptr};  // pinned stages of the streamed single pass, kept between calls
  size_t sp_stage_bytes = 0;
  std::vector<void*> stage_slots;
  std::vector<cudaEvent_t> stage_done;
  size_t stage_bytes = 0;
  size_t stage_next = 0;
  void* a_cache = nullptr;
  size_t a_cache_bytes = 0;
  // Stream-ordered memory pools owned by this context (ws_alloc): small
  // temporaries and large blocks (digit planes) apart, freed memory kept
  // cached between calls, everything returned on rfgpu_ctx_release_memory /
  // destroy. Other allocators in the process never see these blocks.
  cudaMemPool_t pool_small = nullptr, pool_large = nullptr;
  // Host-staged reduction backend (rfgpu_ctx_create_hostsum): the sums over
  // ranks go through the caller's host callback instead of NCCL.
  // Speculative CholeskyQR2 (rsvd / range finder): every orth assumes the
  // fast path and records a failed gate on the device (spec_flags); the call
  // reads the flags once at its end and re-runs without speculation when one
  // is set. No host round trip inside the call (so it can be graph-captured).
  bool spec = false;
  bool capturing = false;      // a call is being recorded into a CUDA graph (rfgpu_rsvd_device)
  struct GraphEntry {
    std::vector<int64_t> key;
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0, rank = 0;
  };
  std::vector<GraphEntry> graphs;               // one replayable graph per rsvd_device argument set
  std::map<std::vector<int64_t>, int> graph_seen;  // eager calls per argument set (capture on the second)
  std::map<std::vector<int64_t>, bool> spec_failed;  // argument sets whose speculation was rejected: run eagerly
  int* spec_flags = nullptr;   // device: [0] orth gate failures, [1] Jacobi non-convergence
  double* spec_vals = nullptr; // device: [0] ||A||_F^2, [1] ||B||_F^2
  void* h_spec = nullptr;      // pinned copy of both (64 bytes)
  rfgpu_host_sum_fn host_sum = nullptr;
  void* host_user = nullptr;
  double* h_stage = nullptr;
  size_t h_stage_n = 0;

  cudaEvent_t get_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};

struct rfgpu_matrix {
  rfgpu_ctx* ctx = nullptr;
  bool f32 = false;
  void* dev = nullptr;
  bool owned = false;
  int64_t m = 0, n = 0, lda = 0, m_global = 0, row0 = 0;
  // Host rows not yet on the device (rfgpu_rsvd_host): the first pass of the
  // range finder uploads them in row panels on ctx->copy_stream and consumes
  // each panel as soon as it lands. Cleared once the upload is issued.
  mutable const double* src = nullptr;
  mutable int64_t src_ld = 0;
};

namespace {

// Scoped CUDA-event timer on the context stream.
// Every phase is also an NVTX range (RFGPU_NVTX=1) for timeline tools (ncu's --nvtx filters, Nsight).
bool nvtx_on() {
  static const bool on = [] {
    const char* e = std::getenv("RFGPU_NVTX");
    return e && e[0] == '1';
  }();
  return on;
}

struct Timed {
  rfgpu_ctx* c;
  std::string name;
  cudaEvent_t a = nullptr;
  Timed(rfgpu_ctx* ctx, const char* nm) : c(ctx), name(nm) {
    if (nvtx_on()) nvtxRangePushA(nm);
    if (c->profile) {
      a = c->get_event();
      cudaEventRecord(a, c->stream);
    }
  }
  ~Timed() {
    if (c->profile && a) {
      cudaEvent_t b = c->get_event();
      cudaEventRecord(b, c->stream);
      c->pending.push_back({name, a, b});
    }
    if (nvtx_on()) nvtxRangePop();
  }
};

void drain_profile(rfgpu_ctx* c) {
  if (c->pending.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& p : c->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    auto& s = c->prof[p.name];
    s.first += 1;
    s.second += ms;
    c->event_pool.push_back(p.a);
    c->event_pool.push_back(p.b);
  }
  c->pending.clear();
}

// The pools of the context whose C-ABI call is running on this thread.
thread_local rfgpu_ctx* t_ctx = nullptr;
constexpr size_t kSmallBlock = size_t{256} << 20;

// Locks the context for one C-ABI call and installs its pools for ws_alloc.
struct CtxCall {
  std::lock_guard<std::mutex> lk;
  rfgpu_ctx* prev;
  explicit CtxCall(rfgpu_ctx* c) : lk(c->mu), prev(t_ctx) {
    t_ctx = c;
    cudaGetLastError();  // a runtime error left on this thread by other code must not be reported as ours
  }
  ~CtxCall() { t_ctx = prev; }
};

}  // namespace

cudaError_t rfgpu::ws_alloc(void** p, size_t bytes, cudaStream_t st) {
  rfgpu_ctx* c = t_ctx;
  if (c && c->capturing) return cudaMallocAsync(p, bytes, st);  // a graph memory node (owned by the graph)
  if (c && c->pool_small) return cudaMallocFromPoolAsync(p, bytes, bytes < kSmallBlock ? c->pool_small : c->pool_large, st);
  return cudaMallocAsync(p, bytes, st);
}

namespace {

// Stream-ordered device buffer from the context's memory pools.
struct DBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  Status alloc(size_t bytes, cudaStream_t st) {
    s = st;
    if (bytes == 0) bytes = 16;
    cudaError_t e = rfgpu::ws_alloc(&p, bytes, st);
    if (e != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      return make_err(RFGPU_ENOMEM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    }
    return {};
  }
  double* d() const { return static_cast<double*>(p); }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

inline int64_t even(int64_t x) { return x + (x & 1); }

// Host-staged sum over ranks (rfgpu_ctx_create_hostsum): the stream is
// drained, the buffer goes through pinned host memory to the caller's
// callback and back; stream order covers the copy back.
cudaError_t host_allreduce(rfgpu_ctx* c, double* buf, int64_t count, cudaStream_t st) {
  if (c->h_stage_n < static_cast<size_t>(count)) {
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return e;
    if (c->h_stage) cudaFreeHost(c->h_stage);
    c->h_stage = nullptr;
    c->h_stage_n = 0;
    e = cudaMallocHost(&c->h_stage, sizeof(double) * count);
    if (e != cudaSuccess) return e;
    c->h_stage_n = static_cast<size_t>(count);
  }
  cudaError_t e = cudaMemcpyAsync(c->h_stage, buf, sizeof(double) * count, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return e;
  const int rc = c->host_sum(c->host_user, c->h_stage, count);
  cudaGetLastError();  // the callback is foreign code: a runtime error it left behind is not ours
  if (rc != 0) return cudaErrorUnknown;
  return cudaMemcpyAsync(buf, c->h_stage, sizeof(double) * count, cudaMemcpyHostToDevice, st);
}

cudaError_t nccl_allreduce_cb(void* vctx, double* buf, int64_t count, cudaStream_t st) {
  rfgpu_ctx* c = static_cast<rfgpu_ctx*>(vctx);
  if (c->world <= 1 || count <= 0) return cudaSuccess;
  if (c->host_sum) return host_allreduce(c, buf, count, st);
  int r = g_nccl.allReduce(buf, buf, static_cast<size_t>(count), kNcclDouble, kNcclSum, c->comm, st);
  return r == 0 ? cudaSuccess : cudaErrorUnknown;
}

DeviceAllreduce allreduce_of(rfgpu_ctx* c) {
  DeviceAllreduce a{};
  if (c->world > 1) {
    a.ctx = c;
    a.fn = nccl_allreduce_cb;
  }
  return a;
}

Status allreduce(rfgpu_ctx* c, double* buf, int64_t count) {
  if (c->world <= 1 || count <= 0) return {};
  Timed t(c, "allreduce");
  if (c->host_sum) {
    cudaError_t e = host_allreduce(c, buf, count, c->stream);
    if (e != cudaSuccess) return make_err(RFGPU_ECUDA, std::string("host-staged allreduce failed: ") + cudaGetErrorString(e));
    return {};
  }
  int r = g_nccl.allReduce(buf, buf, static_cast<size_t>(count), kNcclDouble, kNcclSum, c->comm, c->stream);
  if (r != 0) return make_err(RFGPU_ECUDA, std::string("NCCL allreduce: ") + g_nccl.getErrorString(r));
  return {};
}

// ---- GEMM wrapper -----------------------------------------------------------
Status gemm(rfgpu_ctx* c, bool trans, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
            const double* B, int64_t ldb, double* C, int64_t ldc, double* sumsq_partials = nullptr,
            const char* label = nullptr, bool sym = false, bool tri_b = false) {
  if (M <= 0 || N <= 0) return {};
  const GemmPlan p = plan_gemm(M, N, K, c->num_sms, 0, sym);
  DBuf ws;
  const size_t wb = gemm_workspace_bytes(M, N, p);
  if (wb) RF_TRY(ws.alloc(wb, c->stream));
  {
    Timed t(c, label ? label : (trans ? "gemm_tn" : "gemm_nn"));
    RF_CUDA(gemm_f64(trans, M, N, K, A, lda, B, ldb, C, ldc, ws.d(), wb, sumsq_partials, p, c->stream, tri_b));
  }
  return {};
}

int64_t sumsq_slots(rfgpu_ctx* c, int64_t M, int64_t N, int64_t K) {
  const GemmPlan p = plan_gemm(M, N, K, c->num_sms);
  return static_cast<int64_t>(p.splits) * p.mtiles;
}

// Row panels for streaming a host A in behind the first pass: large enough to
// keep every SM busy on a panel's product (>= 32768 rows), few enough that
// the per-panel launch and event costs vanish; the last panel's product is
// the only compute not hidden under the copy.
std::vector<std::pair<int64_t, int64_t>> upload_panels(int64_t m) {
  int64_t np = m >= (int64_t{1} << 19) ? 16 : (m >= (int64_t{1} << 16) ? 4 : 1);
  // panel boundaries on the digit path's column-exponent chunks, so that each
  // panel's column-scaled digits can be written as soon as it lands
  const int64_t q = ozaki_chunk_rows();
  const int64_t step = ((m + np - 1) / np + q - 1) / q * q;
  std::vector<std::pair<int64_t, int64_t>> out;
  for (int64_t r = 0; r < m; r += step) out.emplace_back(r, std::min(m, r + step));
  if (out.empty()) out.emplace_back(0, 0);
  return out;
}

// Drops every recorded graph of the context (their memory goes back to the driver) and the eager pools'
// cached blocks; true if anything was released. Used when a large allocation fails.
bool release_graph_memory(rfgpu_ctx* c) {
  if (c->graphs.empty()) return false;
  cudaStreamSynchronize(c->stream);
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
  c->graph_seen.clear();
  cudaDeviceGraphMemTrim(c->device);
  for (cudaMemPool_t pool : {c->pool_small, c->pool_large}) cudaMemPoolTrimTo(pool, 0);
  cudaGetLastError();
  return true;
}

// FP64 passes on the INT8 tensor cores (ozaki.cu) for one call: the digit
// planes of A are built once (inside pass 1) and serve every later pass.
struct OzPasses {
  bool on = false;
  bool tn = true;  // A^T Q on the digits (false: the column-scaled set did not fit; DMMA)
  // the thin matrix whose column-scaled digits are in `work` (orth's digit Gram
  // of Q1), reused by the A^T Q1 pass that follows
  const double* thin_src = nullptr;
  int64_t thin_cols = 0;
  OzakiA a{};
  DBuf planes, cplanes, work;
  Status init(rfgpu_ctx* c, const rfgpu_matrix* m, int64_t ell) {
    on = ozaki_enabled(m->m, m->n) && m->m > 0 && m->n > 0;
    if (!on) return {};
    const int digits = m->f32 ? 4 : 7;  // FP32 data: 4 digits (30 bits) per element
    const OzakiA lay = ozaki_layout(m->m, m->n, digits);
    // One digit set takes `digits` bytes per element of A: when HBM cannot
    // hold it next to A, the passes stay on the FP64 tensor pipe (DMMA).
    // Both digit sets in one allocation when they fit (the same size every
    // call, so the stream-ordered pool reuses it); else the row-scaled set
    // alone and columns() decides how A^T Q runs.
    const size_t base = (ozaki_a_bytes(m->m, m->n, digits) + 4095) / 4096 * 4096;
    const size_t set = ozaki_set_bytes(m->m, m->n, digits);
    const size_t wbytes = std::max(ozaki_nn_work_bytes(lay, m->m, ell), ozaki_tn_work_bytes(lay, ell));
    bool both = planes.alloc(base + set, c->stream).ok();
    if (!both && !c->capturing && release_graph_memory(c))  // recorded graphs hold their own copies: free them
      both = planes.alloc(base + set, c->stream).ok();
    if ((!both && !planes.alloc(base, c->stream).ok()) || !work.alloc(wbytes, c->stream).ok()) {
      on = false;
      if (std::getenv("RFGPU_DEBUG")) std::fprintf(stderr, "[rfgpu] digit planes do not fit: DMMA passes\n");
      return {};
    }
    ozaki_bind(planes.p, m->m, m->n, digits, &a);
    if (both) a.cs = static_cast<int8_t*>(planes.p) + base;
    a.cs_rowmajor = ozaki_cs_rowmajor();
    return {};
  }
  // After every row's stats: column exponents and a second, column-scaled
  // (row-major) digit set for A^T Q; if it does not fit, the row-scaled set
  // serves A^T Q when the column scales allow it (ozaki.cu kSharedSpread),
  // else A^T Q stays on DMMA.
  Status columns(rfgpu_ctx* c, const rfgpu_matrix* m) {
    const char* fs = std::getenv("RFGPU_OZAKI_SHARED");
    const bool decide = !a.cs || (fs && fs[0] == '1');  // host decision only for the memory fallback / forced mode
    RF_CUDA(ozaki_col_exponents(&a, c->stream, c->h_info, decide));
    if (!a.shared && !a.cs) {
      if (cplanes.alloc(ozaki_set_bytes(m->m, m->n, a.digits), c->stream).ok()) {
        a.cs = cplanes.as<int8_t>();
      } else if (a.shared_ok) {  // no room for the second set: the row-scaled set serves A^T Q
        a.shared = true;
      } else {
        tn = false;
        if (std::getenv("RFGPU_DEBUG")) std::fprintf(stderr, "[rfgpu] column-scaled digits do not fit: DMMA A^T Q\n");
      }
    }
    if (std::getenv("RFGPU_DEBUG") && decide)
      std::fprintf(stderr, "[rfgpu] digit sets: %s (column exponents %d..%d)\n", a.shared ? "shared" : "two",
                   -c->h_info[1], c->h_info[0]);
    return {};
  }
  // Whole resident A: stats (one read), then the digit set(s) (one read):
  // row-scaled when `rows` (A X) or shared, column-scaled when not shared.
  Status prepare(rfgpu_ctx* c, const rfgpu_matrix* m, double* ssq, bool rows = true) {
    Timed t(c, "ozaki_slice");
    {
      Timed ts(c, "stats");
      RF_CUDA(ozaki_prepare_rows(m->dev, m->f32, m->lda, 0, m->m, a, ssq, false, c->stream));
    }
    RF_TRY(columns(c, m));
    Timed tsl(c, "slicer");
    RF_CUDA(ozaki_slice_sets(m->dev, m->f32, m->lda, a, rows || a.shared, tn && !a.shared, c->stream));
    return {};
  }
};

int64_t pass1_slots(rfgpu_ctx* c, const rfgpu_matrix* a, int64_t ell, const OzPasses& oz) {
  auto slots = [&](int64_t rows) { return oz.on ? ozaki_ssq_slots(rows, a->n) : sumsq_slots(c, rows, ell, a->n); };
  if (!a->src) return slots(a->m);
  int64_t s = 0;
  for (auto& pr : upload_panels(a->m)) s += slots(pr.second - pr.first);
  return s;
}

// One pass-1 block: rows [r0, r1) of Y = A G (+ ||A||_F^2 partials at ssq).
// whole: the block is all of a resident A (both digit sets built here);
// otherwise an upload panel (row digits only; column digits after the last).
Status pass1_rows(rfgpu_ctx* c, const rfgpu_matrix* a, const double* G, int64_t ell, double* Y, int64_t ldy,
                  double* ssq, int64_t r0, int64_t r1, OzPasses& oz, bool whole) {
  const double* A = static_cast<const double*>(a->dev);
  if (oz.on) {
    if (whole) {
      RF_TRY(oz.prepare(c, a, ssq));
    } else {
      Timed t(c, "ozaki_slice");
      RF_CUDA(ozaki_prepare_rows(A, false, a->lda, r0, r1, oz.a, ssq, true, c->stream));
      if (oz.tn && oz.a.cs && !oz.a.shared)  // this panel's column-scaled digits (per-chunk exponents)
        RF_CUDA(ozaki_slice_cols_rows(A, false, a->lda, oz.a, r0, r1, c->stream));
    }
    Timed t(c, "pass_nn");
    RF_CUDA(ozaki_nn(oz.a, r0, r1, G, a->n, ell, Y, ldy, oz.work.p, c->stream));
    return {};
  }
  return gemm(c, false, r1 - r0, ell, a->n, A + r0, a->lda, G, a->n, Y + r0, ldy, ssq, "pass_nn");
}

// Y = A X for the later passes (X n x cols).
Status pass_nn(rfgpu_ctx* c, const rfgpu_matrix* a, const double* X, int64_t cols, double* Y, int64_t ldy,
               OzPasses* oz) {
  if (oz && oz->on) {
    Timed t(c, "pass_nn");
    oz->thin_src = nullptr;  // the thin digits of X overwrite the work buffer
    RF_CUDA(ozaki_nn(oz->a, 0, a->m, X, a->n, cols, Y, ldy, oz->work.p, c->stream));
    return {};
  }
  return gemm(c, false, a->m, cols, a->n, static_cast<const double*>(a->dev), a->lda, X, a->n, Y, ldy, nullptr,
              "pass_nn");
}

// Z = A^T Y (Y m x cols), not summed over ranks.
Status pass_tn_raw(rfgpu_ctx* c, const rfgpu_matrix* a, const double* Y, int64_t ldy, int64_t cols, double* Z,
                   OzPasses* oz) {
  if (oz && oz->on && oz->tn) {
    Timed t(c, "pass_tn");
    const bool pre = oz->thin_src == Y && oz->thin_cols == cols && !oz->a.shared;
    RF_CUDA(ozaki_tn(oz->a, Y, ldy, cols, Z, a->n, oz->work.p, c->stream, pre));
    oz->thin_src = nullptr;  // only orth's Gram hands digits to the pass right after it
    return {};
  }
  return gemm(c, true, a->n, cols, a->m, static_cast<const double*>(a->dev), a->lda, Y, ldy, Z, a->n, nullptr,
              "pass_tn");
}

// ---- pageable host buffers: pinned staging ring ----------------------------------------
// A DMA from pageable memory is staged by the driver synchronously and slowly;
// instead, host threads copy column blocks of the caller's buffer into pinned
// slots (kStageSlots x kStageBytes, allocated once per context) and the copy
// engine moves each slot while the next is being filled.
constexpr int kStageSlots = 4;
constexpr size_t kStageBytes = size_t{128} << 20;

bool host_is_pageable(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return at.type == cudaMemoryTypeUnregistered;
}

// Copies into the pinned slots use non-temporal stores (csrc/host_copy.cpp). Measured on the GPU box's host
// (tools/microbench/hostcopy_nt.cu, 16 threads, 512 KB column chunks): glibc memcpy 48.6 GB/s alone and 36.9
// GB/s while the copy engine reads the previous slot, non-temporal 68.8 / 45.8 GB/s; config 3 from pageable
// memory 0.902 -> 0.887 s. (64-byte AVX-512 stores: 48.8 GB/s in the microbenchmark, but the call itself
// 0.881 / 0.946 s against 0.886 / 0.890 s with AVX2 on one box: not kept.) The staging copy and the DMA slow
// each other down (the DMA alone reaches 55 GB/s, 48-49 GB/s beside the copy): that contention, not PCIe,
// bounds the pageable call.
constexpr bool nt_staging() { return true; }

Status stage_ring(rfgpu_ctx* c) {
  if (!c->stage_slots.empty()) return {};
  // 4 x 128 MiB measured best at config 3 (8 x 128: 0.90 s, 4 x 256: 0.90 s, 8 x 64: 1.39 s, 3 x 512: 0.99 s
  // against 0.89 s): the copy threads and the DMA share the host's memory bandwidth
  const int slots = kStageSlots;
  const size_t bytes = kStageBytes;
  for (int i = 0; i < slots; ++i) {
    void* p = nullptr;
    cudaEvent_t e;
    RF_CUDA(cudaMallocHost(&p, bytes));
    c->stage_slots.push_back(p);
    RF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->stage_done.push_back(e);
  }
  c->stage_bytes = bytes;
  return {};
}

// Parallel strided copy of `cols` columns of `rows` doubles (ld_src -> ld_dst) on the host (the context's
// worker threads; 16 MiB or so per task).
void host_copy_cols(rfgpu_ctx* c, double* dst, int64_t ldd, const double* src, int64_t lds, int64_t rows,
                    int64_t cols, bool stream_dst = false) {
  const int64_t bytes = rows * cols * 8;
  const int nt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(64, bytes >> 23)));  // 8 MiB tasks
  // into a pinned slot (read next by the copy engine only): non-temporal stores (csrc/host_copy.cpp)
  auto cp = [stream_dst](void* d, const void* s, size_t n) {
    if (stream_dst) rfgpu::host_stream_copy(d, s, n);
    else std::memcpy(d, s, n);
  };
  auto part = [&](int t) {
    if (cols >= nt) {
      for (int64_t j = cols * t / nt; j < cols * (t + 1) / nt; ++j)
        cp(dst + j * ldd, src + j * lds, sizeof(double) * rows);
    } else {  // few columns: split the rows
      const int64_t r0 = rows * t / nt, r1 = rows * (t + 1) / nt;
      for (int64_t j = 0; j < cols; ++j) cp(dst + j * ldd + r0, src + j * lds + r0, sizeof(double) * (r1 - r0));
    }
  };
  c->host_pool.run(nt, part);
}

// H2D of rows x cols (column-major, ld lds) from pageable host memory into the
// device (ld ldd) on stream cs through the staging ring. Returns once every
// block is issued (host copies done, DMAs queued).
Status staged_h2d(rfgpu_ctx* c, double* dev, int64_t ldd, const double* host, int64_t lds, int64_t rows, int64_t cols,
                  cudaStream_t cs) {
  if (rows <= 0 || cols <= 0) return {};
  RF_TRY(stage_ring(c));
  const int64_t rstep = static_cast<size_t>(rows) * 8 <= c->stage_bytes ? rows : static_cast<int64_t>(c->stage_bytes / 8);
  for (int64_t r0 = 0; r0 < rows; r0 += rstep) {
    const int64_t rr = std::min(rstep, rows - r0);
    const int64_t cstep = std::max<int64_t>(1, static_cast<int64_t>(c->stage_bytes / (sizeof(double) * rr)));
    for (int64_t c0 = 0; c0 < cols; c0 += cstep) {
      const int64_t cc = std::min(cstep, cols - c0);
      const size_t sl = c->stage_next++ % c->stage_slots.size();
      RF_CUDA(cudaEventSynchronize(c->stage_done[sl]));  // the slot's previous copy has landed
      double* buf = static_cast<double*>(c->stage_slots[sl]);
      host_copy_cols(c, buf, rr, host + c0 * lds + r0, lds, rr, cc, /*stream_dst=*/nt_staging());
      RF_CUDA(cudaMemcpy2DAsync(dev + c0 * ldd + r0, sizeof(double) * ldd, buf, sizeof(double) * rr, sizeof(double) * rr,
                                cc, cudaMemcpyHostToDevice, cs));
      RF_CUDA(cudaEventRecord(c->stage_done[sl], cs));
    }
  }
  return {};
}

// D2H into pageable host memory through the ring (blocks until the data is in `host`).
Status staged_d2h(rfgpu_ctx* c, double* host, int64_t ldh, const double* dev, int64_t ldd, int64_t rows, int64_t cols,
                  cudaStream_t cs) {
  if (rows <= 0 || cols <= 0) return {};
  RF_TRY(stage_ring(c));
  const int64_t rstep = static_cast<size_t>(rows) * 8 <= c->stage_bytes ? rows : static_cast<int64_t>(c->stage_bytes / 8);
  struct Pending {
    size_t slot;
    int64_t r0, rr, c0, cc;
  };
  std::vector<Pending> q;
  auto drain = [&](size_t keep) -> Status {
    while (q.size() > keep) {
      const Pending pd = q.front();
      q.erase(q.begin());
      RF_CUDA(cudaEventSynchronize(c->stage_done[pd.slot]));
      host_copy_cols(c, host + pd.c0 * ldh + pd.r0, ldh, static_cast<double*>(c->stage_slots[pd.slot]), pd.rr, pd.rr, pd.cc);
    }
    return {};
  };
  for (int64_t r0 = 0; r0 < rows; r0 += rstep) {
    const int64_t rr = std::min(rstep, rows - r0);
    const int64_t cstep = std::max<int64_t>(1, static_cast<int64_t>(c->stage_bytes / (sizeof(double) * rr)));
    for (int64_t c0 = 0; c0 < cols; c0 += cstep) {
      const int64_t cc = std::min(cstep, cols - c0);
      RF_TRY(drain(c->stage_slots.size() - 1));  // the next slot in turn is free
      const size_t sl = c->stage_next++ % c->stage_slots.size();
      RF_CUDA(cudaEventSynchronize(c->stage_done[sl]));
      RF_CUDA(cudaMemcpy2DAsync(c->stage_slots[sl], sizeof(double) * rr, dev + c0 * ldd + r0, sizeof(double) * ldd,
                                sizeof(double) * rr, cc, cudaMemcpyDeviceToHost, cs));
      RF_CUDA(cudaEventRecord(c->stage_done[sl], cs));
      q.push_back({sl, r0, rr, c0, cc});
    }
  }
  return drain(0);
}

// Y = A G with ||A||_F^2 partials fused (pass 1). For a handle whose rows are
// still on the host, panel i+1's H2D copy runs on the copy stream while panel
// i's product runs on the compute stream.
Status pass1(rfgpu_ctx* c, const rfgpu_matrix* a, const double* G, int64_t ell, double* Y, int64_t ldy,
             double* ssq, OzPasses& oz) {
  const int64_t m = a->m, n = a->n, lda = a->lda;
  const double* A = static_cast<const double*>(a->dev);
  if (!a->src) return pass1_rows(c, a, G, ell, Y, ldy, ssq, 0, m, oz, true);
  cudaStream_t st = c->stream, cs = c->copy_stream;
  const auto panels = upload_panels(m);
  const bool pageable = host_is_pageable(a->src);
  std::vector<cudaEvent_t> ev(panels.size());
  for (auto& e : ev) RF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  auto copy = [&](size_t i) -> Status {
    const int64_t r0 = panels[i].first, rows = panels[i].second - r0;
    if (rows > 0 && n > 0) {
      if (pageable)  // host threads through the pinned ring; returns once issued
        RF_TRY(staged_h2d(c, const_cast<double*>(A) + r0, lda, a->src + r0, a->src_ld, rows, n, cs));
      else
        RF_CUDA(cudaMemcpy2DAsync(const_cast<double*>(A) + r0, sizeof(double) * lda, a->src + r0,
                                  sizeof(double) * a->src_ld, sizeof(double) * rows, n, cudaMemcpyHostToDevice, cs));
    }
    RF_CUDA(cudaEventRecord(ev[i], cs));
    return {};
  };
  // the device buffer may still be read by the previous call's tail
  cudaEvent_t ready;
  RF_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  RF_CUDA(cudaEventRecord(ready, st));
  RF_CUDA(cudaStreamWaitEvent(cs, ready, 0));
  // panel i's product is queued before panel i+1 is copied: with a pageable
  // source the host is busy staging panel i+1 while the GPU works on panel i
  Status s = copy(0);
  int64_t off = 0;
  for (size_t i = 0; i < panels.size() && s.ok(); ++i) {
    const int64_t r0 = panels[i].first, rows = panels[i].second - r0;
    if (cudaStreamWaitEvent(st, ev[i], 0) != cudaSuccess) {
      s = make_err(RFGPU_ECUDA, "pass 1: stream wait failed");
      break;
    }
    s = pass1_rows(c, a, G, ell, Y, ldy, ssq + off, r0, r0 + rows, oz, false);
    off += oz.on ? ozaki_ssq_slots(rows, a->n) : sumsq_slots(c, rows, ell, n);
    if (s.ok() && i + 1 < panels.size()) s = copy(i + 1);
  }
  if (s.ok() && oz.on) {  // all rows landed: the A^T Q digits unless sliced per panel already
    Timed t(c, "ozaki_slice");
    const bool sliced = oz.tn && oz.a.cs && !oz.a.shared;
    s = oz.columns(c, a);
    if (s.ok() && !sliced &&
        ozaki_slice_sets(A, false, lda, oz.a, false, oz.tn && !oz.a.shared, st) != cudaSuccess)
      s = make_err(RFGPU_ECUDA, "pass 1: slicing failed");
  }
  a->src = nullptr;  // issued: every later consumer is ordered after the waits above
  cudaEventDestroy(ready);
  for (auto& e : ev) cudaEventDestroy(e);  // destruction is deferred until the events complete
  return s;
}

// ---- orth ---------------------------------------------------------------------
// Orthonormal basis of X (m_loc x cols, ld ldx; rows sharded over ranks when
// dist) replacing the reference MGS (dense.cpp:402-431).
//
// CholeskyQR2 fast path, accepted when every Cholesky pivot of the Gram is
// >= 1e-10 trace(G) (each column keeps a residual >= 1e-5 ||X||_F, far above
// the reference's 1e-13 drop threshold, so the reference keeps all columns
// and CholeskyQR2 is orthonormal to working precision):
//   G1 = X^T X, R1 = chol(G1), Q1 = X R1^{-1}, G2 = Q1^T Q1, R2 = chol(G2).
// The basis is Q = Q1 R2^{-1}. With fold = true, Q1 and R2^{-1} are returned
// separately (Q is never formed; consumers apply R2^{-1} on the l-sized
// side), saving one m x l x l product per orth. Otherwise Q is formed.
// R (optional) = R2 R1, so that X = Q R.
//
// Fallback (rank-deficient / ill-conditioned X): Gram-Schmidt with the
// reference's drop rule; the basis is returned directly (folded = false).
struct Basis {
  double* Q = nullptr;      // m_loc x r (Q1 when folded)
  int64_t ldq = 0;
  int64_t r = 0;
  double* R2inv = nullptr;  // r x r (folded only)
  bool folded = false;
  bool fast = false;
};

constexpr double kCholGate = 1e-10;  // min pivot / trace(G)

// RFGPU_DIGIT_GRAM=0 keeps the tall orth Grams on DMMA.
bool digit_grams() {
  const char* e = std::getenv("RFGPU_DIGIT_GRAM");
  return !(e && e[0] == '0');
}

// single = true: CholeskyQR (one Gram) only — a basis of range(X) that is orthonormal only to ~eps kappa(X)^2,
// for an intermediate power-iteration basis whose one consumer is a product followed by another orth: for
// Q1 = Q S (S upper triangular, near identity) the next orthonormalised basis is the same matrix (the QR factor
// with positive R diagonal is unique), so the second Gram, Cholesky and fold are skipped.
Status orth(rfgpu_ctx* c, const double* X, int64_t m, int64_t cols, int64_t ldx, Basis* out, double* R2inv_buf,
            double* R, bool dist, bool fold, OzPasses* oz = nullptr, bool single = false) {
  Timed t(c, "orth");
  out->r = 0;
  out->folded = false;
  out->fast = false;
  out->R2inv = nullptr;
  if (cols == 0) return {};
  cudaStream_t st = c->stream;
  const int64_t cc = cols * cols;
  DBuf small;
  RF_TRY(small.alloc(sizeof(double) * (6 * cc + 16) + chol_inv_work_bytes(cols) + 64, st));
  double* G1 = small.d();
  double* R1 = G1 + cc;
  double* R1i = R1 + cc;
  double* G2 = R1i + cc;
  double* R2 = G2 + cc;
  double* R2i = R2 + cc;
  double* infod = R2i + cc;  // 2 doubles (+pad)
  double* cwork = infod + 8;  // chol_inv_work_bytes(cols)
  int* info = reinterpret_cast<int*>(infod + 4);
  DBuf q1buf;
  double* Q1 = out->Q;  // folded or single: Q1 lands directly in the output buffer
  int64_t ldq1 = out->ldq;
  if (!fold && !single) {
    ldq1 = even(m);
    RF_TRY(q1buf.alloc(sizeof(double) * std::max<int64_t>(1, ldq1 * cols), st));
    Q1 = q1buf.d();
  }

  // Tall orth over A's rows with the passes on the digit path: both Grams on
  // the INT8 tensor cores too (column-scaled digits of X, then of Q1; Q1's
  // digits stay in the work buffer for the A^T Q1 pass that follows).
  const bool dig = oz && oz->on && oz->tn && !oz->a.shared && m == oz->a.m && fold && digit_grams();
  auto gram = [&](const double* M, int64_t ldm, double* G) -> Status {
    if (!dig) return gemm(c, true, cols, cols, m, M, ldm, M, ldm, G, cols, nullptr, "gram", /*sym=*/true);
    Timed tg(c, "gram");
    RF_CUDA(ozaki_slice_thin(oz->a, M, ldm, cols, oz->work.p, st));
    RF_CUDA(ozaki_gram_thin(oz->a, cols, oz->work.p, G, cols, st));
    oz->thin_src = M;
    oz->thin_cols = cols;
    return {};
  };
  RF_TRY(gram(X, ldx, G1));
  if (dist) RF_TRY(allreduce(c, G1, cc));
  {
    Timed tc(c, "chol");
    RF_CUDA(chol_inv(G1, cols, R1, R1i, cwork, info, infod, st));
  }
  // Outside speculation the first factorization is checked at once: a sketch that fails it (the plain power
  // mode's, a rank-deficient one) goes straight to the fallbacks without the m x l product and second Gram.
  bool first_ok = true;
  if (!c->spec) {
    RF_CUDA(cudaMemcpyAsync(c->h_info, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaMemcpyAsync(c->h_d, infod, sizeof(double), cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaStreamSynchronize(st));
    first_ok = c->h_info[0] == 0 && c->h_d[0] >= kCholGate;
  }
  // (an INT8 digit-path TRSM from X's digits measured 4.1 ms against 2.9 ms on DMMA at config 3: K = l is too
  // short for the digit GEMM's per-tile fetch and epilogue)
  if (first_ok)
    RF_TRY(gemm(c, false, m, cols, cols, X, ldx, R1i, cols, Q1, ldq1, nullptr, "trsm", false, /*tri_b=*/true));
  if (!first_ok) {
  } else if (single) {
    RF_CUDA(cudaMemsetAsync(info + 1, 0, sizeof(int), st));
  } else {
    RF_TRY(gram(Q1, ldq1, G2));
    if (dist) RF_TRY(allreduce(c, G2, cc));
    Timed tc(c, "chol");
    RF_CUDA(chol_inv(G2, cols, R2, R2i, cwork, info + 1, infod + 1, st));
  }
  bool fast;
  if (!first_ok) {
    fast = false;
  } else if (c->spec) {  // decided at the end of the call (spec_flags)
    rfgpu::orth_gate_kernel<<<1, 1, 0, st>>>(info, infod, kCholGate, c->spec_flags);
    count_launch();
    RF_CUDA(cudaGetLastError());
    fast = true;
  } else {
    RF_CUDA(cudaMemcpyAsync(c->h_info, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaMemcpyAsync(c->h_d, infod, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaStreamSynchronize(st));
    fast = c->h_info[0] == 0 && c->h_info[1] == 0 && c->h_d[0] >= kCholGate;
  }
  if (fast && single) {  // the CholeskyQR basis itself (already in out->Q)
    out->fast = true;
    out->r = cols;
    if (R) RF_CUDA(cudaMemcpyAsync(R, R1, sizeof(double) * cc, cudaMemcpyDeviceToDevice, st));
    return {};
  }
  if (fast) {
    out->fast = true;
    out->r = cols;
    if (R) RF_TRY(gemm(c, false, cols, cols, cols, R2, cols, R1, cols, R, cols));
    if (fold) {
      RF_CUDA(cudaMemcpyAsync(R2inv_buf, R2i, sizeof(double) * cc, cudaMemcpyDeviceToDevice, st));
      out->R2inv = R2inv_buf;
      out->folded = true;
    } else {
      RF_TRY(gemm(c, false, m, cols, cols, Q1, ldq1, R2i, cols, out->Q, out->ldq, nullptr, "trsm", false, true));
    }
    return {};
  }
  // Ill-conditioned but full-rank X (the plain power mode's sketch (A A^T)^q A G, kappa ~ (s1/sl)^(2q+1)):
  // shifted CholeskyQR3 (Fukaya et al. 2020). Q1 = X R1^-1 with R1^T R1 = X^T X + shift tr(X^T X) I has
  // kappa(Q1) ~ sqrt(shift) kappa(X), then CholeskyQR2 on Q1. X = Q (R3 R2 R1) is then THE QR factorization
  // of X, whose diagonal is the residual norm the reference's Gram-Schmidt tests against 1e-13 ||X||_F
  // (dense.cpp:404,423): accepted only if every residual clears ten times that, so the reference keeps every
  // column too; anything closer goes to Gram-Schmidt with the reference's rule itself. Not speculative (host
  // round trips), not for intermediate bases (single) and only when the fast path has just failed.
  if (!c->spec && !single && cols > 1) {
    Timed ts(c, "scholqr3");
    constexpr double kShift = 1e-11, kMidGate = 1e-14, kDropMargin = 1e-12;
    DBuf sb, q2buf;
    RF_TRY(sb.alloc(sizeof(double) * (3 * cc + 16), st));
    double* R3 = sb.d();
    double* R3i = R3 + cc;
    double* G3 = R3i + cc;
    double* stat = G3 + cc;  // trace, min residual ratio
    // G1 still holds X^T X (summed over ranks): the Cholesky kernels do not write their input
    rfgpu::shift_diag_kernel<<<1, 256, 0, st>>>(G1, static_cast<int>(cols), kShift, stat);
    count_launch();
    RF_CUDA(chol_inv(G1, cols, R1, R1i, cwork, info, infod, st));
    // Q1 into a temporary, Q2 into the output buffer
    const int64_t ldt = even(m);
    RF_TRY(q2buf.alloc(sizeof(double) * std::max<int64_t>(1, ldt * cols), st));
    double* T1 = q2buf.d();
    RF_TRY(gemm(c, false, m, cols, cols, X, ldx, R1i, cols, T1, ldt, nullptr, "trsm", false, true));
    RF_TRY(gram(T1, ldt, G2));
    if (dist) RF_TRY(allreduce(c, G2, cc));
    RF_CUDA(chol_inv(G2, cols, R2, R2i, cwork, info + 1, infod + 1, st));
    RF_CUDA(cudaMemcpyAsync(c->h_info, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaMemcpyAsync(c->h_d, infod, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaStreamSynchronize(st));
    bool ok = c->h_info[0] == 0 && c->h_info[1] == 0 && c->h_d[1] >= kMidGate;
    double* Q2 = fold ? out->Q : Q1;
    const int64_t ldq2 = fold ? out->ldq : ldq1;
    if (ok) {
      RF_TRY(gemm(c, false, m, cols, cols, T1, ldt, R2i, cols, Q2, ldq2, nullptr, "trsm", false, true));
      RF_TRY(gram(Q2, ldq2, G3));
      if (dist) RF_TRY(allreduce(c, G3, cc));
      RF_CUDA(chol_inv(G3, cols, R3, R3i, cwork, info, infod, st));
      rfgpu::rdiag_min_kernel<<<1, 256, 0, st>>>(R1, R2, R3, static_cast<int>(cols), stat, stat + 1);
      count_launch();
      RF_CUDA(cudaMemcpyAsync(c->h_info, info, sizeof(int), cudaMemcpyDeviceToHost, st));
      RF_CUDA(cudaMemcpyAsync(c->h_d, infod, sizeof(double), cudaMemcpyDeviceToHost, st));
      RF_CUDA(cudaMemcpyAsync(c->h_d + 1, stat + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
      RF_CUDA(cudaStreamSynchronize(st));
      ok = c->h_info[0] == 0 && c->h_d[0] >= kCholGate && c->h_d[1] >= kDropMargin;
      if (std::getenv("RFGPU_DEBUG"))
        std::fprintf(stderr, "[rfgpu] orth: shifted CholeskyQR3 %s (min residual / ||X||_F = %.3e, gate %.3e)\n",
                     ok ? "accepted" : "rejected", c->h_d[1], c->h_d[0]);
    }
    if (ok) {
      out->fast = true;
      out->r = cols;
      if (R) {  // R = R3 R2 R1
        RF_TRY(gemm(c, false, cols, cols, cols, R2, cols, R1, cols, G2, cols));
        RF_TRY(gemm(c, false, cols, cols, cols, R3, cols, G2, cols, R, cols));
      }
      if (fold) {
        RF_CUDA(cudaMemcpyAsync(R2inv_buf, R3i, sizeof(double) * cc, cudaMemcpyDeviceToDevice, st));
        out->R2inv = R2inv_buf;
        out->folded = true;
      } else {
        RF_TRY(gemm(c, false, m, cols, cols, Q2, ldq2, R3i, cols, out->Q, out->ldq, nullptr, "trsm", false, true));
      }
      return {};
    }
  }
  // Gram-Schmidt with the reference's drop rule (its basis replaces Q1 in out->Q).
  if (oz) oz->thin_src = nullptr;
  DBuf gw;
  RF_TRY(gw.alloc(sizeof(double) * gs_orth_work_doubles(m, cols) + 64, st));
  int64_t* r_dev = reinterpret_cast<int64_t*>(gw.d() + gs_orth_work_doubles(m, cols));
  RF_CUDA(gs_orth(X, m, cols, ldx, out->Q, out->ldq, r_dev, gw.d(), dist ? allreduce_of(c) : DeviceAllreduce{}, st));
  RF_CUDA(cudaMemcpyAsync(c->h_i64, r_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  RF_CUDA(cudaStreamSynchronize(st));
  out->r = c->h_i64[0];
  return {};
}

// Z (n x r) = A^T Q for a (possibly folded) basis: (A^T Q1) R2^{-1}; summed
// over ranks. tmp: n x r scratch.
Status pass_tn(rfgpu_ctx* c, const rfgpu_matrix* a, const Basis& b, double* Z, double* tmp, OzPasses* oz = nullptr) {
  const int64_t n = a->n;
  double* dst = b.folded ? tmp : Z;
  RF_TRY(pass_tn_raw(c, a, b.Q, b.ldq, b.r, dst, oz));
  RF_TRY(allreduce(c, dst, n * b.r));
  if (b.folded) RF_TRY(gemm(c, false, n, b.r, b.r, tmp, n, b.R2inv, b.r, Z, n, nullptr, nullptr, false, true));
  return {};
}

// The Jacobi sweeps of a triangular QR factor R run on R^T (on R's rows): R R^T is closer to diagonal than
// R^T R, so the one-sided sweeps converge sooner (Drmac & Veselic's preconditioning, here without the column
// pivoting). R^T = U' S V'^T  =>  R = V' S U'^T: the two output buffers swap roles. Measured on graded
// l x l factors (tools/jac_bench.py): l = 110 / 220 / 330: 14 -> 11, 16 -> 13, 18 -> 13 block sweeps,
// 2.46 -> 1.93, 6.05 -> 4.70, 13.8 -> 9.86 ms; config 4: 85.4 -> 83.3 ms.
constexpr bool kJacobiOnTranspose = true;
inline bool jacobi_on_transpose() { return kJacobiOnTranspose; }

// ---- small SVD of B (ell x n) given Bt = B^T (n x ell, replicated) -------------
// Produces Ub (ell x ell: left singular vectors of B), D (ell), Vb (n x ell:
// right singular vectors of B), matching svd_dense(B) (dense.cpp:690-701).
Status small_svd_of_bt(rfgpu_ctx* c, const double* Bt, int64_t n, int64_t ell, double* Ub, double* D, double* Vb) {
  Timed t(c, "small_svd");
  cudaStream_t st = c->stream;
  const int64_t ldn = even(n);
  DBuf qb, rb, r2i, ur, ur2, jw, inf;
  RF_TRY(qb.alloc(sizeof(double) * ldn * ell, st));
  RF_TRY(rb.alloc(sizeof(double) * ell * ell, st));
  RF_TRY(r2i.alloc(sizeof(double) * ell * ell, st));
  RF_TRY(inf.alloc(64, st));
  Basis bq;
  bq.Q = qb.d();
  bq.ldq = ldn;
  RF_TRY(orth(c, Bt, n, ell, n, &bq, r2i.d(), rb.d(), /*dist=*/false, /*fold=*/true));
  int* info = inf.as<int>();
  if (bq.fast) {
    // Bt = Q1 R2^{-1} R; R = Ur S Vr^T  =>  B = Vr S (Q1 R2^{-1} Ur)^T
    RF_TRY(ur.alloc(sizeof(double) * ell * ell, st));
    RF_TRY(ur2.alloc(sizeof(double) * ell * ell, st));
    const size_t jwb = jacobi_work_bytes(ell, ell);
    if (jwb) RF_TRY(jw.alloc(jwb, st));
    DBuf rt;
    if (jacobi_on_transpose()) {
      RF_TRY(rt.alloc(sizeof(double) * ell * ell, st));
      RF_CUDA(transpose(rb.d(), ell, ell, ell, rt.d(), ell, st));
    }
    {
      Timed tj(c, "jacobi");
      if (rt.d())
        RF_CUDA(jacobi_svd(rt.d(), ell, ell, Ub, D, ur.d(), jw.d(), info, info + 1, st));
      else
        RF_CUDA(jacobi_svd(rb.d(), ell, ell, ur.d(), D, Ub, jw.d(), info, info + 1, st));
    }
    RF_TRY(gemm(c, false, ell, ell, ell, bq.R2inv, ell, ur.d(), ell, ur2.d(), ell));
    RF_TRY(gemm(c, false, n, ell, ell, bq.Q, ldn, ur2.d(), ell, Vb, n));
  } else {
    // rank-deficient / ill-conditioned B: Jacobi directly on the tall Bt
    const size_t jwb = jacobi_work_bytes(n, ell);
    if (jwb) RF_TRY(jw.alloc(jwb, st));
    Timed tj(c, "jacobi");
    RF_CUDA(jacobi_svd(Bt, n, ell, Vb, D, Ub, jw.d(), info, info + 1, st, /*sorted=*/true));
  }
  if (c->spec) {  // convergence checked at the end of the call
    rfgpu::jacobi_gate_kernel<<<1, 1, 0, st>>>(info, c->spec_flags);
    count_launch();
    RF_CUDA(cudaGetLastError());
    return {};
  }
  RF_CUDA(cudaMemcpyAsync(c->h_info, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  RF_CUDA(cudaStreamSynchronize(st));
  if (std::getenv("RFGPU_DEBUG"))
    std::fprintf(stderr, "[rfgpu] small_svd ell=%lld fast=%d jacobi info=%d sweeps=%d\n", (long long)ell,
                 (int)bq.fast, c->h_info[0], c->h_info[1]);
  if (c->h_info[0] == 1) return make_err(RFGPU_ECONVERGENCE, "svd_dense: Jacobi sweeps did not converge");
  return {};
}

// ---- range finder core ------------------------------------------------------------
struct RangeOut {
  Basis basis;           // Q (possibly folded: Q = basis.Q * basis.R2inv)
  double a_frob2 = 0.0;  // ||A||_F^2 (global)
};

// A (m_loc x n) handle; G (n x ell) on the device. Qbuf (ldq x ell) and
// R2ibuf (ell x ell) receive the basis; Bt (n x ell, ld n) receives
// B^T = A^T Q (summed over ranks). power_range, rangefinder.cpp:63-80.
Status range_core(rfgpu_ctx* c, const rfgpu_matrix* a, const double* G, int64_t ell, int64_t q, bool reorth,
                  double* Qbuf, int64_t ldq, double* R2ibuf, double* Bt, RangeOut* out) {
  cudaStream_t st = c->stream;
  const int64_t m = a->m, n = a->n;
  DBuf y, z, w, tmp, ssq, scal;
  RF_TRY(y.alloc(sizeof(double) * std::max<int64_t>(1, ldq * ell), st));
  RF_TRY(z.alloc(sizeof(double) * n * ell, st));
  RF_TRY(w.alloc(sizeof(double) * n * ell, st));
  RF_TRY(tmp.alloc(sizeof(double) * n * ell, st));
  OzPasses oz;
  RF_TRY(oz.init(c, a, ell));
  const int64_t slots = pass1_slots(c, a, ell, oz);
  RF_TRY(ssq.alloc(sizeof(double) * std::max<int64_t>(1, slots), st));
  RF_TRY(scal.alloc(sizeof(double) * 4, st));
  RF_CUDA(cudaMemsetAsync(ssq.d(), 0, sizeof(double) * std::max<int64_t>(1, slots), st));

  Basis& Qb = out->basis;
  Qb.Q = Qbuf;
  Qb.ldq = ldq;
  // pass 1: Y = A G, with ||A||_F^2 fused (streams a host A in by panels)
  RF_TRY(pass1(c, a, G, ell, y.d(), ldq, ssq.d(), oz));
  RF_CUDA(sum_array(ssq.d(), slots, scal.d(), st));
  RF_TRY(allreduce(c, scal.d(), 1));

  if (!reorth) {
    for (int64_t j = 0; j < q; ++j) {
      RF_TRY(pass_tn_raw(c, a, y.d(), ldq, ell, z.d(), &oz));
      RF_TRY(allreduce(c, z.d(), n * ell));
      RF_TRY(pass_nn(c, a, z.d(), ell, y.d(), ldq, &oz));
    }
    RF_TRY(orth(c, y.d(), m, ell, ldq, &Qb, R2ibuf, nullptr, true, true, &oz));
  } else {
    // every basis but the last only feeds the next product: CholeskyQR (one Gram) suffices for it (orth's
    // `single`); the last one (B = Q^T A, U = Q Ub) is CholeskyQR2
    RF_TRY(orth(c, y.d(), m, ell, ldq, &Qb, R2ibuf, nullptr, true, true, &oz, /*single=*/q > 0));
    for (int64_t j = 0; j < q && Qb.r > 0; ++j) {
      RF_TRY(pass_tn(c, a, Qb, z.d(), tmp.d(), &oz));
      Basis Wb;
      Wb.Q = w.d();
      Wb.ldq = n;
      RF_TRY(orth(c, z.d(), n, Qb.r, n, &Wb, nullptr, nullptr, false, false, nullptr, /*single=*/true));
      if (Wb.r == 0) {
        Qb.r = 0;
        break;
      }
      RF_TRY(pass_nn(c, a, w.d(), Wb.r, y.d(), ldq, &oz));
      RF_TRY(orth(c, y.d(), m, Wb.r, ldq, &Qb, R2ibuf, nullptr, true, true, &oz, /*single=*/j + 1 < q));
    }
  }
  // projection: B^T = A^T Q (finish_with_projection, rangefinder.cpp:24-30)
  if (Qb.r > 0) RF_TRY(pass_tn(c, a, Qb, Bt, tmp.d(), &oz));
  if (c->spec) {  // read once at the end of the call (spec_finish)
    RF_CUDA(cudaMemcpyAsync(c->spec_vals, scal.d(), sizeof(double), cudaMemcpyDeviceToDevice, st));
    out->a_frob2 = -1.0;
    return {};
  }
  RF_CUDA(cudaMemcpyAsync(c->h_d, scal.d(), sizeof(double), cudaMemcpyDeviceToHost, st));
  RF_CUDA(cudaStreamSynchronize(st));
  out->a_frob2 = c->h_d[0];
  return {};
}

// Explicit Q (m x r, ld ldo) from a possibly folded basis.
Status materialize_q(rfgpu_ctx* c, int64_t m, const Basis& b, double* Qo, int64_t ldo) {
  if (b.r == 0 || m == 0) return {};
  if (b.folded) return gemm(c, false, m, b.r, b.r, b.Q, b.ldq, b.R2inv, b.r, Qo, ldo, nullptr, "trsm", false, true);
  RF_CUDA(cudaMemcpy2DAsync(Qo, sizeof(double) * ldo, b.Q, sizeof(double) * b.ldq, sizeof(double) * m, b.r,
                            cudaMemcpyDeviceToDevice, c->stream));
  return {};
}

constexpr int kSpecRetry = 100;  // internal: a speculative call must be re-run without speculation

// frob_residual (rangefinder.cpp:45-54) from ||A||_F^2 and B^T on the device.
Status frob_residual_dev(rfgpu_ctx* c, double a_frob2, const double* Bt, int64_t count, double* resid) {
  cudaStream_t st = c->stream;
  if (c->spec) {  // ||B||_F^2 into spec_vals[1]; compared with ||A||_F^2 in spec_finish
    DBuf part;
    RF_TRY(part.alloc(sizeof(double) * 1024, st));
    if (count > 0)
      RF_CUDA(sumsq(Bt, count, part.d(), c->spec_vals + 1, st));
    else
      RF_CUDA(cudaMemsetAsync(c->spec_vals + 1, 0, sizeof(double), st));
    return {};
  }
  DBuf part, out;
  RF_TRY(part.alloc(sizeof(double) * 1024, st));
  RF_TRY(out.alloc(sizeof(double), st));
  double bn2 = 0.0;
  if (count > 0) {
    RF_CUDA(sumsq(Bt, count, part.d(), out.d(), st));
    RF_CUDA(cudaMemcpyAsync(c->h_d, out.d(), sizeof(double), cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaStreamSynchronize(st));
    bn2 = c->h_d[0];
  }
  const double a_frob = std::sqrt(a_frob2);
  const double bn = std::sqrt(bn2);
  if (bn > a_frob * (1.0 + 1e-8))
    return make_err(RFGPU_ENUMERICAL,
                    "frob_residual: projection exceeds the total norm; basis orthonormality was lost upstream");
  const double diff = a_frob * a_frob - bn * bn;
  if (resid) *resid = std::sqrt(std::max(0.0, diff));
  return {};
}

// End of a speculative call: the one host round trip. kSpecRetry when an orth
// gate or a Jacobi failed (the caller re-runs without speculation), else the
// frob_residual check and value.
Status spec_check(rfgpu_ctx* c, double* resid);

Status spec_finish(rfgpu_ctx* c, double* resid) {
  cudaStream_t st = c->stream;
  RF_CUDA(cudaMemcpyAsync(c->h_spec, c->spec_flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  RF_CUDA(cudaMemcpyAsync(static_cast<char*>(c->h_spec) + 16, c->spec_vals, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                          st));
  if (c->capturing) return {};  // checked after each replay of the graph
  return spec_check(c, resid);
}

Status spec_check(rfgpu_ctx* c, double* resid) {
  RF_CUDA(cudaStreamSynchronize(c->stream));
  const int* fl = static_cast<const int*>(c->h_spec);
  const double* v = reinterpret_cast<const double*>(static_cast<const char*>(c->h_spec) + 16);
  if (fl[0] || fl[1]) {
    if (std::getenv("RFGPU_DEBUG"))
      std::fprintf(stderr, "[rfgpu] speculation failed (orth gate %d, jacobi %d): re-running\n", fl[0], fl[1]);
    return make_err(kSpecRetry, "speculative CholeskyQR2 rejected");
  }
  const double a_frob = std::sqrt(v[0]), bn = std::sqrt(v[1]);
  if (bn > a_frob * (1.0 + 1e-8))
    return make_err(RFGPU_ENUMERICAL,
                    "frob_residual: projection exceeds the total norm; basis orthonormality was lost upstream");
  if (resid) *resid = std::sqrt(std::max(0.0, a_frob * a_frob - bn * bn));
  return {};
}

// Runs body() speculatively (no host round trip inside; RFGPU_SPECULATE=0
// disables) and again without speculation if the speculation failed.
// Argument set of a call (entry point, matrix, shape, sketch parameters) for the per-context memo of
// rejected speculations and recorded graphs.
std::vector<int64_t> call_key(int entry, const rfgpu_matrix* a, int64_t k, int64_t ell, int64_t q, int reorth) {
  return {entry, reinterpret_cast<int64_t>(a), reinterpret_cast<int64_t>(a ? a->dev : nullptr), a ? a->m : 0,
          a ? a->n : 0, a ? a->lda : 0, k, ell, q, reorth};
}

template <class F>
Status with_speculation(rfgpu_ctx* c, const std::vector<int64_t>& key, F&& body) {
  const char* e = std::getenv("RFGPU_SPECULATE");
  if ((e && e[0] == '0') || c->spec_failed.count(key)) return body();
  RF_CUDA(cudaMemsetAsync(c->spec_flags, 0, 2 * sizeof(int), c->stream));
  c->spec = true;
  Status s = body();
  c->spec = false;
  if (s.code == kSpecRetry) {  // the same arguments will fail again (rank-deficient or plain-mode sketch)
    c->spec_failed[key] = true;
    s = body();
  }
  return s;
}

// ---- CUDA graphs of whole calls --------------------------------------------------------------
// RFGPU_GRAPH=0 disables. Not with profiling (per-phase events), multi-rank contexts or a host-resident input.
bool graphs_enabled(rfgpu_ctx* c) {
  const char* e = std::getenv("RFGPU_GRAPH");
  // single GPU only: multi-rank calls keep their collectives outside graphs (not exercised on one-GPU boxes)
  return !(e && e[0] == '0') && !c->profile && !c->host_sum && c->world == 1;
}

// The RFGPU_* switches decide which kernels a call records (digit path or DMMA, Gram kernel, Jacobi variant):
// their values are part of a graph's key, so a call made under different switches never replays a graph
// recorded under the old ones (bench.py's DMMA self-check re-runs the same call with RFGPU_OZAKI=0).
int64_t env_signature() {
  uint64_t h = 1469598103934665603ull;
  for (const char* name : {"RFGPU_OZAKI", "RFGPU_OZAKI_SHARED", "RFGPU_DIGIT_GRAM",
                           "RFGPU_JACOBI_BLOCK"}) {
    const char* v = std::getenv(name);
    for (const char* p = v ? v : "\x01"; *p; ++p) h = (h ^ static_cast<unsigned char>(*p)) * 1099511628211ull;
    h = (h ^ 0xffu) * 1099511628211ull;
  }
  return static_cast<int64_t>(h);
}

void graph_drop(rfgpu_ctx* c, const std::vector<int64_t>& key) {
  for (size_t i = 0; i < c->graphs.size(); ++i)
    if (c->graphs[i].key == key) {
      cudaGraphExecDestroy(c->graphs[i].exec);
      c->graphs.erase(c->graphs.begin() + static_cast<long>(i));
      break;
    }
  c->graph_seen[key] = -1000000;
  cudaDeviceGraphMemTrim(c->device);  // the dropped graph's memory back to the driver
}

rfgpu_ctx::GraphEntry* graph_lookup(rfgpu_ctx* c, const std::vector<int64_t>& key) {
  for (auto& g : c->graphs)
    if (g.key == key) return &g;
  return nullptr;
}

// Records body() (speculative, ending in spec_finish's flag copies) into a graph. Returns nullptr (and leaves
// the stream usable) when the call cannot be captured; the caller then runs it eagerly.
template <class F>
rfgpu_ctx::GraphEntry* graph_capture(rfgpu_ctx* c, const std::vector<int64_t>& key, F&& body, int64_t* rank) {
  cudaStream_t st = c->stream;
  if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  const int64_t l0 = launch_counter();
  c->capturing = true;
  c->spec = true;
  Status s;
  if (cudaMemsetAsync(c->spec_flags, 0, 2 * sizeof(int), st) != cudaSuccess) s = make_err(RFGPU_ECUDA, "capture");
  if (s.ok()) s = body();
  c->capturing = false;
  c->spec = false;
  const int64_t recorded = launch_counter() - l0;
  count_launch(static_cast<int>(-recorded));  // recorded, not launched
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(st, &g);
  cudaGraphExec_t exec = nullptr;
  const bool ok = s.ok() && e == cudaSuccess && g && cudaGraphInstantiate(&exec, g, 0) == cudaSuccess;
  if (g) cudaGraphDestroy(g);
  if (!ok) {
    cudaGetLastError();
    if (std::getenv("RFGPU_DEBUG")) std::fprintf(stderr, "[rfgpu] graph capture failed (%s): eager\n", s.msg.c_str());
    c->graph_seen[key] = -1000000;  // do not try again for these arguments
    return nullptr;
  }
  // the eager calls' cached blocks are not needed by the graph (it owns its memory)
  for (cudaMemPool_t pool : {c->pool_small, c->pool_large}) cudaMemPoolTrimTo(pool, 0);
  c->graphs.push_back({key, exec, recorded, *rank});
  return &c->graphs.back();
}

Status check_sample(const rfgpu_matrix* a, int64_t k, int64_t ell, const char* where) {
  if (k < 1) return make_err(RFGPU_EPARAM, std::string(where) + ": k must be at least 1");
  if (ell < k) return make_err(RFGPU_EPARAM, std::string(where) + ": p must be non-negative");
  if (ell > std::min(a->m_global, a->n)) return make_err(RFGPU_EPARAM, std::string(where) + ": k + p exceeds min(m, n)");
  // the l x l factorizations (Cholesky / triangular inverse of the Gram matrices) hold a block column in one
  // CTA's shared memory: l <= 736 (no such bound in the reference; reported as a parameter error, not a crash)
  if (ell > 736) return make_err(RFGPU_EPARAM, std::string(where) + ": k + p above 736 is not supported on the device");
  return {};
}

// rsvd on device buffers; U (ldu x ell), D (ell), V (n x ell). lowrank.cpp:74-96.
Status rsvd_core(rfgpu_ctx* c, const rfgpu_matrix* a, const double* G, int64_t k, int64_t ell, int64_t q, bool keep_over,
                 bool reorth, double* U, int64_t ldu, double* D, double* V, int64_t* rank_out, double* Uhost = nullptr,
                 int64_t ldh = 0) {
  cudaStream_t st = c->stream;
  const int64_t m = a->m, n = a->n;
  const int64_t ldq = even(m);
  DBuf Q, R2i, Bt, Ub, Ub2, Vb, Dd;
  RF_TRY(Q.alloc(sizeof(double) * std::max<int64_t>(1, ldq * ell), st));
  RF_TRY(R2i.alloc(sizeof(double) * ell * ell, st));
  RF_TRY(Bt.alloc(sizeof(double) * n * ell, st));
  RangeOut ro;
  RF_TRY(range_core(c, a, G, ell, q, reorth, Q.d(), ldq, R2i.d(), Bt.d(), &ro));
  const Basis& b = ro.basis;
  const int64_t r = b.r;
  RF_TRY(frob_residual_dev(c, ro.a_frob2, Bt.d(), n * r, nullptr));
  if (r == 0) {
    *rank_out = 0;
    return {};
  }
  RF_TRY(Ub.alloc(sizeof(double) * r * r, st));
  RF_TRY(Ub2.alloc(sizeof(double) * r * r, st));
  RF_TRY(Vb.alloc(sizeof(double) * n * r, st));
  RF_TRY(Dd.alloc(sizeof(double) * r, st));
  RF_TRY(small_svd_of_bt(c, Bt.d(), n, r, Ub.d(), Dd.d(), Vb.d()));
  const int64_t keep = keep_over ? r : std::min(k, r);
  // lift: U = Q Ub(:, :keep) = Q1 (R2^{-1} Ub(:, :keep))
  const double* ub = Ub.d();
  if (b.folded) {
    RF_TRY(gemm(c, false, r, keep, r, b.R2inv, r, Ub.d(), r, Ub2.d(), r));
    ub = Ub2.d();
  }
  if (Uhost && c->copy_stream && host_is_pageable(Uhost)) {
    // pageable destination: lift, then read U back through the pinned ring (copy stream, host copy threads)
    RF_TRY(gemm(c, false, m, keep, r, b.Q, b.ldq, ub, r, U, ldu, nullptr, "lift"));
    cudaEvent_t lifted;
    RF_CUDA(cudaEventCreateWithFlags(&lifted, cudaEventDisableTiming));
    RF_CUDA(cudaEventRecord(lifted, st));
    RF_CUDA(cudaStreamWaitEvent(c->copy_stream, lifted, 0));
    cudaEventDestroy(lifted);
    RF_TRY(staged_d2h(c, Uhost, ldh, U, ldu, m, keep, c->copy_stream));
  } else if (Uhost && c->copy_stream && m >= 65536) {
    // Lift in row panels and read each one back on the copy stream while the next is computed. All the
    // GEMMs are queued before the first copy so a pageable destination (whose copy blocks the host)
    // cannot serialise them.
    constexpr int kPanels = 8;
    const int64_t step = (m + kPanels * 128 - 1) / (kPanels * 128) * 128;  // keeps every panel base 16-byte aligned
    cudaEvent_t ev[kPanels];
    int np = 0;
    Status gs;
    cudaError_t e = cudaSuccess;
    for (int64_t r0 = 0; r0 < m && gs.ok() && e == cudaSuccess; r0 += step) {
      const int64_t rows = std::min(step, m - r0);
      gs = gemm(c, false, rows, keep, r, b.Q + r0, b.ldq, ub, r, U + r0, ldu, nullptr, "lift");
      if (gs.ok()) e = cudaEventCreateWithFlags(&ev[np], cudaEventDisableTiming);
      if (gs.ok() && e == cudaSuccess) {
        ++np;
        e = cudaEventRecord(ev[np - 1], st);
      }
    }
    if (!gs.ok()) {
      for (int p = 0; p < np; ++p) cudaEventDestroy(ev[p]);
      return gs;
    }
    for (int p = 0; p < np; ++p) {
      const int64_t r0 = p * step, rows = std::min(step, m - r0);
      if (e == cudaSuccess) e = cudaStreamWaitEvent(c->copy_stream, ev[p], 0);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(Uhost + r0, sizeof(double) * ldh, U + r0, sizeof(double) * ldu, sizeof(double) * rows,
                              keep, cudaMemcpyDeviceToHost, c->copy_stream);
      cudaEventDestroy(ev[p]);
    }
    if (e == cudaSuccess) {
      cudaEvent_t done;
      e = cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
      if (e == cudaSuccess) {
        e = cudaEventRecord(done, c->copy_stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, done, 0);
        cudaEventDestroy(done);
      }
    }
    RF_CUDA(e);
  } else {
    RF_TRY(gemm(c, false, m, keep, r, b.Q, b.ldq, ub, r, U, ldu, nullptr, "lift"));
    if (Uhost) {
      RF_CUDA(cudaMemcpy2DAsync(Uhost, sizeof(double) * ldh, U, sizeof(double) * ldu, sizeof(double) * m, keep,
                                cudaMemcpyDeviceToHost, st));
    }
  }
  RF_CUDA(cudaMemcpyAsync(V, Vb.d(), sizeof(double) * n * keep, cudaMemcpyDeviceToDevice, st));
  RF_CUDA(cudaMemcpyAsync(D, Dd.d(), sizeof(double) * keep, cudaMemcpyDeviceToDevice, st));
  if (c->spec) RF_TRY(spec_finish(c, nullptr));
  *rank_out = keep;
  return {};
}

// ---- interpolative decompositions ------------------------------------------------
inline unsigned grid1d(int64_t n) { return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1184))); }

// SVD of a tall replicated matrix M (rows x c, ld ldm): M = Um diag(S) Vm^T
// (svd_dense semantics, dense.cpp:585-701) via CholeskyQR2 + Jacobi on the
// c x c factor, Jacobi on M itself when CholeskyQR is not accepted.
Status svd_tall_dev(rfgpu_ctx* c, const double* M, int64_t rows, int64_t cols, int64_t ldm, double* Um, double* S,
                    double* Vm, bool dist = false) {
  cudaStream_t st = c->stream;
  const int64_t ldr = even(rows);
  DBuf q, rr, r2i, ur, ur2, jw, inf, mc;
  RF_TRY(q.alloc(sizeof(double) * std::max<int64_t>(1, ldr * cols), st));
  RF_TRY(rr.alloc(sizeof(double) * cols * cols, st));
  RF_TRY(r2i.alloc(sizeof(double) * cols * cols, st));
  RF_TRY(inf.alloc(64, st));
  Basis b;
  b.Q = q.d();
  b.ldq = ldr;
  RF_TRY(orth(c, M, rows, cols, ldm, &b, r2i.d(), rr.d(), dist, true));
  int* info = inf.as<int>();
  if (dist && !b.fast) {
    // Row-sharded M, rank-deficient / ill-conditioned: the Gram-Schmidt basis
    // Q (rows x r) spans M's columns up to the reference drop rule, so
    // M = Q R with R = Q^T M (summed over ranks); SVD of the replicated R.
    const int64_t r = b.r;
    DBuf rq;
    RF_TRY(rq.alloc(sizeof(double) * std::max<int64_t>(1, r * cols), st));
    RF_TRY(ur.alloc(sizeof(double) * std::max<int64_t>(1, r * cols), st));
    if (r > 0) {
      RF_TRY(gemm(c, true, r, cols, rows, b.Q, b.ldq, M, ldm, rq.d(), r));
      RF_TRY(allreduce(c, rq.d(), r * cols));
      const size_t jwb = jacobi_work_bytes(r, cols);
      if (jwb) RF_TRY(jw.alloc(jwb, st));
      Timed tj(c, "jacobi");
      RF_CUDA(jacobi_svd(rq.d(), r, cols, ur.d(), S, Vm, jw.d(), info, info + 1, st, /*sorted=*/true));
    }
    RF_CUDA(cudaMemsetAsync(Um, 0, sizeof(double) * rows * cols, st));
    if (r > 0) RF_TRY(gemm(c, false, rows, cols, r, b.Q, b.ldq, ur.d(), r, Um, rows));
    if (r == 0) {
      RF_CUDA(cudaMemsetAsync(S, 0, sizeof(double) * cols, st));
      return {};
    }
  } else if (b.fast) {
    RF_TRY(ur.alloc(sizeof(double) * cols * cols, st));
    RF_TRY(ur2.alloc(sizeof(double) * cols * cols, st));
    const size_t jwb = jacobi_work_bytes(cols, cols);
    if (jwb) RF_TRY(jw.alloc(jwb, st));
    DBuf rt;
    if (jacobi_on_transpose()) {
      RF_TRY(rt.alloc(sizeof(double) * cols * cols, st));
      RF_CUDA(transpose(rr.d(), cols, cols, cols, rt.d(), cols, st));
    }
    {
      Timed tj(c, "jacobi");
      if (rt.d())
        RF_CUDA(jacobi_svd(rt.d(), cols, cols, Vm, S, ur.d(), jw.d(), info, info + 1, st));
      else
        RF_CUDA(jacobi_svd(rr.d(), cols, cols, ur.d(), S, Vm, jw.d(), info, info + 1, st));
    }
    RF_TRY(gemm(c, false, cols, cols, cols, b.R2inv, cols, ur.d(), cols, ur2.d(), cols));
    RF_TRY(gemm(c, false, rows, cols, cols, b.Q, ldr, ur2.d(), cols, Um, rows));
  } else {
    // Jacobi reads rows with stride `rows`: compact copy when ldm != rows
    const double* src = M;
    if (ldm != rows) {
      RF_TRY(mc.alloc(sizeof(double) * rows * cols, st));
      RF_CUDA(cudaMemcpy2DAsync(mc.d(), sizeof(double) * rows, M, sizeof(double) * ldm, sizeof(double) * rows, cols,
                                cudaMemcpyDeviceToDevice, st));
      src = mc.d();
    }
    const size_t jwb = jacobi_work_bytes(rows, cols);
    if (jwb) RF_TRY(jw.alloc(jwb, st));
    Timed tj(c, "jacobi");
    RF_CUDA(jacobi_svd(src, rows, cols, Um, S, Vm, jw.d(), info, info + 1, st, /*sorted=*/true));
  }
  RF_CUDA(cudaMemcpyAsync(c->h_info, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  RF_CUDA(cudaStreamSynchronize(st));
  if (std::getenv("RFGPU_DEBUG"))
    std::fprintf(stderr, "[rfgpu] svd_tall %lldx%lld fast=%d jacobi info=%d sweeps=%d\n", (long long)rows,
                 (long long)cols, (int)b.fast, c->h_info[0], c->h_info[1]);
  if (c->h_info[0] == 1) return make_err(RFGPU_ECONVERGENCE, "svd_dense: Jacobi sweeps did not converge");
  return {};
}

// col_id_core (lowrank.cpp:51-70) of Y (m x n, ld ldy; not modified). Z_dev
// receives ke x n (ld ke); Js_dev / Js_host (either may be null) the skeleton.
Status col_id_dev(rfgpu_ctx* c, const double* Y, int64_t m, int64_t n, int64_t ldy, int64_t k, int64_t* Js_dev,
                  int64_t* Js_host, double* Z, int64_t* ke_out, int* truncated) {
  Timed t(c, "col_id");
  cudaStream_t st = c->stream;
  if (m > 512) return make_err(RFGPU_EPARAM, "col_id: sketch height above 512 is not supported on the device path");
  if (k < 0 || k > std::min(m, n)) return make_err(RFGPU_EPARAM, "cpqr: rank target out of range");
  const int64_t ldw = even(m);
  DBuf W, perm, work, part, scal, R11i, T;
  RF_TRY(W.alloc(sizeof(double) * ldw * std::max<int64_t>(1, n), st));
  RF_TRY(perm.alloc(sizeof(int64_t) * std::max<int64_t>(1, n), st));
  RF_TRY(work.alloc(cpqr_work_bytes(n, c->num_sms, static_cast<int>(m)), st));
  RF_TRY(part.alloc(sizeof(double) * 1024, st));
  RF_TRY(scal.alloc(64, st));
  if (n > 0 && m > 0)
    RF_CUDA(cudaMemcpy2DAsync(W.d(), sizeof(double) * ldw, Y, sizeof(double) * ldy, sizeof(double) * m, n,
                              cudaMemcpyDeviceToDevice, st));
  // halt = 1e-14 ||Y||_F (dense.cpp:473-474)
  double fro2 = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += 1) {
    if (ldw == m) {
      RF_CUDA(sumsq(W.d(), m * n, part.d(), scal.d(), st));
      break;
    }
    // ld padding: zero the pad row so a flat sum of squares is exact
    RF_CUDA(cudaMemset2DAsync(W.d() + m, sizeof(double) * ldw, 0, sizeof(double), n, st));
    RF_CUDA(sumsq(W.d(), ldw * n, part.d(), scal.d(), st));
    break;
  }
  int* stopped = reinterpret_cast<int*>(scal.d() + 2);
  RF_CUDA(cudaMemsetAsync(stopped, 0, 2 * sizeof(int), st));
  RF_CUDA(cudaMemcpyAsync(c->h_d, scal.d(), sizeof(double), cudaMemcpyDeviceToHost, st));
  RF_CUDA(cudaStreamSynchronize(st));
  fro2 = c->h_d[0];
  {
    Timed tq(c, "cpqr");
    RF_CUDA(cpqr_rank(W.d(), ldw, static_cast<int>(m), n, static_cast<int>(k), 1e-14 * std::sqrt(fro2), perm.as<int64_t>(),
                      work.p, stopped, stopped + 1, c->num_sms, st));
  }
  RF_CUDA(cudaMemcpyAsync(c->h_info, stopped, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  RF_CUDA(cudaStreamSynchronize(st));
  const int64_t ke = std::min<int64_t>(k, c->h_info[0]);
  *ke_out = ke;
  if (truncated) *truncated = ke < k ? 1 : 0;
  if (std::getenv("RFGPU_DEBUG"))
    std::fprintf(stderr, "[rfgpu] cpqr m=%lld n=%lld k=%lld stopped=%d recomputes=%d\n", (long long)m, (long long)n,
                 (long long)k, c->h_info[0], c->h_info[1]);
  if (Js_dev && ke > 0) RF_CUDA(cudaMemcpyAsync(Js_dev, perm.d(), sizeof(int64_t) * ke, cudaMemcpyDeviceToDevice, st));
  if (Js_host && ke > 0) RF_CUDA(cudaMemcpyAsync(Js_host, perm.d(), sizeof(int64_t) * ke, cudaMemcpyDeviceToHost, st));
  if (ke > 0) {
    RF_TRY(T.alloc(sizeof(double) * ke * std::max<int64_t>(1, n - ke), st));
    if (n > ke) {
      RF_TRY(R11i.alloc(sizeof(double) * ke * ke, st));
      RF_CUDA(trinv_upper(W.d(), ldw, static_cast<int>(ke), R11i.d(), st));
      // T = S11^{-1} S12 (solve_upper, dense.cpp:788-804)
      RF_TRY(gemm(c, false, ke, n - ke, ke, R11i.d(), ke, W.d() + ke * ldw, ldw, T.d(), ke, nullptr, "trsm_id"));
    }
    RF_CUDA(assemble_z(perm.as<int64_t>(), static_cast<int>(ke), n, T.d(), Z, st));
  }
  RF_CUDA(cudaStreamSynchronize(st));
  return {};
}

// Transposed row sketch Yt = (G A)^T = A^T G^T (n x ell), q power passes
// (lowrank.cpp:351-355: y <- (y A^T) A). Gt: m_loc x ell (this rank's rows of
// G^T, ld ldg). Summed over ranks.
Status row_sketch_t(rfgpu_ctx* c, const rfgpu_matrix* a, const double* Gt, int64_t ldg, int64_t ell, int64_t q,
                    double* Yt) {
  const int64_t m = a->m, n = a->n;
  OzPasses oz;  // the passes over A on the INT8 tensor cores at pass sizes
  RF_TRY(oz.init(c, a, ell));
  if (oz.on) {
    DBuf ssq;
    RF_TRY(ssq.alloc(sizeof(double) * ozaki_ssq_slots(m, n), c->stream));
    RF_TRY(oz.prepare(c, a, ssq.d(), q > 0));
  }
  RF_TRY(pass_tn_raw(c, a, Gt, ldg, ell, Yt, &oz));
  RF_TRY(allreduce(c, Yt, n * ell));
  if (q > 0) {
    DBuf t;
    RF_TRY(t.alloc(sizeof(double) * std::max<int64_t>(1, even(m) * ell), c->stream));
    for (int64_t j = 0; j < q; ++j) {
      RF_TRY(pass_nn(c, a, Yt, ell, t.d(), even(m), &oz));
      RF_TRY(pass_tn_raw(c, a, t.d(), even(m), ell, Yt, &oz));
      RF_TRY(allreduce(c, Yt, n * ell));
    }
  }
  return {};
}

// Two tall SVDs of the same width (svd_tall_dev semantics each): both
// orthonormalised, then their l x l Jacobi SVDs in ONE launch (one cluster
// each), so the two latency-bound round sequences run side by side.
struct TallSvd {
  const double* M;
  int64_t rows, ldm;
  double* U;
  double* S;
  double* V;
  bool dist;
};

Status svd_tall_pair(rfgpu_ctx* c, const TallSvd& x, const TallSvd& y, int64_t cols) {
  cudaStream_t st = c->stream;
  struct Side {
    DBuf q, rr, r2i, ur, ur2, jw, inf, rt;
    Basis b;
    int64_t ldr = 0;
  };
  Side sd[2];
  const TallSvd* t[2] = {&x, &y};
  for (int i = 0; i < 2; ++i) {
    sd[i].ldr = even(t[i]->rows);
    RF_TRY(sd[i].q.alloc(sizeof(double) * std::max<int64_t>(1, sd[i].ldr * cols), st));
    RF_TRY(sd[i].rr.alloc(sizeof(double) * cols * cols, st));
    RF_TRY(sd[i].r2i.alloc(sizeof(double) * cols * cols, st));
    RF_TRY(sd[i].inf.alloc(64, st));
    sd[i].b.Q = sd[i].q.d();
    sd[i].b.ldq = sd[i].ldr;
    RF_TRY(orth(c, t[i]->M, t[i]->rows, cols, t[i]->ldm, &sd[i].b, sd[i].r2i.d(), sd[i].rr.d(), t[i]->dist, true));
  }
  if (!sd[0].b.fast || !sd[1].b.fast) {  // rank-deficient side: one at a time
    RF_TRY(svd_tall_dev(c, x.M, x.rows, cols, x.ldm, x.U, x.S, x.V, x.dist));
    return svd_tall_dev(c, y.M, y.rows, cols, y.ldm, y.U, y.S, y.V, y.dist);
  }
  JacobiProblem pj[2];
  for (int i = 0; i < 2; ++i) {
    RF_TRY(sd[i].ur.alloc(sizeof(double) * cols * cols, st));
    RF_TRY(sd[i].ur2.alloc(sizeof(double) * cols * cols, st));
    const size_t jwb = jacobi_work_bytes(cols, cols);
    RF_TRY(sd[i].jw.alloc(std::max<size_t>(jwb, 16), st));
    int* info = sd[i].inf.as<int>();
    if (jacobi_on_transpose()) {  // on R^T: U and V swap (see jacobi_on_transpose)
      RF_TRY(sd[i].rt.alloc(sizeof(double) * cols * cols, st));
      RF_CUDA(transpose(sd[i].rr.d(), cols, cols, cols, sd[i].rt.d(), cols, st));
      pj[i] = JacobiProblem{sd[i].rt.d(), t[i]->V, t[i]->S, sd[i].ur.d(), sd[i].jw.d(), info, info + 1};
    } else {
      pj[i] = JacobiProblem{sd[i].rr.d(), sd[i].ur.d(), t[i]->S, t[i]->V, sd[i].jw.d(), info, info + 1};
    }
  }
  {
    Timed tj(c, "jacobi");
    RF_CUDA(jacobi_svd_pair(pj[0], pj[1], cols, cols, st));
  }
  for (int i = 0; i < 2; ++i) {
    RF_TRY(gemm(c, false, cols, cols, cols, sd[i].b.R2inv, cols, sd[i].ur.d(), cols, sd[i].ur2.d(), cols));
    RF_TRY(gemm(c, false, t[i]->rows, cols, cols, sd[i].b.Q, sd[i].ldr, sd[i].ur2.d(), cols, t[i]->U, t[i]->rows));
  }
  int h[4];
  for (int i = 0; i < 2; ++i)
    RF_CUDA(cudaMemcpyAsync(h + 2 * i, sd[i].inf.d(), 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  RF_CUDA(cudaStreamSynchronize(st));
  if (std::getenv("RFGPU_DEBUG"))
    std::fprintf(stderr, "[rfgpu] svd_tall pair %lldx%lld + %lldx%lld jacobi info=%d/%d sweeps=%d/%d\n",
                 (long long)x.rows, (long long)cols, (long long)y.rows, (long long)cols, h[0], h[2], h[1], h[3]);
  if (h[0] == 1 || h[2] == 1) return make_err(RFGPU_ECONVERGENCE, "svd_dense: Jacobi sweeps did not converge");
  return {};
}

// ---- single pass (lowrank.cpp:160-220) ------------------------------------------
// Core of single_pass_svd from the two sketches, all on the device:
// dominant_left(Yc, k), dominant_left(Yr, k) (:178-179), the small products
// P = Gr^T Qc, E = Yr^T Qr, W = Qr^T Gc, F = Qc^T Yc (:184-187), the core C
// from the normal equations of the reference's stacked least squares
// (P^T P C + C W W^T = P^T E + F W^T) solved in the
// eigenbases of P^T P and W W^T (right singular vectors of P and W^T), then
// svd(C) and the lift U = Qc Uc, V = Qr Vc (:214-218).
//
// Row-sharded A (dist): Yc, Gr (ld ldgr) and U hold this rank's rows; Yr
// (already summed) is replicated; the two products over m (P, F) are summed
// over ranks and the tall SVD of Yc runs on the sharded rows.
Status single_pass_core(rfgpu_ctx* c, const double* Yc, int64_t m, const double* Yr, int64_t n, const double* Gc,
                        const double* Gr, int64_t ldgr, int64_t k, int64_t ell, double* U, int64_t ldu, double* D,
                        double* V, int64_t* rank_out, bool dist = false) {
  Timed t(c, "single_pass_core");
  cudaStream_t st = c->stream;
  const int64_t kk = std::min(k, ell);
  DBuf uc, sc, vc, ur, sr, vr, P, E, W, F, Wt, up, sp, vp, uw, sw, vw, rhs, tmp, tmp2, cm, cu, cs, cv, den;
  RF_TRY(uc.alloc(sizeof(double) * m * ell, st));
  RF_TRY(sc.alloc(sizeof(double) * ell, st));
  RF_TRY(vc.alloc(sizeof(double) * ell * ell, st));
  RF_TRY(ur.alloc(sizeof(double) * n * ell, st));
  RF_TRY(sr.alloc(sizeof(double) * ell, st));
  RF_TRY(vr.alloc(sizeof(double) * ell * ell, st));
  // Qc = uc(:, :kk), Qr = ur(:, :kk): the two dominant_left SVDs side by side
  RF_TRY(svd_tall_pair(c, TallSvd{Yc, m, m, uc.d(), sc.d(), vc.d(), dist}, TallSvd{Yr, n, n, ur.d(), sr.d(), vr.d(), false},
                       ell));
  RF_TRY(P.alloc(sizeof(double) * ell * kk, st));
  RF_TRY(E.alloc(sizeof(double) * ell * kk, st));
  RF_TRY(W.alloc(sizeof(double) * kk * ell, st));
  RF_TRY(F.alloc(sizeof(double) * kk * ell, st));
  RF_TRY(Wt.alloc(sizeof(double) * ell * kk, st));
  RF_TRY(gemm(c, true, ell, kk, m, Gr, ldgr, uc.d(), m, P.d(), ell));   // P = Gr^T Qc
  if (dist) RF_TRY(allreduce(c, P.d(), ell * kk));
  RF_TRY(gemm(c, true, ell, kk, n, Yr, n, ur.d(), n, E.d(), ell));   // E = Yr^T Qr
  RF_TRY(gemm(c, true, kk, ell, n, ur.d(), n, Gc, n, W.d(), kk));    // W = Qr^T Gc
  RF_TRY(gemm(c, true, kk, ell, m, uc.d(), m, Yc, m, F.d(), kk));    // F = Qc^T Yc
  if (dist) RF_TRY(allreduce(c, F.d(), kk * ell));
  RF_CUDA(transpose(W.d(), kk, ell, kk, Wt.d(), ell, st));
  // P = Up Sp Vp^T  =>  P^T P = Vp Sp^2 Vp^T;  W^T = Uw Sw Vw^T => W W^T = Vw Sw^2 Vw^T
  RF_TRY(up.alloc(sizeof(double) * ell * kk, st));
  RF_TRY(sp.alloc(sizeof(double) * kk, st));
  RF_TRY(vp.alloc(sizeof(double) * kk * kk, st));
  RF_TRY(uw.alloc(sizeof(double) * ell * kk, st));
  RF_TRY(sw.alloc(sizeof(double) * kk, st));
  RF_TRY(vw.alloc(sizeof(double) * kk * kk, st));
  RF_TRY(svd_tall_pair(c, TallSvd{P.d(), ell, ell, up.d(), sp.d(), vp.d(), false},
                       TallSvd{Wt.d(), ell, ell, uw.d(), sw.d(), vw.d(), false}, kk));
  // RHS = P^T E + F W^T
  RF_TRY(rhs.alloc(sizeof(double) * kk * kk, st));
  RF_TRY(tmp.alloc(sizeof(double) * kk * kk, st));
  RF_TRY(tmp2.alloc(sizeof(double) * kk * kk, st));
  RF_TRY(gemm(c, true, kk, kk, ell, P.d(), ell, E.d(), ell, rhs.d(), kk));
  RF_TRY(gemm(c, false, kk, kk, ell, F.d(), kk, Wt.d(), ell, tmp.d(), kk));
  add_inplace_kernel<<<grid1d(kk * kk), 256, 0, st>>>(rhs.d(), tmp.d(), kk * kk);
  count_launch();
  // Ct = Vp^T RHS Vw ./ (sp_i^2 + sw_j^2);  C = Vp Ct Vw^T
  RF_TRY(gemm(c, true, kk, kk, kk, vp.d(), kk, rhs.d(), kk, tmp.d(), kk));
  RF_TRY(gemm(c, false, kk, kk, kk, tmp.d(), kk, vw.d(), kk, tmp2.d(), kk));
  sylvester_scale_kernel<<<grid1d(kk * kk), 256, 0, st>>>(tmp2.d(), kk, sp.d(), sw.d());
  count_launch();
  RF_CUDA(transpose(vw.d(), kk, kk, kk, tmp.d(), kk, st));  // Vw^T
  RF_TRY(cm.alloc(sizeof(double) * kk * kk, st));
  DBuf tmp3;
  RF_TRY(tmp3.alloc(sizeof(double) * kk * kk, st));
  RF_TRY(gemm(c, false, kk, kk, kk, vp.d(), kk, tmp2.d(), kk, tmp3.d(), kk));
  RF_TRY(gemm(c, false, kk, kk, kk, tmp3.d(), kk, tmp.d(), kk, cm.d(), kk));
  // svd(C) and the lift
  RF_TRY(cu.alloc(sizeof(double) * kk * kk, st));
  RF_TRY(cv.alloc(sizeof(double) * kk * kk, st));
  RF_TRY(svd_tall_dev(c, cm.d(), kk, kk, kk, cu.d(), D, cv.d()));
  RF_TRY(gemm(c, false, m, kk, kk, uc.d(), m, cu.d(), kk, U, ldu, nullptr, "lift"));
  RF_TRY(gemm(c, false, n, kk, kk, ur.d(), n, cv.d(), kk, V, n, nullptr, "lift"));
  *rank_out = kk;
  return {};
}

// Dual sketch of the single pass (lowrank.cpp:170-176) for a resident column
// block A(:, c0:c0+b) (m x b, ld lda): Yc += A_blk Gc(c0:c0+b, :), Yr(c0:c0+b, :)
// = A_blk^T Gr. Both products run on the block while it is in HBM; the block
// is consumed from the stream exactly once.
Status dual_sketch_block(rfgpu_ctx* c, const double* Ablk, int64_t m, int64_t b, int64_t lda, int64_t c0, int64_t n,
                         const double* Gc, const double* Gr, int64_t ldgr, int64_t ell, double* Yc, double* Yr,
                         double* scratch, bool first) {
  cudaStream_t st = c->stream;
  RF_TRY(gemm(c, false, m, ell, b, Ablk, lda, Gc + c0, n, first ? Yc : scratch, m, nullptr, "sketch_nn"));
  if (!first) {
    add_inplace_kernel<<<grid1d(m * ell), 256, 0, st>>>(Yc, scratch, m * ell);
    count_launch();
    RF_CUDA(cudaGetLastError());
  }
  RF_TRY(gemm(c, true, b, ell, m, Ablk, lda, Gr, ldgr, Yr + c0, n, nullptr, "sketch_tn"));
  return {};
}

// ---- host gaussian (randfact::gaussian) ----------------------------------------------
inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

inline uint64_t fnv1a(const char* s) {
  uint64_t h = 0xCBF29CE484222325ULL;
  for (const unsigned char* p = reinterpret_cast<const unsigned char*>(s); *p; ++p) {
    h ^= *p;
    h *= 0x100000001B3ULL;
  }
  return h;
}

void gaussian_span(uint64_t key, int64_t e0, int64_t e1, double* out) {
  constexpr double kTwoPi = 6.283185307179586476925286766559;
  for (int64_t e = e0; e < e1; ++e) {
    const uint64_t pair = static_cast<uint64_t>(e / 2);
    const uint64_t x1 = mix64(key + 0x9E3779B97F4A7C15ULL * (2 * pair + 1)) >> 11;
    const uint64_t x2 = mix64(key + 0x9E3779B97F4A7C15ULL * (2 * pair + 2)) >> 11;
    const double u1 = (static_cast<double>(x1) + 0.5) * 0x1.0p-53;
    const double u2 = (static_cast<double>(x2) + 0.5) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    out[e - e0] = (e % 2 == 0) ? r * std::cos(kTwoPi * u2) : r * std::sin(kTwoPi * u2);
  }
}

Status ensure_device(rfgpu_ctx* c) {
  RF_CUDA(cudaSetDevice(c->device));
  return {};
}

// Global row count and this rank's row offset for a row-sharded A.
Status global_rows(rfgpu_ctx* c, rfgpu_matrix* h) {
  h->m_global = h->m;
  h->row0 = 0;
  if (c->world <= 1) return {};
  DBuf b;
  RF_TRY(b.alloc(sizeof(double) * c->world * 2, c->stream));
  std::vector<double> v(c->world * 2, 0.0);
  v[c->rank] = static_cast<double>(h->m);
  RF_CUDA(cudaMemcpyAsync(b.d(), v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, c->stream));
  RF_TRY(allreduce(c, b.d(), c->world));
  RF_CUDA(cudaMemcpyAsync(v.data(), b.d(), sizeof(double) * c->world, cudaMemcpyDeviceToHost, c->stream));
  RF_CUDA(cudaStreamSynchronize(c->stream));
  int64_t tot = 0, off = 0;
  for (int r = 0; r < c->world; ++r) {
    if (r < c->rank) off += static_cast<int64_t>(v[r]);
    tot += static_cast<int64_t>(v[r]);
  }
  h->m_global = tot;
  h->row0 = off;
  return {};
}

}  // namespace

// ============================================================ C ABI ======
extern "C" {

const char* rfgpu_last_error(void) { return t_err.c_str(); }
int rfgpu_version(void) { return 1; }

int rfgpu_gaussian_range(uint64_t seed, const char* tag, int64_t e0, int64_t count, double* out) {
  if (e0 < 0 || count < 0 || !tag) return finish(make_err(RFGPU_EPARAM, "gaussian: negative dimension"));
  const uint64_t key = mix64(seed ^ fnv1a(tag));
  const int64_t per = 1 << 16;
  const int nt = static_cast<int>(std::min<int64_t>(std::max(1u, std::thread::hardware_concurrency()),
                                                    std::max<int64_t>(1, count / per)));
  if (nt <= 1) {
    gaussian_span(key, e0, e0 + count, out);
    return RFGPU_OK;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t) {
    const int64_t a = count * t / nt, b = count * (t + 1) / nt;
    th.emplace_back(gaussian_span, key, e0 + a, e0 + b, out + a);
  }
  for (auto& x : th) x.join();
  return RFGPU_OK;
}

int rfgpu_gaussian(uint64_t seed, const char* tag, int64_t m, int64_t n, double* out) {
  if (m < 0 || n < 0) return finish(make_err(RFGPU_EPARAM, "gaussian: negative dimension"));
  return rfgpu_gaussian_range(seed, tag, 0, m * n, out);
}

int rfgpu_ctx_create(int device, rfgpu_ctx** out) { return rfgpu_ctx_create_dist(device, 0, 1, nullptr, 0, out); }

int rfgpu_nccl_unique_id(void* id, size_t id_bytes) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  std::string why;
  if (id_bytes < 128) return finish(make_err(RFGPU_EPARAM, "nccl id buffer must hold 128 bytes"));
  if (!g_nccl.load(&why)) return finish(make_err(RFGPU_ECUDA, why));
  int r = g_nccl.getUniqueId(static_cast<NcclUniqueId*>(id));
  if (r != 0) return finish(make_err(RFGPU_ECUDA, std::string("ncclGetUniqueId: ") + g_nccl.getErrorString(r)));
  return RFGPU_OK;
}

// One-GPU check of the NCCL transport the multi-rank contexts use (every gpurun box has one GPU, so the
// multi-rank tests run on host-staged sums): loads NCCL, creates a ONE-rank communicator from a fresh id with
// the same bindings rfgpu_ctx_create_dist uses, sums `count` doubles in place on the device with
// ncclAllReduce (one rank: the sum is the input) and destroys the communicator. The sum of the result is
// returned in *checksum.
int rfgpu_nccl_selftest(int device, const double* values, int64_t count, double* out) {
  if (!values || !out || count <= 0) return finish(make_err(RFGPU_EPARAM, "nccl_selftest: bad arguments"));
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  std::string why;
  if (cudaSetDevice(device) != cudaSuccess) {
    cudaGetLastError();
    return finish(make_err(RFGPU_ECUDA, "no CUDA device available (rfgpu has no CPU fallback)"));
  }
  if (!g_nccl.load(&why)) return finish(make_err(RFGPU_ECUDA, why));
  NcclUniqueId id;
  int r = g_nccl.getUniqueId(&id);
  if (r != 0) return finish(make_err(RFGPU_ECUDA, std::string("ncclGetUniqueId: ") + g_nccl.getErrorString(r)));
  void* comm = nullptr;
  r = g_nccl.commInitRank(&comm, 1, id, 0);
  if (r != 0) return finish(make_err(RFGPU_ECUDA, std::string("ncclCommInitRank: ") + g_nccl.getErrorString(r)));
  double* d = nullptr;
  cudaStream_t st = nullptr;
  Status s = [&]() -> Status {
    RF_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    RF_CUDA(cudaMalloc(&d, sizeof(double) * count));
    RF_CUDA(cudaMemcpyAsync(d, values, sizeof(double) * count, cudaMemcpyHostToDevice, st));
    const int rr = g_nccl.allReduce(d, d, static_cast<size_t>(count), kNcclDouble, kNcclSum, comm, st);
    if (rr != 0) return make_err(RFGPU_ECUDA, std::string("ncclAllReduce: ") + g_nccl.getErrorString(rr));
    RF_CUDA(cudaMemcpyAsync(out, d, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaStreamSynchronize(st));
    return {};
  }();
  if (d) cudaFree(d);
  if (st) cudaStreamDestroy(st);
  g_nccl.commDestroy(comm);
  return finish(s);
}

}  // extern "C"

namespace {

void ctx_free(rfgpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drain_profile(c);
  for (auto e : c->event_pool) cudaEventDestroy(e);
  if (c->comm) g_nccl.commDestroy(c->comm);
  if (c->h_info) cudaFreeHost(c->h_info);
  if (c->h_d) cudaFreeHost(c->h_d);
  if (c->h_i64) cudaFreeHost(c->h_i64);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  for (void* sl : c->stage_slots) cudaFreeHost(sl);
  for (cudaEvent_t e : c->stage_done) cudaEventDestroy(e);
  for (double* h : c->sp_stage_h)
    if (h) cudaFreeHost(h);
  if (c->h_spec) cudaFreeHost(c->h_spec);
  if (c->spec_flags) cudaFree(c->spec_flags);
  if (c->copy_stream) {
    cudaStreamSynchronize(c->copy_stream);
    cudaStreamDestroy(c->copy_stream);
  }
  if (c->a_cache) cudaFree(c->a_cache);
  if (c->stream) cudaStreamDestroy(c->stream);
  // every block of the context's pools goes back to the driver
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  if (c->pool_small) cudaMemPoolDestroy(c->pool_small);
  if (c->pool_large) cudaMemPoolDestroy(c->pool_large);
  delete c;
}

// Device checks, stream, pinned scratch and the context's two memory pools.
int ctx_create_common(int device, int rank, int world, rfgpu_ctx** out) {
  if (!out) return finish(make_err(RFGPU_EPARAM, "ctx_create: null output"));
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return finish(make_err(RFGPU_EPARAM, "ctx_create: bad rank/world"));
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return finish(make_err(RFGPU_ECUDA, "no CUDA device available (rfgpu has no CPU fallback)"));
  }
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return finish(make_err(RFGPU_ECUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)));
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10) {
    return finish(make_err(RFGPU_ECUDA, std::string("rfgpu is built for sm_100a (B200); device is ") + prop.name));
  }
  auto c = new rfgpu_ctx();
  c->device = device;
  c->rank = rank;
  c->world = world;
  c->num_sms = prop.multiProcessorCount;
  bool ok = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMallocHost(&c->h_info, 64) == cudaSuccess && cudaMallocHost(&c->h_d, 64) == cudaSuccess &&
            cudaMallocHost(&c->h_i64, 64) == cudaSuccess && cudaMallocHost(&c->h_spec, 64) == cudaSuccess &&
            cudaMalloc(&c->spec_flags, 64) == cudaSuccess;
  if (ok) c->spec_vals = reinterpret_cast<double*>(c->spec_flags + 4);
  // freed pool memory stays cached (stream-ordered temporaries are reused call after call)
  cudaMemPoolProps pp{};
  pp.allocType = cudaMemAllocationTypePinned;
  pp.location.type = cudaMemLocationTypeDevice;
  pp.location.id = device;
  uint64_t thr = UINT64_MAX;
  for (cudaMemPool_t* pool : {&c->pool_small, &c->pool_large}) {
    ok = ok && cudaMemPoolCreate(pool, &pp) == cudaSuccess &&
         cudaMemPoolSetAttribute(*pool, cudaMemPoolAttrReleaseThreshold, &thr) == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    ctx_free(c);
    return finish(make_err(RFGPU_ECUDA, "ctx_create: stream / pinned memory / memory pool creation failed"));
  }
  c->launch_base = launch_counter();
  *out = c;
  return RFGPU_OK;
}

}  // namespace

extern "C" {

int rfgpu_ctx_create_dist(int device, int rank, int world, const void* nccl_id, size_t id_bytes, rfgpu_ctx** out) {
  if (world > 1 && (!nccl_id || id_bytes < 128))
    return finish(make_err(RFGPU_EPARAM, "ctx_create_dist: nccl id required"));
  rfgpu_ctx* c = nullptr;
  int st = ctx_create_common(device, rank, world, &c);
  if (st != RFGPU_OK) return st;
  if (world > 1) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    std::string why;
    if (!g_nccl.load(&why)) {
      ctx_free(c);
      return finish(make_err(RFGPU_ECUDA, why));
    }
    NcclUniqueId idb;
    std::memcpy(idb.internal, nccl_id, 128);
    int r = g_nccl.commInitRank(&c->comm, world, idb, rank);
    if (r != 0) {
      c->comm = nullptr;
      ctx_free(c);
      return finish(make_err(RFGPU_ECUDA, std::string("ncclCommInitRank: ") + g_nccl.getErrorString(r)));
    }
  }
  *out = c;
  return RFGPU_OK;
}

int rfgpu_ctx_create_hostsum(int device, int rank, int world, rfgpu_host_sum_fn sum, void* user, rfgpu_ctx** out) {
  if (world > 1 && !sum) return finish(make_err(RFGPU_EPARAM, "ctx_create_hostsum: sum callback required"));
  rfgpu_ctx* c = nullptr;
  int st = ctx_create_common(device, rank, world, &c);
  if (st != RFGPU_OK) return st;
  c->host_sum = sum;
  c->host_user = user;
  *out = c;
  return RFGPU_OK;
}

int rfgpu_ctx_destroy(rfgpu_ctx* c) {
  ctx_free(c);
  return RFGPU_OK;
}

int rfgpu_ctx_release_memory(rfgpu_ctx* c) {
  if (!c) return finish(make_err(RFGPU_EPARAM, "ctx_release_memory: null context"));
  CtxCall lk(c);
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
  if (c->a_cache) cudaFree(c->a_cache);
  c->a_cache = nullptr;
  c->a_cache_bytes = 0;
  for (double*& h : c->sp_stage_h) {  // pinned host stages too
    if (h) cudaFreeHost(h);
    h = nullptr;
  }
  c->sp_stage_bytes = 0;
  for (auto& g : c->graphs) cudaGraphExecDestroy(g.exec);
  c->graphs.clear();
  c->graph_seen.clear();
  cudaDeviceGraphMemTrim(c->device);
  for (cudaMemPool_t pool : {c->pool_small, c->pool_large})
    if (pool) cudaMemPoolTrimTo(pool, 0);
  return RFGPU_OK;
}

int64_t rfgpu_ctx_pool_bytes(rfgpu_ctx* c) {
  if (!c) return -1;
  uint64_t tot = 0;
  for (cudaMemPool_t pool : {c->pool_small, c->pool_large}) {
    uint64_t v = 0;
    if (pool && cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &v) == cudaSuccess) tot += v;
  }
  return static_cast<int64_t>(tot + c->a_cache_bytes);
}

int rfgpu_ctx_rank(const rfgpu_ctx* c) { return c ? c->rank : -1; }
int rfgpu_ctx_world(const rfgpu_ctx* c) { return c ? c->world : -1; }
void* rfgpu_ctx_stream(rfgpu_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int rfgpu_ctx_synchronize(rfgpu_ctx* c) {
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return finish(make_err(RFGPU_ECUDA, cudaGetErrorString(e)));
  return RFGPU_OK;
}

int rfgpu_profile_enable(rfgpu_ctx* c, int on) {
  CtxCall lk(c);
  c->profile = on != 0;
  return RFGPU_OK;
}

int rfgpu_profile_reset(rfgpu_ctx* c) {
  CtxCall lk(c);
  drain_profile(c);
  c->prof.clear();
  c->launch_base = launch_counter();
  return RFGPU_OK;
}

int rfgpu_profile_read(rfgpu_ctx* c, const char* name, int64_t* launches, double* total_ms) {
  CtxCall lk(c);
  drain_profile(c);
  auto it = c->prof.find(name);
  *launches = it == c->prof.end() ? 0 : it->second.first;
  *total_ms = it == c->prof.end() ? 0.0 : it->second.second;
  return RFGPU_OK;
}

int64_t rfgpu_launch_count(rfgpu_ctx* c) { return launch_counter() - c->launch_base; }

static int matrix_make(rfgpu_ctx* c, const void* host, const void* dev, bool f32, int64_t m, int64_t n, int64_t lda,
                       rfgpu_matrix** out) {
  if (!c || !out) return finish(make_err(RFGPU_EPARAM, "matrix: null argument"));
  if (m < 0 || n < 0) return finish(make_err(RFGPU_EPARAM, "DenseMatrix: negative dimension"));
  if (lda < std::max<int64_t>(1, m)) return finish(make_err(RFGPU_EPARAM, "matrix: lda < m"));
  CtxCall lk(c);
  cudaSetDevice(c->device);
  auto h = std::make_unique<rfgpu_matrix>();
  h->ctx = c;
  h->f32 = f32;
  h->m = m;
  h->n = n;
  const size_t es = f32 ? sizeof(float) : sizeof(double);
  if (dev) {
    h->dev = const_cast<void*>(dev);
    h->lda = lda;
  } else {
    h->lda = f32 ? ((m + 3) / 4) * 4 : even(std::max<int64_t>(1, m));
    const size_t bytes = es * static_cast<size_t>(h->lda) * std::max<int64_t>(1, n);
    if (cudaMalloc(&h->dev, bytes) != cudaSuccess) {
      cudaGetLastError();
      return finish(make_err(RFGPU_ENOMEM, "matrix upload: device allocation failed"));
    }
    h->owned = true;
    if (m > 0 && n > 0) {
      cudaError_t e = cudaMemcpy2DAsync(h->dev, es * h->lda, host, es * lda, es * m, n, cudaMemcpyHostToDevice, c->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
      if (e != cudaSuccess) {
        cudaFree(h->dev);
        return finish(make_err(RFGPU_ECUDA, std::string("matrix upload: ") + cudaGetErrorString(e)));
      }
    }
  }
  Status s = global_rows(c, h.get());
  if (!s.ok()) return finish(s);
  *out = h.release();
  return RFGPU_OK;
}

int rfgpu_matrix_upload(rfgpu_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda, rfgpu_matrix** out) {
  return matrix_make(c, a, nullptr, false, m, n, lda, out);
}
int rfgpu_matrix_wrap_device(rfgpu_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda, rfgpu_matrix** out) {
  return matrix_make(c, nullptr, a, false, m, n, lda, out);
}
int rfgpu_matrix_upload_f32(rfgpu_ctx* c, const float* a, int64_t m, int64_t n, int64_t lda, rfgpu_matrix** out) {
  return matrix_make(c, a, nullptr, true, m, n, lda, out);
}
int rfgpu_matrix_wrap_device_f32(rfgpu_ctx* c, const float* a, int64_t m, int64_t n, int64_t lda,
                                 rfgpu_matrix** out) {
  return matrix_make(c, nullptr, a, true, m, n, lda, out);
}

int rfgpu_matrix_free(rfgpu_matrix* h) {
  if (!h) return RFGPU_OK;
  if (h->owned) {
    cudaSetDevice(h->ctx->device);
    cudaStreamSynchronize(h->ctx->stream);
    cudaFree(h->dev);
  }
  delete h;
  return RFGPU_OK;
}

int rfgpu_matrix_shape(const rfgpu_matrix* h, int64_t* m_local, int64_t* n, int64_t* m_global, int64_t* row0) {
  if (!h) return finish(make_err(RFGPU_EPARAM, "matrix_shape: null handle"));
  if (m_local) *m_local = h->m;
  if (n) *n = h->n;
  if (m_global) *m_global = h->m_global;
  if (row0) *row0 = h->row0;
  return RFGPU_OK;
}

static Status copy_out(rfgpu_ctx* c, double* host, int64_t ldh, const double* dev, int64_t ldd, int64_t rows,
                       int64_t cols) {
  if (!host || rows <= 0 || cols <= 0) return {};
  RF_CUDA(cudaMemcpy2DAsync(host, sizeof(double) * ldh, dev, sizeof(double) * ldd, sizeof(double) * rows, cols,
                            cudaMemcpyDeviceToHost, c->stream));
  return {};
}

int rfgpu_multiply(rfgpu_ctx* c, const rfgpu_matrix* a, int trans, const double* x, int64_t ncols, double* out) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "multiply: bad handle"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    RF_TRY(ensure_device(c));
    cudaStream_t st = c->stream;
    const int64_t m = a->m, n = a->n;
    const int64_t xr = trans ? m : n, cr = trans ? n : m;
    DBuf xd, cd;
    RF_TRY(xd.alloc(sizeof(double) * std::max<int64_t>(1, xr * ncols), st));
    RF_TRY(cd.alloc(sizeof(double) * std::max<int64_t>(1, cr * ncols), st));
    if (xr * ncols > 0) RF_CUDA(cudaMemcpyAsync(xd.d(), x, sizeof(double) * xr * ncols, cudaMemcpyHostToDevice, st));
    OzPasses oz;
    RF_TRY(oz.init(c, a, ncols));
    if (oz.on && ncols > 0) {
      // the same INT8-tensor-core path the range finder takes at this size
      DBuf ssq;
      RF_TRY(ssq.alloc(sizeof(double) * ozaki_ssq_slots(m, n), st));
      RF_TRY(oz.prepare(c, a, ssq.d()));
      if (trans)
        RF_TRY(pass_tn_raw(c, a, xd.d(), std::max<int64_t>(1, xr), ncols, cd.d(), &oz));
      else
        RF_TRY(pass_nn(c, a, xd.d(), ncols, cd.d(), std::max<int64_t>(1, cr), &oz));
    } else {
      RF_TRY(gemm(c, trans != 0, cr, ncols, trans ? m : n, static_cast<const double*>(a->dev), a->lda, xd.d(),
                  std::max<int64_t>(1, xr), cd.d(), std::max<int64_t>(1, cr)));
    }
    if (trans) RF_TRY(allreduce(c, cd.d(), cr * ncols));
    RF_TRY(copy_out(c, out, std::max<int64_t>(1, cr), cd.d(), std::max<int64_t>(1, cr), cr, ncols));
    RF_CUDA(cudaStreamSynchronize(st));
    return {};
  }();
  return finish(s);
}

int rfgpu_range_finder(rfgpu_ctx* c, const rfgpu_matrix* a, const double* g, int64_t ell, int64_t q, int reorth,
                       double* Qh, double* Bh, double* resid, int64_t* ell_out) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "range_finder: bad handle"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    if (q < 0) return make_err(RFGPU_EPARAM, "power_range: q must be non-negative");
    if (ell < 1 || ell > std::min(a->m_global, a->n))
      return make_err(RFGPU_EPARAM, "power_range: k + p exceeds min(m, n)");
    if (ell > 736) return make_err(RFGPU_EPARAM, "power_range: k + p above 736 is not supported on the device");
    RF_TRY(ensure_device(c));
    cudaStream_t st = c->stream;
    const int64_t m = a->m, n = a->n, ldq = even(m);
    DBuf gd, Q, Qx, R2i, Bt, Bd;
    RF_TRY(gd.alloc(sizeof(double) * n * ell, st));
    RF_TRY(Q.alloc(sizeof(double) * std::max<int64_t>(1, ldq * ell), st));
    RF_TRY(Qx.alloc(sizeof(double) * std::max<int64_t>(1, ldq * ell), st));
    RF_TRY(R2i.alloc(sizeof(double) * ell * ell, st));
    RF_TRY(Bt.alloc(sizeof(double) * n * ell, st));
    RF_TRY(Bd.alloc(sizeof(double) * n * ell, st));
    RF_CUDA(cudaMemcpyAsync(gd.d(), g, sizeof(double) * n * ell, cudaMemcpyHostToDevice, st));
    RangeOut ro;
    double res = 0.0;
    RF_TRY(with_speculation(c, call_key(1, a, 0, ell, q, reorth), [&]() -> Status {
      RF_TRY(range_core(c, a, gd.d(), ell, q, reorth != 0, Q.d(), ldq, R2i.d(), Bt.d(), &ro));
      RF_TRY(frob_residual_dev(c, ro.a_frob2, Bt.d(), n * ro.basis.r, &res));
      if (c->spec) RF_TRY(spec_finish(c, &res));
      return {};
    }));
    const int64_t r = ro.basis.r;
    if (resid) *resid = res;
    if (ell_out) *ell_out = r;
    if (Qh) {
      RF_TRY(materialize_q(c, m, ro.basis, Qx.d(), ldq));
      RF_TRY(copy_out(c, Qh, std::max<int64_t>(1, m), Qx.d(), ldq, m, r));
    }
    if (Bh && r > 0) {
      RF_CUDA(transpose(Bt.d(), n, r, n, Bd.d(), r, st));
      RF_TRY(copy_out(c, Bh, r, Bd.d(), r, r, n));
    }
    RF_CUDA(cudaStreamSynchronize(st));
    return {};
  }();
  return finish(s);
}

int rfgpu_rsvd_device(rfgpu_ctx* c, const rfgpu_matrix* a, const double* g_dev, int64_t k, int64_t ell, int64_t q,
                      int keep_over, int reorth, double* U, double* D, double* V, int64_t* rank_out) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "rsvd: bad handle"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    RF_TRY(check_sample(a, k, ell, "power_range"));
    if (q < 0) return make_err(RFGPU_EPARAM, "power_range: q must be non-negative");
    RF_TRY(ensure_device(c));
    int64_t r = 0;
    auto body = [&] {
      return rsvd_core(c, a, g_dev, k, ell, q, keep_over != 0, reorth != 0, U, std::max<int64_t>(1, a->m), D, V, &r);
    };
    // Replayable call: from the second call with the same arguments on, the whole speculative rsvd is one CUDA
    // graph launch (no per-kernel launch latency, no host round trip until the final check).
    const std::vector<int64_t> key = {reinterpret_cast<int64_t>(a), reinterpret_cast<int64_t>(a->dev), a->m, a->n,
                                      a->lda, reinterpret_cast<int64_t>(g_dev), k, ell, q, keep_over, reorth,
                                      reinterpret_cast<int64_t>(U), reinterpret_cast<int64_t>(D),
                                      reinterpret_cast<int64_t>(V), env_signature()};
    rfgpu_ctx::GraphEntry* ge = graphs_enabled(c) ? graph_lookup(c, key) : nullptr;  // profiling: eager phases
    if (!ge && graphs_enabled(c) && !c->spec_failed.count(key) && c->graph_seen[key]++ >= 1)
      ge = graph_capture(c, key, body, &r);
    if (ge) {
      cudaError_t le = cudaGraphLaunch(ge->exec, c->stream);
      Status cs;
      if (le == cudaSuccess) {
        count_launch(static_cast<int>(ge->launches));
        cs = spec_check(c, nullptr);
        if (cs.code != kSpecRetry) {
          if (!cs.ok()) return cs;
          if (rank_out) *rank_out = ge->rank;
          return {};
        }
        c->spec_failed[key] = true;  // speculation rejected: these arguments run eagerly from now on
      } else {
        cudaGetLastError();  // e.g. no room for the graph's memory next to the eager pools: eager from now on
        cudaStreamSynchronize(c->stream);
      }
      graph_drop(c, key);
      RF_TRY(body());
    } else {
      RF_TRY(with_speculation(c, key, body));
    }
    if (rank_out) *rank_out = r;
    return {};
  }();
  return finish(s);
}

int rfgpu_rsvd(rfgpu_ctx* c, const rfgpu_matrix* a, const double* g, int64_t k, int64_t ell, int64_t q, int keep_over,
               int reorth, double* Uh, double* Dh, double* Vh, int64_t* rank_out) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "rsvd: bad handle"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    RF_TRY(check_sample(a, k, ell, "power_range"));
    if (q < 0) return make_err(RFGPU_EPARAM, "power_range: q must be non-negative");
    RF_TRY(ensure_device(c));
    cudaStream_t st = c->stream;
    const int64_t m = a->m, n = a->n, ldu = std::max<int64_t>(1, m);
    DBuf gd, U, D, V;
    RF_TRY(gd.alloc(sizeof(double) * n * ell, st));
    RF_TRY(U.alloc(sizeof(double) * ldu * ell, st));
    RF_TRY(D.alloc(sizeof(double) * ell, st));
    RF_TRY(V.alloc(sizeof(double) * n * ell, st));
    RF_CUDA(cudaMemcpyAsync(gd.d(), g, sizeof(double) * n * ell, cudaMemcpyHostToDevice, st));
    int64_t r = 0;
    RF_TRY(with_speculation(c, call_key(2, a, k, ell, q, reorth), [&] {
      return rsvd_core(c, a, gd.d(), k, ell, q, keep_over != 0, reorth != 0, U.d(), ldu, D.d(), V.d(), &r);
    }));
    RF_TRY(copy_out(c, Uh, ldu, U.d(), ldu, m, r));
    RF_TRY(copy_out(c, Dh, std::max<int64_t>(1, r), D.d(), std::max<int64_t>(1, r), r, 1));
    RF_TRY(copy_out(c, Vh, n, V.d(), n, n, r));
    RF_CUDA(cudaStreamSynchronize(st));
    if (rank_out) *rank_out = r;
    return {};
  }();
  return finish(s);
}

// rsvd straight from host memory: the value-semantics drop-in call
// (randfact::rsvd(const DenseMatrix&, ...), lowrank.hpp:15-16). A is copied
// into a device buffer cached on the context, in row panels that overlap the
// first pass; U, D, V come back to host buffers.
int rfgpu_rsvd_host(rfgpu_ctx* c, const double* a, int64_t m, int64_t n, int64_t lda, const double* g, int64_t k,
                    int64_t ell, int64_t q, int keep_over, int reorth, double* Uh, double* Dh, double* Vh,
                    int64_t* rank_out) {
  if (!c) return finish(make_err(RFGPU_EPARAM, "rsvd: null context"));
  if (m < 0 || n < 0) return finish(make_err(RFGPU_EPARAM, "DenseMatrix: negative dimension"));
  if (lda < std::max<int64_t>(1, m) || (!a && m * n > 0)) return finish(make_err(RFGPU_EPARAM, "rsvd: bad host matrix"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    RF_TRY(ensure_device(c));
    rfgpu_matrix h;
    h.ctx = c;
    h.m = m;
    h.n = n;
    h.m_global = m;
    RF_TRY(global_rows(c, &h));
    RF_TRY(check_sample(&h, k, ell, "power_range"));
    if (q < 0) return make_err(RFGPU_EPARAM, "power_range: q must be non-negative");
    if (!c->copy_stream) RF_CUDA(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    h.lda = even(std::max<int64_t>(1, m));
    const size_t bytes = sizeof(double) * static_cast<size_t>(h.lda) * std::max<int64_t>(1, n);
    if (c->a_cache_bytes < bytes) {
      RF_CUDA(cudaStreamSynchronize(c->stream));
      if (c->a_cache) cudaFree(c->a_cache);
      c->a_cache = nullptr;
      c->a_cache_bytes = 0;
      if (cudaMalloc(&c->a_cache, bytes) != cudaSuccess) {
        cudaGetLastError();
        return make_err(RFGPU_ENOMEM, "matrix upload: device allocation failed");
      }
      c->a_cache_bytes = bytes;
    }
    h.dev = c->a_cache;
    h.src = a;
    h.src_ld = lda;
    cudaStream_t st = c->stream;
    const int64_t ldu = std::max<int64_t>(1, m);
    DBuf gd, U, D, V;
    RF_TRY(gd.alloc(sizeof(double) * n * ell, st));
    RF_TRY(U.alloc(sizeof(double) * ldu * ell, st));
    RF_TRY(D.alloc(sizeof(double) * ell, st));
    RF_TRY(V.alloc(sizeof(double) * n * ell, st));
    RF_CUDA(cudaMemcpyAsync(gd.d(), g, sizeof(double) * n * ell, cudaMemcpyHostToDevice, st));
    int64_t r = 0;
    Status cs = with_speculation(c, {3, m, n, lda, k, ell, q, reorth}, [&] {
      return rsvd_core(c, &h, gd.d(), k, ell, q, keep_over != 0, reorth != 0, U.d(), ldu, D.d(), V.d(), &r, Uh, ldu);
    });
    if (!cs.ok()) {
      cudaStreamSynchronize(c->copy_stream);  // never leave a copy from or into the caller's buffers in flight
      return cs;
    }
    RF_TRY(copy_out(c, Dh, std::max<int64_t>(1, r), D.d(), std::max<int64_t>(1, r), r, 1));
    RF_TRY(copy_out(c, Vh, n, V.d(), n, n, r));
    RF_CUDA(cudaStreamSynchronize(st));
    if (rank_out) *rank_out = r;
    return {};
  }();
  return finish(s);
}

int rfgpu_row_sketch_device(rfgpu_ctx* c, const rfgpu_matrix* a, const double* g, int64_t ell, double* Y) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "row_sketch: bad handle"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    if (ell < 1) return make_err(RFGPU_EPARAM, "row_sketch: ell must be at least 1");
    RF_TRY(ensure_device(c));
    cudaStream_t st = c->stream;
    const int64_t mg = a->m_global, n = a->n;
    DBuf gt, yt;
    RF_TRY(gt.alloc(sizeof(double) * mg * ell, st));
    RF_TRY(yt.alloc(sizeof(double) * n * ell, st));
    RF_CUDA(transpose(g, ell, mg, ell, gt.d(), mg, st));  // G (ell x m) -> G^T (m x ell)
    RF_TRY(row_sketch_t(c, a, gt.d() + a->row0, mg, ell, 0, yt.d()));
    RF_CUDA(transpose(yt.d(), n, ell, n, Y, ell, st));
    RF_CUDA(cudaStreamSynchronize(st));
    return {};
  }();
  return finish(s);
}

int rfgpu_row_sketch(rfgpu_ctx* c, const rfgpu_matrix* a, const double* g, int64_t ell, double* Yh) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "row_sketch: bad handle"));
  DBuf gd, yd;
  Status s = [&]() -> Status {
    RF_TRY(ensure_device(c));
    RF_TRY(gd.alloc(sizeof(double) * a->m_global * ell, c->stream));
    RF_TRY(yd.alloc(sizeof(double) * a->n * ell, c->stream));
    RF_CUDA(cudaMemcpyAsync(gd.d(), g, sizeof(double) * a->m_global * ell, cudaMemcpyHostToDevice, c->stream));
    return {};
  }();
  if (!s.ok()) return finish(s);
  int r = rfgpu_row_sketch_device(c, a, gd.d(), ell, yd.d());
  if (r) return r;
  cudaMemcpyAsync(Yh, yd.d(), sizeof(double) * a->n * ell, cudaMemcpyDeviceToHost, c->stream);
  return rfgpu_ctx_synchronize(c);
}

int rfgpu_col_id_device(rfgpu_ctx* c, const double* Y, int64_t m, int64_t n, int64_t k, int64_t* Js, double* Z,
                        int64_t* rank_out, int* truncated) {
  if (!c) return finish(make_err(RFGPU_EPARAM, "col_id: null context"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    if (k < 1) return make_err(RFGPU_EPARAM, "id_deterministic: k must be at least 1");
    if (k > std::min(m, n)) return make_err(RFGPU_EPARAM, "id_deterministic: k exceeds min(m, n)");
    RF_TRY(ensure_device(c));
    int64_t ke = 0;
    RF_TRY(col_id_dev(c, Y, m, n, m, k, nullptr, Js, Z, &ke, truncated));
    if (rank_out) *rank_out = ke;
    return {};
  }();
  return finish(s);
}

int rfgpu_col_id(rfgpu_ctx* c, const double* Yh, int64_t m, int64_t n, int64_t k, int64_t* Js, double* Zh,
                 int64_t* rank_out, int* truncated) {
  if (!c) return finish(make_err(RFGPU_EPARAM, "col_id: null context"));
  DBuf yd, zd;
  Status s = [&]() -> Status {
    RF_TRY(ensure_device(c));
    RF_TRY(yd.alloc(sizeof(double) * std::max<int64_t>(1, m * n), c->stream));
    RF_TRY(zd.alloc(sizeof(double) * std::max<int64_t>(1, std::max<int64_t>(k, 1) * n), c->stream));
    if (m * n > 0) RF_CUDA(cudaMemcpyAsync(yd.d(), Yh, sizeof(double) * m * n, cudaMemcpyHostToDevice, c->stream));
    return {};
  }();
  if (!s.ok()) return finish(s);
  int64_t ke = 0;
  int r = rfgpu_col_id_device(c, yd.d(), m, n, k, Js, zd.d(), &ke, truncated);
  if (r) return r;
  if (rank_out) *rank_out = ke;
  if (ke > 0) cudaMemcpyAsync(Zh, zd.d(), sizeof(double) * ke * n, cudaMemcpyDeviceToHost, c->stream);
  return rfgpu_ctx_synchronize(c);
}

int rfgpu_randomized_id(rfgpu_ctx* c, const rfgpu_matrix* a, const double* g, int64_t k, int64_t ell, int64_t q,
                        int64_t* Is, double* Xh, int64_t* rank_out, int* truncated) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "randomized_id: bad handle"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    RF_TRY(check_sample(a, k, ell, "randomized_id"));
    if (q < 0) return make_err(RFGPU_EPARAM, "randomized_id: q must be non-negative");
    RF_TRY(ensure_device(c));
    cudaStream_t st = c->stream;
    // Row-sharded A (world > 1): Y stays row-local, A^T Y is summed over
    // ranks, and Y^T (ell x m_global) is assembled on every rank (zero-padded
    // columns + allreduce) for the replicated CPQR; Is are global row
    // indices, X holds this rank's rows.
    const int64_t m = a->m, mg = a->m_global, n = a->n, ldy = even(m);
    DBuf gd, y, z, yt, zt, x;
    RF_TRY(gd.alloc(sizeof(double) * n * ell, st));
    RF_TRY(y.alloc(sizeof(double) * ldy * ell, st));
    RF_TRY(z.alloc(sizeof(double) * n * ell, st));
    RF_TRY(yt.alloc(sizeof(double) * ell * mg, st));
    RF_TRY(zt.alloc(sizeof(double) * k * mg, st));
    RF_TRY(x.alloc(sizeof(double) * m * k, st));
    RF_CUDA(cudaMemcpyAsync(gd.d(), g, sizeof(double) * n * ell, cudaMemcpyHostToDevice, st));
    // tall sketch Y = (A A^T)^q A G (lowrank.cpp:316-320)
    OzPasses oz;  // the passes over A on the INT8 tensor cores at pass sizes
    RF_TRY(oz.init(c, a, ell));
    if (oz.on) {
      DBuf ssq;
      RF_TRY(ssq.alloc(sizeof(double) * ozaki_ssq_slots(m, n), st));
      RF_TRY(oz.prepare(c, a, ssq.d(), true));
    }
    RF_TRY(pass_nn(c, a, gd.d(), ell, y.d(), ldy, &oz));
    for (int64_t j = 0; j < q; ++j) {
      RF_TRY(pass_tn_raw(c, a, y.d(), ldy, ell, z.d(), &oz));
      RF_TRY(allreduce(c, z.d(), n * ell));
      RF_TRY(pass_nn(c, a, z.d(), ell, y.d(), ldy, &oz));
    }
    if (c->world > 1) RF_CUDA(cudaMemsetAsync(yt.d(), 0, sizeof(double) * ell * mg, st));
    RF_CUDA(transpose(y.d(), m, ell, ldy, yt.d() + a->row0 * ell, ell, st));  // Y^T (ell x m), this rank's columns
    RF_TRY(allreduce(c, yt.d(), ell * mg));
    int64_t ke = 0;
    RF_TRY(col_id_dev(c, yt.d(), ell, mg, ell, k, nullptr, Is, zt.d(), &ke, truncated));
    if (ke > 0) {
      RF_CUDA(transpose(zt.d() + a->row0 * ke, ke, m, ke, x.d(), m, st));  // X = Z^T, this rank's rows
      RF_CUDA(cudaMemcpyAsync(Xh, x.d(), sizeof(double) * m * ke, cudaMemcpyDeviceToHost, st));
    }
    RF_CUDA(cudaStreamSynchronize(st));
    if (rank_out) *rank_out = ke;
    return {};
  }();
  return finish(s);
}

int rfgpu_randomized_cur(rfgpu_ctx* c, const rfgpu_matrix* a, const double* g, int64_t k, int64_t ell, int64_t q,
                         int64_t* Js, int64_t* Is, double* Uh, double* cond_c, double* cond_r, int* warning,
                         int64_t* kc_out, int64_t* kr_out) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "randomized_cur: bad handle"));
  CtxCall lk(c);
  Status s = [&]() -> Status {
    RF_TRY(check_sample(a, k, ell, "randomized_cur"));
    if (q < 0) return make_err(RFGPU_EPARAM, "randomized_cur: q must be non-negative");
    RF_TRY(ensure_device(c));
    cudaStream_t st = c->stream;
    // Row-sharded A (world > 1): the wide sketch is summed over ranks inside
    // row_sketch_t; C = A(:, Js) is assembled on every rank (zero-padded
    // rows + allreduce), R = A(Is, :) likewise; every later step is
    // replicated and deterministic, so all ranks return the same Js, Is, U.
    const int64_t m = a->m, mg = a->m_global, n = a->n;
    const double* A = static_cast<const double*>(a->dev);
    DBuf gd, gt, yt, y, z, jsd, isd, cm, ct, zr, rm, rt, zt, um, sv, vm, w1, w2, xx, uc;
    RF_TRY(gd.alloc(sizeof(double) * ell * mg, st));
    RF_TRY(gt.alloc(sizeof(double) * mg * ell, st));
    RF_TRY(yt.alloc(sizeof(double) * n * ell, st));
    RF_TRY(y.alloc(sizeof(double) * ell * n, st));
    RF_TRY(z.alloc(sizeof(double) * k * n, st));
    RF_TRY(jsd.alloc(sizeof(int64_t) * k, st));
    RF_TRY(isd.alloc(sizeof(int64_t) * k, st));
    RF_CUDA(cudaMemcpyAsync(gd.d(), g, sizeof(double) * ell * mg, cudaMemcpyHostToDevice, st));
    RF_CUDA(transpose(gd.d(), ell, mg, ell, gt.d(), mg, st));
    // wide sketch Y = G A (+ q passes), lowrank.cpp:351-355
    RF_TRY(row_sketch_t(c, a, gt.d() + a->row0, mg, ell, q, yt.d()));
    RF_CUDA(transpose(yt.d(), n, ell, n, y.d(), ell, st));
    // column ID of Y -> Js, Z (:357)
    int64_t kc = 0, kr = 0;
    int trc = 0, trr = 0;
    RF_TRY(col_id_dev(c, y.d(), ell, n, ell, k, jsd.as<int64_t>(), Js, z.d(), &kc, &trc));
    *kc_out = kc;
    if (kc == 0) {
      *kr_out = 0;
      *cond_c = *cond_r = INFINITY;
      *warning = 1;
      return {};
    }
    // C = A(:, Js) (m x kc); row ID of C: col_id_core(C^T, kc) (:360-364)
    RF_TRY(cm.alloc(sizeof(double) * mg * kc, st));
    RF_TRY(ct.alloc(sizeof(double) * kc * mg, st));
    RF_TRY(zr.alloc(sizeof(double) * kc * mg, st));
    if (c->world > 1) RF_CUDA(cudaMemsetAsync(cm.d(), 0, sizeof(double) * mg * kc, st));
    gather_cols_kernel<<<grid1d(m * kc), 256, 0, st>>>(A, a->lda, m, jsd.as<int64_t>(), kc, cm.d() + a->row0, mg);
    count_launch();
    RF_CUDA(cudaGetLastError());
    RF_TRY(allreduce(c, cm.d(), mg * kc));  // all rows of C on every rank
    RF_CUDA(transpose(cm.d(), mg, kc, mg, ct.d(), kc, st));
    RF_TRY(col_id_dev(c, ct.d(), kc, mg, kc, kc, isd.as<int64_t>(), Is, zr.d(), &kr, &trr));
    *kr_out = kr;
    // R = A(Is, :) (kr x n); U = (lsq(R^T, Z^T))^T  (:365-367)
    RF_TRY(rm.alloc(sizeof(double) * kr * n, st));
    RF_TRY(rt.alloc(sizeof(double) * n * kr, st));
    RF_TRY(zt.alloc(sizeof(double) * n * kc, st));
    gather_rows_kernel<<<grid1d(n * kr), 256, 0, st>>>(A, a->lda, n, isd.as<int64_t>(), kr, rm.d(), kr, a->row0, m);
    count_launch();
    RF_CUDA(cudaGetLastError());
    RF_TRY(allreduce(c, rm.d(), kr * n));  // rows Is live on their owning ranks
    RF_CUDA(transpose(rm.d(), kr, n, kr, rt.d(), n, st));
    RF_CUDA(transpose(z.d(), kc, n, kc, zt.d(), n, st));
    RF_TRY(um.alloc(sizeof(double) * n * kr, st));
    RF_TRY(sv.alloc(sizeof(double) * std::max(kr, kc), st));
    RF_TRY(vm.alloc(sizeof(double) * kr * kr, st));
    RF_TRY(svd_tall_dev(c, rt.d(), n, kr, n, um.d(), sv.d(), vm.d()));
    std::vector<double> sr(kr);
    RF_CUDA(cudaMemcpyAsync(sr.data(), sv.d(), sizeof(double) * kr, cudaMemcpyDeviceToHost, st));
    // X = V diag(1/s) U^T Z^T  (least_squares, dense.cpp:825-837)
    RF_TRY(w1.alloc(sizeof(double) * kr * kc, st));
    RF_TRY(xx.alloc(sizeof(double) * kr * kc, st));
    RF_TRY(uc.alloc(sizeof(double) * kc * kr, st));
    RF_TRY(gemm(c, true, kr, kc, n, um.d(), n, zt.d(), n, w1.d(), kr));
    lsq_scale_kernel<<<grid1d(kr * kc), 256, 0, st>>>(w1.d(), kr, kc, sv.d());
    count_launch();
    RF_CUDA(cudaGetLastError());
    RF_TRY(gemm(c, false, kr, kc, kr, vm.d(), kr, w1.d(), kr, xx.d(), kr));
    RF_CUDA(transpose(xx.d(), kr, kc, kr, uc.d(), kc, st));  // U = X^T (kc x kr)
    RF_CUDA(cudaMemcpyAsync(Uh, uc.d(), sizeof(double) * kc * kr, cudaMemcpyDeviceToHost, st));
    // cond numbers (cond_number, lowrank.cpp:37-41): singular values of C and R
    DBuf uc2, sc, vc2;
    RF_TRY(uc2.alloc(sizeof(double) * mg * kc, st));
    RF_TRY(sc.alloc(sizeof(double) * kc, st));
    RF_TRY(vc2.alloc(sizeof(double) * kc * kc, st));
    RF_TRY(svd_tall_dev(c, cm.d(), mg, kc, mg, uc2.d(), sc.d(), vc2.d()));
    std::vector<double> scv(kc);
    RF_CUDA(cudaMemcpyAsync(scv.data(), sc.d(), sizeof(double) * kc, cudaMemcpyDeviceToHost, st));
    RF_CUDA(cudaStreamSynchronize(st));
    auto cond = [](const std::vector<double>& d) {
      if (d.empty() || d.back() <= 0.0) return static_cast<double>(INFINITY);
      return d.front() / d.back();
    };
    *cond_c = cond(scv);
    *cond_r = cond(sr);
    *warning = (*cond_c > 1e8 || *cond_r > 1e8) ? 1 : 0;
    return {};
  }();
  return finish(s);
}

int rfgpu_dual_sketch_f32(rfgpu_ctx* c, const rfgpu_matrix* a, const float* gc, const float* gr, int64_t ell,
                          float* yc, float* yr) {
  if (!c || !a || !a->f32) return finish(make_err(RFGPU_EPARAM, "dual_sketch_f32: needs an fp32 handle"));
  CtxCall lk(c);
  Status st = [&]() -> Status {
    RF_TRY(ensure_device(c));
    cudaStream_t s = c->stream;
    const int64_t m = a->m, n = a->n, ldc = even(m);
    const int64_t chunk = std::max<int64_t>(256, std::min<int64_t>(n, (int64_t(1) << 28) / std::max<int64_t>(1, m)));
    DBuf g32, gcd, grd, ycd, yrd, scratch, conv, out32;
    RF_TRY(g32.alloc(sizeof(float) * std::max(m, n) * ell, s));
    RF_TRY(gcd.alloc(sizeof(double) * n * ell, s));
    RF_TRY(grd.alloc(sizeof(double) * m * ell, s));
    RF_TRY(ycd.alloc(sizeof(double) * m * ell, s));
    RF_TRY(yrd.alloc(sizeof(double) * n * ell, s));
    RF_TRY(scratch.alloc(sizeof(double) * m * ell, s));
    RF_TRY(conv.alloc(sizeof(double) * ldc * chunk, s));
    RF_TRY(out32.alloc(sizeof(float) * std::max(m, n) * ell, s));
    RF_CUDA(cudaMemcpyAsync(g32.p, gc, sizeof(float) * n * ell, cudaMemcpyHostToDevice, s));
    f32_to_f64_kernel<<<grid1d(n * ell), 256, 0, s>>>(g32.as<float>(), n, ell, n, gcd.d(), n);
    RF_CUDA(cudaMemcpyAsync(g32.p, gr, sizeof(float) * m * ell, cudaMemcpyHostToDevice, s));
    f32_to_f64_kernel<<<grid1d(m * ell), 256, 0, s>>>(g32.as<float>(), m, ell, m, grd.d(), m);
    count_launch(2);
    bool first = true;
    for (int64_t c0 = 0; c0 < n; c0 += chunk) {
      const int64_t b = std::min(chunk, n - c0);
      f32_to_f64_kernel<<<grid1d(m * b), 256, 0, s>>>(static_cast<const float*>(a->dev) + c0 * a->lda, m, b, a->lda,
                                                      conv.d(), ldc);
      count_launch();
      RF_TRY(dual_sketch_block(c, conv.d(), m, b, ldc, c0, n, gcd.d(), grd.d(), m, ell, ycd.d(), yrd.d(), scratch.d(),
                               first));
      first = false;
    }
    f64_to_f32_kernel<<<grid1d(m * ell), 256, 0, s>>>(ycd.d(), m * ell, out32.as<float>());
    count_launch();
    RF_CUDA(cudaMemcpyAsync(yc, out32.p, sizeof(float) * m * ell, cudaMemcpyDeviceToHost, s));
    RF_CUDA(cudaStreamSynchronize(s));
    f64_to_f32_kernel<<<grid1d(n * ell), 256, 0, s>>>(yrd.d(), n * ell, out32.as<float>());
    count_launch();
    RF_CUDA(cudaMemcpyAsync(yr, out32.p, sizeof(float) * n * ell, cudaMemcpyDeviceToHost, s));
    RF_CUDA(cudaStreamSynchronize(s));
    return {};
  }();
  return finish(st);
}

}  // extern "C"

struct rfgpu_single_pass {
  rfgpu_ctx* ctx = nullptr;
  int64_t m = 0, n = 0, ell = 0, chunk = 0;
  double* gc = nullptr;  // device n x ell
  double* gr = nullptr;  // device m x ell
  double* yc = nullptr;  // device m x ell
  double* yr = nullptr;  // device n x ell
  double* scratch = nullptr;  // m x ell
  // two column-block stages: while the device sketches one, the host fills the other and the copy engine
  // moves it (pinned host stage -> device stage on the copy stream)
  double* stage_d[2] = {nullptr, nullptr};  // device m x chunk
  double* stage_h[2] = {nullptr, nullptr};  // pinned m x chunk
  cudaEvent_t copied[2] = {nullptr, nullptr};  // host stage consumed / device stage filled
  cudaEvent_t used[2] = {nullptr, nullptr};    // device stage sketched
  int cur = 0;
  int64_t staged = 0, stage_c0 = 0, next_col = 0;
  bool first = true;
};

namespace {
// Sketch the filled stage asynchronously: H2D on the copy stream, both products on the compute stream.
Status sp_flush(rfgpu_single_pass* s) {
  if (s->staged == 0) return {};
  rfgpu_ctx* c = s->ctx;
  const int b = s->cur;
  RF_CUDA(cudaStreamWaitEvent(c->copy_stream, s->used[b], 0));  // the device stage's previous block is sketched
  RF_CUDA(cudaMemcpyAsync(s->stage_d[b], s->stage_h[b], sizeof(double) * s->m * s->staged, cudaMemcpyHostToDevice,
                          c->copy_stream));
  RF_CUDA(cudaEventRecord(s->copied[b], c->copy_stream));
  RF_CUDA(cudaStreamWaitEvent(c->stream, s->copied[b], 0));
  RF_TRY(dual_sketch_block(c, s->stage_d[b], s->m, s->staged, s->m, s->stage_c0, s->n, s->gc, s->gr, s->m, s->ell,
                           s->yc, s->yr, s->scratch, s->first));
  RF_CUDA(cudaEventRecord(s->used[b], c->stream));
  s->first = false;
  s->stage_c0 += s->staged;
  s->staged = 0;
  s->cur ^= 1;
  return {};
}

void sp_free(rfgpu_single_pass* s) {
  if (!s) return;
  cudaSetDevice(s->ctx->device);
  if (s->ctx->copy_stream) cudaStreamSynchronize(s->ctx->copy_stream);
  for (double* p : {s->gc, s->gr, s->yc, s->yr, s->scratch, s->stage_d[0], s->stage_d[1]})
    if (p) cudaFreeAsync(p, s->ctx->stream);
  cudaStreamSynchronize(s->ctx->stream);  // the pinned stages (the context's) may be refilled by the next call
  for (cudaEvent_t e : {s->copied[0], s->copied[1], s->used[0], s->used[1]})
    if (e) cudaEventDestroy(e);
  delete s;
}
}  // namespace

extern "C" {

int rfgpu_single_pass_begin(rfgpu_ctx* c, int64_t m, int64_t n, int64_t ell, const double* gc, const double* gr,
                            rfgpu_single_pass** out) {
  if (!c || !out) return finish(make_err(RFGPU_EPARAM, "single_pass: null argument"));
  if (m < 1 || n < 1 || ell < 1) return finish(make_err(RFGPU_EPARAM, "single_pass_svd: bad dimensions"));
  CtxCall lk(c);
  // Row-sharded stream (world > 1): every rank streams the column blocks of
  // ITS rows (m = local rows) and passes the FULL m_global x ell Gr.
  rfgpu_matrix shape;
  shape.m = m;
  {
    cudaSetDevice(c->device);
    Status gs = global_rows(c, &shape);
    if (!gs.ok()) return finish(gs);
  }
  auto s = new rfgpu_single_pass();
  s->ctx = c;
  s->m = m;
  s->n = n;
  s->ell = ell;
  // staging chunk: ~512 MiB of columns per stage (two stages), at least 256 columns
  s->chunk = std::max<int64_t>(256, std::min<int64_t>(n, (int64_t(1) << 26) / std::max<int64_t>(1, m)));
  cudaSetDevice(c->device);
  // device buffers from the context's pools (stream-ordered); the pinned stages are kept on the context, so
  // repeated streamed calls do not page-lock 1 GiB each time
  const size_t stage_bytes = sizeof(double) * m * s->chunk;
  bool ok = c->copy_stream || cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) == cudaSuccess;
  cudaStream_t st = c->stream;
  auto dalloc = [&](double** p, size_t bytes) {
    ok = ok && ws_alloc(reinterpret_cast<void**>(p), bytes, st) == cudaSuccess;
  };
  dalloc(&s->gc, sizeof(double) * n * ell);
  dalloc(&s->gr, sizeof(double) * m * ell);
  dalloc(&s->yc, sizeof(double) * m * ell);
  dalloc(&s->yr, sizeof(double) * n * ell);
  dalloc(&s->scratch, sizeof(double) * m * ell);
  dalloc(&s->stage_d[0], stage_bytes);
  dalloc(&s->stage_d[1], stage_bytes);
  if (ok && c->sp_stage_bytes < stage_bytes) {
    cudaStreamSynchronize(st);
    for (double*& h : c->sp_stage_h) {
      if (h) cudaFreeHost(h);
      h = nullptr;
    }
    c->sp_stage_bytes = 0;
    ok = cudaMallocHost(&c->sp_stage_h[0], stage_bytes) == cudaSuccess &&
         cudaMallocHost(&c->sp_stage_h[1], stage_bytes) == cudaSuccess;
    if (ok) c->sp_stage_bytes = stage_bytes;
  }
  for (int b = 0; b < 2 && ok; ++b) {
    s->stage_h[b] = c->sp_stage_h[b];
    ok = cudaEventCreateWithFlags(&s->copied[b], cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&s->used[b], cudaEventDisableTiming) == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    sp_free(s);
    return finish(make_err(RFGPU_ENOMEM, "single_pass: device allocation failed"));
  }
  cudaError_t ce = cudaMemcpyAsync(s->gc, gc, sizeof(double) * n * ell, cudaMemcpyHostToDevice, st);
  if (ce == cudaSuccess)
    ce = cudaMemcpy2DAsync(s->gr, sizeof(double) * m, gr + shape.row0, sizeof(double) * shape.m_global,
                           sizeof(double) * m, ell, cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) {
    sp_free(s);
    return finish(make_err(RFGPU_ECUDA, std::string("single_pass: ") + cudaGetErrorString(ce)));
  }
  *out = s;
  return RFGPU_OK;
}

int rfgpu_single_pass_push(rfgpu_single_pass* s, int64_t col0, const double* blk, int64_t b) {
  if (!s) return finish(make_err(RFGPU_EPARAM, "single_pass: null state"));
  rfgpu_ctx* c = s->ctx;
  CtxCall lk(c);
  Status st = [&]() -> Status {
    if (col0 != s->next_col || b < 0 || col0 + b > s->n)
      return make_err(RFGPU_ESTREAM, "single_pass: blocks must arrive once, in column order");
    RF_TRY(ensure_device(c));
    int64_t done = 0;
    while (done < b) {
      // a host stage is refilled once its previous copy to the device is done
      if (s->staged == 0) RF_CUDA(cudaEventSynchronize(s->copied[s->cur]));
      const int64_t take = std::min(b - done, s->chunk - s->staged);
      host_copy_cols(c, s->stage_h[s->cur] + s->m * s->staged, s->m, blk + s->m * done, s->m, s->m, take,
                     /*stream_dst=*/nt_staging());
      s->staged += take;
      done += take;
      if (s->staged == s->chunk) RF_TRY(sp_flush(s));
    }
    s->next_col += b;
    return {};
  }();
  return finish(st);
}

int rfgpu_single_pass_finish(rfgpu_single_pass* s, int64_t k, double* Uh, double* Dh, double* Vh, int64_t* rank_out) {
  if (!s) return finish(make_err(RFGPU_EPARAM, "single_pass: null state"));
  rfgpu_ctx* c = s->ctx;
  Status st;
  {
    CtxCall lk(c);
    st = [&]() -> Status {
      if (s->next_col != s->n) return make_err(RFGPU_ESTREAM, "single_pass: stream not fully consumed");
      RF_TRY(ensure_device(c));
      RF_TRY(sp_flush(s));
      RF_CUDA(cudaStreamSynchronize(c->copy_stream));
      const int64_t m = s->m, n = s->n, kk = std::min(k, s->ell);
      DBuf U, D, V;
      RF_TRY(U.alloc(sizeof(double) * m * kk, c->stream));
      RF_TRY(D.alloc(sizeof(double) * kk, c->stream));
      RF_TRY(V.alloc(sizeof(double) * n * kk, c->stream));
      int64_t r = 0;
      if (c->world > 1) RF_TRY(allreduce(c, s->yr, n * s->ell));  // Yr = sum over row shards of A^T Gr
      RF_TRY(single_pass_core(c, s->yc, m, s->yr, n, s->gc, s->gr, m, k, s->ell, U.d(), m, D.d(), V.d(), &r,
                              c->world > 1));
      RF_TRY(copy_out(c, Uh, m, U.d(), m, m, r));
      RF_TRY(copy_out(c, Dh, r, D.d(), r, r, 1));
      RF_TRY(copy_out(c, Vh, n, V.d(), n, n, r));
      RF_CUDA(cudaStreamSynchronize(c->stream));
      if (rank_out) *rank_out = r;
      return {};
    }();
  }
  sp_free(s);
  return finish(st);
}

int rfgpu_single_pass_abort(rfgpu_single_pass* s) {
  sp_free(s);
  return RFGPU_OK;
}

int rfgpu_single_pass_svd_device(rfgpu_ctx* c, const rfgpu_matrix* a, const double* gc, const double* gr, int64_t k,
                                 int64_t ell, double* U, double* D, double* V, int64_t* rank_out) {
  if (!c || !a) return finish(make_err(RFGPU_EPARAM, "single_pass_svd: bad handle"));
  CtxCall lk(c);
  Status st = [&]() -> Status {
    RF_TRY(check_sample(a, k, ell, "single_pass_svd"));
    RF_TRY(ensure_device(c));
    cudaStream_t s = c->stream;
    // row-sharded A: gr is the FULL m_global x ell Gr; this rank uses its rows
    const int64_t m = a->m, n = a->n, ldgr = a->m_global;
    gr += a->row0;
    Timed tt(c, "sp_total");
    // The digit planes are allocated first and held to the end of the call,
    // as in rsvd: released before the core, their pool block was carved up by
    // the core's temporaries and the next call's 34 GB request (config 4)
    // grew the pool again (22-118 ms per call outside every kernel).
    OzPasses oz;  // both sketches on the INT8 tensor cores at pass sizes (FP32 data: 4 digits)
    DBuf yc, yr, scratch, conv;
    bool on_digits = false;
    {
      {
        Timed ta(c, "sp_alloc");
        RF_TRY(oz.init(c, a, ell));
        RF_TRY(yc.alloc(sizeof(double) * m * ell, s));
        RF_TRY(yr.alloc(sizeof(double) * n * ell, s));
        RF_TRY(scratch.alloc(sizeof(double) * m * ell, s));
      }
      if (oz.on) {
        RF_TRY(oz.prepare(c, a, nullptr, true));
        RF_TRY(pass_nn(c, a, gc, ell, yc.d(), m, &oz));                       // Yc = A Gc
        RF_TRY(pass_tn_raw(c, a, gr, ldgr, ell, yr.d(), &oz));                // Yr = A^T Gr
        on_digits = true;
      }
    }
    if (!on_digits) {
      Timed t(c, "dual_sketch");
      if (!a->f32) {
        RF_TRY(dual_sketch_block(c, static_cast<const double*>(a->dev), m, n, a->lda, 0, n, gc, gr, ldgr, ell, yc.d(), yr.d(),
                                 scratch.d(), true));
      } else {
        // fp32 matrix: widened to fp64 one column chunk at a time (each entry read once)
        const int64_t chunk = std::max<int64_t>(256, std::min<int64_t>(n, (int64_t(1) << 28) / std::max<int64_t>(1, m)));
        const int64_t ldc = even(m);
        RF_TRY(conv.alloc(sizeof(double) * ldc * chunk, s));
        bool first = true;
        for (int64_t c0 = 0; c0 < n; c0 += chunk) {
          const int64_t b = std::min(chunk, n - c0);
          f32_to_f64_kernel<<<grid1d(m * b), 256, 0, s>>>(static_cast<const float*>(a->dev) + c0 * a->lda, m, b, a->lda,
                                                          conv.d(), ldc);
          count_launch();
          RF_CUDA(cudaGetLastError());
          RF_TRY(dual_sketch_block(c, conv.d(), m, b, ldc, c0, n, gc, gr, ldgr, ell, yc.d(), yr.d(), scratch.d(), first));
          first = false;
        }
      }
    }
    RF_TRY(allreduce(c, yr.d(), n * ell));  // Yr = sum over row shards of A^T Gr
    int64_t r = 0;
    RF_TRY(single_pass_core(c, yc.d(), m, yr.d(), n, gc, gr, ldgr, k, ell, U, m, D, V, &r, c->world > 1));
    if (rank_out) *rank_out = r;
    return {};
  }();
  return finish(st);
}


// frob_residual (rangefinder.cpp:45-54): sqrt(max(0, a_frob^2 - ||B||_F^2)) with ||B||_F summed on the
// device; NumericalError when ||B||_F > a_frob (1 + 1e-8) (basis orthonormality lost upstream).
int rfgpu_frob_residual(rfgpu_ctx* c, double a_frob, const double* Bh, int64_t count, double* resid) {
  if (!c) return finish(make_err(RFGPU_EPARAM, "frob_residual: null context"));
  if (!(a_frob >= 0.0)) return finish(make_err(RFGPU_EPARAM, "frob_residual: norm must be non-negative"));
  if (count < 0 || (count > 0 && !Bh)) return finish(make_err(RFGPU_EPARAM, "frob_residual: bad matrix"));
  CtxCall lk(c);
  Status st = [&]() -> Status {
    RF_TRY(ensure_device(c));
    DBuf b;
    RF_TRY(b.alloc(sizeof(double) * std::max<int64_t>(1, count), c->stream));
    if (count > 0) RF_CUDA(cudaMemcpyAsync(b.d(), Bh, sizeof(double) * count, cudaMemcpyHostToDevice, c->stream));
    return frob_residual_dev(c, a_frob * a_frob, b.d(), count, resid);
  }();
  return finish(st);
}

// ||A - L R||_F and the CLI's spectral probes ||(A - L R) g_i|| (cli.cpp:191-206 error block) for a
// device-resident A: L R is formed 256 columns at a time on the FP64 tensor pipe and subtracted in a
// fused sum-of-squares pass, so no m x n temporary exists.
int rfgpu_lowrank_error(rfgpu_ctx* c, const rfgpu_matrix* a, const double* Lh, const double* Rh, int64_t k,
                        const double* probes, int64_t nprobes, double* frob_abs, double* probe_norms) {
  if (!c || !a || a->f32) return finish(make_err(RFGPU_EPARAM, "lowrank_error: bad handle"));
  if (k < 0 || nprobes < 0 || (nprobes > 0 && (!probes || !probe_norms)))
    return finish(make_err(RFGPU_EPARAM, "lowrank_error: bad arguments"));
  CtxCall lk(c);
  Status st = [&]() -> Status {
    RF_TRY(ensure_device(c));
    cudaStream_t s = c->stream;
    const int64_t m = a->m, n = a->n;
    const double* A = static_cast<const double*>(a->dev);
    constexpr int64_t W = 256;
    constexpr int kBlocks = 592;
    const int64_t nblk = (n + W - 1) / W;
    DBuf L, R, S, part, tot;
    RF_TRY(L.alloc(sizeof(double) * std::max<int64_t>(1, m * k), s));
    RF_TRY(R.alloc(sizeof(double) * std::max<int64_t>(1, k * n), s));
    RF_TRY(S.alloc(sizeof(double) * std::max<int64_t>(1, m * std::min(W, n)), s));
    RF_TRY(part.alloc(sizeof(double) * kBlocks * std::max<int64_t>(nblk, nprobes), s));
    RF_TRY(tot.alloc(sizeof(double) * 16, s));
    if (m * k > 0) RF_CUDA(cudaMemcpyAsync(L.d(), Lh, sizeof(double) * m * k, cudaMemcpyHostToDevice, s));
    if (k * n > 0) RF_CUDA(cudaMemcpyAsync(R.d(), Rh, sizeof(double) * k * n, cudaMemcpyHostToDevice, s));
    RF_CUDA(cudaMemsetAsync(S.d(), 0, sizeof(double) * std::max<int64_t>(1, m * std::min(W, n)), s));
    for (int64_t b = 0; b < nblk; ++b) {
      const int64_t c0 = b * W, w = std::min(W, n - c0);
      if (k > 0) RF_TRY(gemm(c, false, m, w, k, L.d(), m, R.d() + c0 * k, k, S.d(), m, nullptr, "lowrank_error"));
      diff_sumsq_kernel<<<kBlocks, 256, 0, s>>>(A + c0 * a->lda, a->lda, S.d(), m, m, w, part.d() + b * kBlocks);
      count_launch();
      RF_CUDA(cudaGetLastError());
    }
    RF_CUDA(sum_array(part.d(), kBlocks * nblk, tot.d(), s));
    RF_CUDA(cudaMemcpyAsync(c->h_d, tot.d(), sizeof(double), cudaMemcpyDeviceToHost, s));
    RF_CUDA(cudaStreamSynchronize(s));
    *frob_abs = std::sqrt(c->h_d[0]);
    if (nprobes > 0) {
      DBuf G, Y, T, Wm;
      RF_TRY(G.alloc(sizeof(double) * n * nprobes, s));
      RF_TRY(Y.alloc(sizeof(double) * m * nprobes, s));
      RF_TRY(T.alloc(sizeof(double) * std::max<int64_t>(1, k * nprobes), s));
      RF_TRY(Wm.alloc(sizeof(double) * m * nprobes, s));
      RF_CUDA(cudaMemcpyAsync(G.d(), probes, sizeof(double) * n * nprobes, cudaMemcpyHostToDevice, s));
      RF_TRY(gemm(c, false, m, nprobes, n, A, a->lda, G.d(), n, Y.d(), m));          // A g
      RF_CUDA(cudaMemsetAsync(Wm.d(), 0, sizeof(double) * m * nprobes, s));
      if (k > 0) {
        RF_TRY(gemm(c, false, k, nprobes, n, R.d(), k, G.d(), n, T.d(), k));         // R g
        RF_TRY(gemm(c, false, m, nprobes, k, L.d(), m, T.d(), k, Wm.d(), m));        // L (R g)
      }
      for (int64_t j = 0; j < nprobes; ++j) {
        diff_sumsq_kernel<<<kBlocks, 256, 0, s>>>(Y.d() + j * m, m, Wm.d() + j * m, m, m, 1, part.d() + j * kBlocks);
        count_launch();
        RF_CUDA(cudaGetLastError());
        RF_CUDA(sum_array(part.d() + j * kBlocks, kBlocks, tot.d() + j % 16, s));
        RF_CUDA(cudaMemcpyAsync(c->h_d, tot.d() + j % 16, sizeof(double), cudaMemcpyDeviceToHost, s));
        RF_CUDA(cudaStreamSynchronize(s));
        probe_norms[j] = std::sqrt(c->h_d[0]);
      }
    }
    return {};
  }();
  return finish(st);
}

int rfgpu_svd(rfgpu_ctx* c, const double* Mh, int64_t rows, int64_t cols, double* Uh, double* Sh, double* Vh,
              int* sweeps) {
  if (!c) return finish(make_err(RFGPU_EPARAM, "svd: null context"));
  CtxCall lk(c);
  Status st = [&]() -> Status {
    if (rows < cols) return make_err(RFGPU_EPARAM, "svd: device path expects rows >= cols (transpose wide input)");
    if (cols < 1 || cols > 736) return make_err(RFGPU_EPARAM, "svd: 1 <= cols <= 736 on the device");
    RF_TRY(ensure_device(c));
    cudaStream_t s = c->stream;
    DBuf M, U, S, V;
    RF_TRY(M.alloc(sizeof(double) * rows * cols, s));
    RF_TRY(U.alloc(sizeof(double) * rows * cols, s));
    RF_TRY(S.alloc(sizeof(double) * cols, s));
    RF_TRY(V.alloc(sizeof(double) * cols * cols, s));
    RF_CUDA(cudaMemcpyAsync(M.d(), Mh, sizeof(double) * rows * cols, cudaMemcpyHostToDevice, s));
    RF_TRY(svd_tall_dev(c, M.d(), rows, cols, rows, U.d(), S.d(), V.d()));
    if (sweeps) *sweeps = c->h_info[1];
    RF_TRY(copy_out(c, Uh, rows, U.d(), rows, rows, cols));
    RF_TRY(copy_out(c, Sh, cols, S.d(), cols, cols, 1));
    RF_TRY(copy_out(c, Vh, cols, V.d(), cols, cols, cols));
    RF_CUDA(cudaStreamSynchronize(s));
    return {};
  }();
  return finish(st);
}

}  // extern "C"
