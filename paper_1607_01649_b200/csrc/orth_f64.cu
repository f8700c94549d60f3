// Gram-Schmidt fallback for orth() on sketches that CholeskyQR cannot take.
//
// Reference semantics (proj/src/dense.cpp:402-431): columns are processed in
// order, each is orthogonalised twice against the kept basis and kept only if
// its residual norm exceeds drop = 1e-13 ||X||_F. The device version uses
// classical Gram-Schmidt per pass (CGS2; "twice is enough") so that each pass
// is two bandwidth-bound sweeps over the kept basis. The kept count lives in
// device memory so no host round trip happens per column; only the final
// count is read back by the orchestrator.
#include <algorithm>
#include <cooperative_groups.h>

#include "common.cuh"
#include "rfgpu_internal.h"

namespace rfgpu {

namespace {

namespace cg = cooperative_groups;

constexpr int kRowsPerChunk = 4096;

__global__ void copy_col_kernel(const double* __restrict__ x, int64_t m, double* __restrict__ v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    v[i] = x[i];
}

// partial[chunk][c] = sum over the chunk's rows of Q(i, c) * v(i), *base <= c < *r.
__global__ void dots_partial_kernel(const double* __restrict__ Q, int64_t ldq, int64_t m,
                                    const int64_t* __restrict__ r_dev, const int64_t* __restrict__ base,
                                    const double* __restrict__ v, double* __restrict__ partial, int64_t cmax) {
  const int64_t r = *r_dev, c0 = *base;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kRowsPerChunk;
  const int64_t row1 = min(m, row0 + kRowsPerChunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t c = c0 + warp; c < r; c += nw) {
    const double* q = Q + c * ldq;
    double s = 0.0;
    for (int64_t i = row0 + lane; i < row1; i += 32) s = fma(q[i], v[i], s);
    s = warp_sum(s);
    if (lane == 0) partial[blockIdx.x * cmax + c] = s;
  }
}

__global__ void dots_reduce_kernel(const double* __restrict__ partial, int chunks, int64_t cmax,
                                   const int64_t* __restrict__ r_dev, const int64_t* __restrict__ base,
                                   double* __restrict__ dots) {
  const int64_t r = *r_dev;
  for (int64_t c = *base + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < r;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < chunks; ++k) s += partial[k * cmax + c];
    dots[c] = s;
  }
}

// v(i) -= sum_c dots(c) Q(i, c), *base <= c < *r
__global__ void update_kernel(const double* __restrict__ Q, int64_t ldq, int64_t m,
                              const int64_t* __restrict__ r_dev, const int64_t* __restrict__ base,
                              const double* __restrict__ dots, double* __restrict__ v) {
  const int64_t r = *r_dev, c0 = *base;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double acc = v[i];
    for (int64_t c = c0; c < r; ++c) acc -= dots[c] * Q[c * ldq + i];
    v[i] = acc;
  }
}

// scal[0] = ||v||^2 (already reduced), scal[1] = ||X||_F^2. Decide keep/drop.
__global__ void accept_kernel(const double* __restrict__ scal, int64_t* r_dev, double* flag) {
  const double nrm = sqrt(scal[0]);
  const double drop = 1e-13 * sqrt(scal[1]);
  const bool keep = nrm > drop && nrm > 0.0;
  flag[0] = keep ? nrm : 0.0;
  flag[1] = static_cast<double>(*r_dev);
  if (keep) *r_dev += 1;
}

__global__ void store_col_kernel(const double* __restrict__ v, int64_t m, const double* __restrict__ flag,
                                 double* __restrict__ Q, int64_t ldq) {
  const double nrm = flag[0];
  if (nrm == 0.0) return;
  const int64_t col = static_cast<int64_t>(flag[1]);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < m;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    Q[col * ldq + i] = v[i] / nrm;
}

__global__ void snapshot_kernel(const int64_t* __restrict__ r_dev, int64_t* __restrict__ base) { *base = *r_dev; }

// W(:, 0:b) -= T(:, 0:b) (both ld m)
__global__ void sub_kernel(double* __restrict__ W, const double* __restrict__ T, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    W[i] -= T[i];
}

__global__ void copy_cols_kernel(const double* __restrict__ X, int64_t ldx, int64_t m, int64_t b,
                                 double* __restrict__ W) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < m * b;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / m, i = e - j * m;
    W[e] = X[j * ldx + i];
  }
}

// The in-block part of the blocked Gram-Schmidt for one block of b columns W (m x b, already orthogonalised
// against every earlier block), in ONE cooperative launch: column after column, two passes of projection
// against the block's kept columns, then the drop rule and normalisation. Each CTA owns a contiguous row
// range; the sums over rows are per-CTA partials reduced by every CTA in the same fixed order (identical
// results everywhere, no extra barrier), with a grid barrier between writing and reading partials (three
// per column) and alternating partial buffers. The kept count lives on the device (*r_dev, base *r0_dev).
__global__ void __launch_bounds__(256) gs_block_kernel(double* __restrict__ W, int64_t m, int b,
                                                       double* __restrict__ Q, int64_t ldq,
                                                       int64_t* __restrict__ r_dev, const int64_t* __restrict__ r0_dev,
                                                       const double* __restrict__ xnorm2, double* __restrict__ part,
                                                       int cmax) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[8][33];
  __shared__ double dots[64];
  const int G = gridDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rows_per = (m + G - 1) / G;
  const int64_t i0 = min(m, static_cast<int64_t>(blockIdx.x) * rows_per), i1 = min(m, i0 + rows_per);
  const int64_t r0 = *r0_dev;
  int64_t r = r0;
  const double drop = 1e-13 * sqrt(*xnorm2);
  int buf = 0;
  // CTA partial sums of up to 32 values at once: vals[j] for j < nv, written to part[buf][cta][j]
  auto cta_partials = [&](const double* vals, int nv) {
    for (int j = 0; j < nv; ++j) {
      double s2 = warp_sum(vals[j]);
      if (lane == 0) red[warp][j] = s2;
    }
    __syncthreads();
    if (tid < nv) {
      double s2 = 0.0;
      for (int w = 0; w < 8; ++w) s2 += red[w][tid];
      part[(static_cast<int64_t>(buf) * G + blockIdx.x) * cmax + tid] = s2;
    }
    __syncthreads();
  };
  auto reduce_all = [&](int nv) {  // dots[j] = sum over CTAs, fixed order (every CTA the same bits)
    for (int j = tid; j < nv; j += blockDim.x) {
      double s2 = 0.0;
      for (int g = 0; g < G; ++g) s2 += part[(static_cast<int64_t>(buf) * G + g) * cmax + j];
      dots[j] = s2;
    }
    __syncthreads();
    buf ^= 1;
  };
  for (int t = 0; t < b; ++t) {
    double* v = W + static_cast<int64_t>(t) * m;
    const int nk = static_cast<int>(r - r0);  // the block's kept columns so far (< 32)
    for (int pass = 0; pass < 2 && nk > 0; ++pass) {
      double acc[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[j] = 0.0;
      for (int64_t i = i0 + tid; i < i1; i += blockDim.x) {
        const double vi = v[i];
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nk) acc[j] = fma(Q[(r0 + j) * ldq + i], vi, acc[j]);
      }
      cta_partials(acc, nk);
      grid.sync();
      reduce_all(nk);
      for (int64_t i = i0 + tid; i < i1; i += blockDim.x) {
        double x = v[i];
        for (int j = 0; j < nk; ++j) x -= dots[j] * Q[(r0 + j) * ldq + i];
        v[i] = x;
      }
    }
    double sq[1] = {0.0};
    for (int64_t i = i0 + tid; i < i1; i += blockDim.x) sq[0] = fma(v[i], v[i], sq[0]);
    cta_partials(sq, 1);
    grid.sync();
    reduce_all(1);
    const double nrm = sqrt(dots[0]);
    if (nrm > drop && nrm > 0.0) {
      for (int64_t i = i0 + tid; i < i1; i += blockDim.x) Q[r * ldq + i] = v[i] / nrm;
      ++r;
    }
    __syncthreads();  // dots[] is rewritten by the next column
  }
  if (blockIdx.x == 0 && tid == 0) *r_dev = r;
}

inline int grid_for(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(1184, (n + 255) / 256))); }

}  // namespace

// Blocked: columns in blocks of kBlock. Each block is first orthogonalised
// twice against every column kept so far with two FP64 tensor-core GEMMs per
// pass (C = Q^T W, W -= Q C; Q is zero beyond the kept count, so the GEMMs
// need no host-side count), then column by column against the block's own
// kept columns (CGS2, drop rule). In exact arithmetic every residual equals
// the reference's (the kept columns of earlier blocks are orthogonal to the
// block's), so the same columns are kept; rounding-level differences only.
constexpr int64_t kBlock = 16;  // the in-block traffic grows with the block width (c b), the GEMMs' with c^2

GemmPlan block_plan_tn(int64_t m, int64_t c) { return plan_gemm(c, kBlock, m, 148); }
GemmPlan block_plan_nn(int64_t m, int64_t c) { return plan_gemm(m, kBlock, c, 148); }

size_t gs_orth_work_doubles(int64_t m, int64_t c) {
  const int64_t chunks = (m + kRowsPerChunk - 1) / kRowsPerChunk;
  const size_t ws = std::max(gemm_workspace_bytes(c, kBlock, block_plan_tn(m, c)),
                             gemm_workspace_bytes(m, kBlock, block_plan_nn(m, c)));
  return static_cast<size_t>(m) + chunks * c + c + 1024 + 8 + 2 * static_cast<size_t>(m) * kBlock + c * kBlock +
         (ws + 7) / 8 + 8;
}

cudaError_t gs_orth(const double* X, int64_t m, int64_t c, int64_t ldx, double* Q, int64_t ldq, int64_t* r_dev,
                    double* work, const DeviceAllreduce& ar, cudaStream_t st) {
  const int chunks = static_cast<int>((m + kRowsPerChunk - 1) / kRowsPerChunk);
  double* v = work;
  double* partial = v + m;
  double* dots = partial + static_cast<int64_t>(chunks) * c;
  double* sq_part = dots + c;      // 1024 partials for sumsq
  double* scal = sq_part + 1024;   // [0] ||v||^2, [1] ||X||^2, [2..3] flag, [4] scratch, [5] r0 (int64)
  int64_t* r0_dev = reinterpret_cast<int64_t*>(scal + 5);
  double* W = scal + 8;            // m x kBlock
  double* T = W + m * kBlock;      // m x kBlock
  double* Cb = T + m * kBlock;     // c x kBlock
  double* gws = Cb + c * kBlock;
  const GemmPlan ptn = block_plan_tn(m, c), pnn = block_plan_nn(m, c);
  const size_t gws_bytes = std::max(gemm_workspace_bytes(c, kBlock, ptn), gemm_workspace_bytes(m, kBlock, pnn));
  cudaError_t e = cudaMemsetAsync(r_dev, 0, sizeof(int64_t), st);
  if (e != cudaSuccess) return e;
  for (int64_t j = 0; j < c; ++j) {  // Q beyond the kept count must read as zero for the block GEMMs
    e = cudaMemsetAsync(Q + j * ldq, 0, sizeof(double) * m, st);
    if (e != cudaSuccess) return e;
  }
  // ||X||_F^2 (column by column to honour ldx), accumulated in fixed order
  e = cudaMemsetAsync(scal + 1, 0, sizeof(double), st);
  if (e != cudaSuccess) return e;
  if (ldx == m) {  // contiguous: one fixed-order reduction
    e = sumsq(X, m * c, sq_part, scal + 1, st);
    if (e != cudaSuccess) return e;
  } else {
    for (int64_t j = 0; j < c; ++j) {
      e = sumsq(X + j * ldx, m, sq_part, scal + 4, st);
      if (e != cudaSuccess) return e;
      e = add_scalar(scal + 1, scal + 4, st);
      if (e != cudaSuccess) return e;
    }
  }
  if (ar.fn) {
    e = ar.fn(ar.ctx, scal + 1, 1, st);
    if (e != cudaSuccess) return e;
  }
  for (int64_t j0 = 0; j0 < c; j0 += kBlock) {
    const int64_t b = std::min(kBlock, c - j0);
    copy_cols_kernel<<<grid_for(m * b), 256, 0, st>>>(X + j0 * ldx, ldx, m, b, W);
    snapshot_kernel<<<1, 1, 0, st>>>(r_dev, r0_dev);
    count_launch(2);
    if (j0 > 0) {  // twice against the columns kept by earlier blocks
      for (int pass = 0; pass < 2; ++pass) {
        e = gemm_f64(true, c, b, m, Q, ldq, W, m, Cb, c, gws, gws_bytes, nullptr, block_plan_tn(m, c), st);
        if (e != cudaSuccess) return e;
        if (ar.fn) {
          e = ar.fn(ar.ctx, Cb, c * b, st);
          if (e != cudaSuccess) return e;
        }
        e = gemm_f64(false, m, b, c, Q, ldq, Cb, c, T, m, gws, gws_bytes, nullptr, block_plan_nn(m, c), st);
        if (e != cudaSuccess) return e;
        sub_kernel<<<grid_for(m * b), 256, 0, st>>>(W, T, m * b);
        count_launch();
      }
    }
    if (!ar.fn) {  // one cooperative launch for the block's columns
      static int coop_blocks = 0;
      if (coop_blocks == 0) {
        int per_sm = 0, dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gs_block_kernel, 256, 0);
        coop_blocks = std::max(1, std::min(2, per_sm)) * sms;
      }
      int G = static_cast<int>(std::min<int64_t>(coop_blocks, std::max<int64_t>(1, (m + 1023) / 1024)));
      int bb = static_cast<int>(b), cm = 32;
      const double* xn = scal + 1;
      double* gpart = T;  // m x kBlock scratch, free here: 2 x G x 32 partials
      void* args[] = {&W, const_cast<int64_t*>(&m), &bb, &Q, &ldq, &r_dev, &r0_dev, &xn, &gpart, &cm};
      e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(gs_block_kernel), dim3(G), dim3(256), args, 0, st);
      count_launch();
      if (e != cudaSuccess) return e;
      continue;
    }
    for (int64_t t = 0; t < b; ++t) {  // then within the block, column by column (CGS2, drop rule)
      copy_col_kernel<<<grid_for(m), 256, 0, st>>>(W + t * m, m, v);
      count_launch();
      if (t > 0) {
        for (int pass = 0; pass < 2; ++pass) {
          dots_partial_kernel<<<chunks, 256, 0, st>>>(Q, ldq, m, r_dev, r0_dev, v, partial, c);
          dots_reduce_kernel<<<1, 256, 0, st>>>(partial, chunks, c, r_dev, r0_dev, dots);
          count_launch(2);
          if (ar.fn) {
            e = ar.fn(ar.ctx, dots, c, st);  // zero-padded beyond r on every rank
            if (e != cudaSuccess) return e;
          }
          update_kernel<<<grid_for(m), 256, 0, st>>>(Q, ldq, m, r_dev, r0_dev, dots, v);
          count_launch();
        }
      }
      e = sumsq(v, m, sq_part, scal, st);
      if (e != cudaSuccess) return e;
      if (ar.fn) {
        e = ar.fn(ar.ctx, scal, 1, st);
        if (e != cudaSuccess) return e;
      }
      accept_kernel<<<1, 1, 0, st>>>(scal, r_dev, scal + 2);
      store_col_kernel<<<grid_for(m), 256, 0, st>>>(v, m, scal + 2, Q, ldq);
      count_launch(2);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace rfgpu
