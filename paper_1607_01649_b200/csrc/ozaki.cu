// FP64 passes over A on the INT8 tensor cores (tcgen05.mma kind::i8, TMEM
// accumulators): Ozaki-scheme splitting of both operands into kS = 7 signed
// 8-bit digits, exact int32 digit products on the tensor cores, recombined in
// FP64 in the epilogue.
//
// Why: B200's FP64 pipe (DMMA) peaks at 37 TF/s, its INT8 tensor cores at
// 4.6 POPS (profiles/r01_i8_peak.txt). A pass over A (Y = A X, Z = A^T Q:
// proj/src/dense.cpp:102-126 on the reference's hot path,
// rangefinder.cpp:68-78, lowrank.cpp:92) needs 2 m n l flops; as 28 int8
// digit products it runs ~2x faster than DMMA can.
//
// Numerics. Row i of A is scaled by 2^-e_i (|A(i,:)| < 2^e_i) for A X, column
// j by 2^-f_j for A^T Q, every column c of the thin operand by 2^-g_c. A
// scaled value x in (-1, 1) becomes the integer X = trunc(x 2^54) (exact
// exponent arithmetic + one truncating conversion), written in balanced
// base 256: X = sum_{k<7} d_k 256^k with d_k in [-128, 127] (add 0x80 to
// every byte of X, read the bytes back minus 0x80 — no carry chain). Digit
// plane s holds d_{6-s}. The product keeps the digit pairs with s + t <= 6
// (28 of 49), grouped by g = s + t into 7 int32 TMEM accumulators (exact:
// 7 * K * 128^2 < 2^31 for K <= 16384, the split size), and sums
// sum_g 2^-(12+8g) acc_g in FP64 (one rounding per group), then scales by
// 2^(e + g_c). Per term the result is within ~8 * 2^-54 of the exact product
// relative to max|row| max|column| — FP64-class (measured below 1e-14 of the
// extended-precision product in tests/test_gpu_ozaki.py).
//
// Layouts:
//   digits of A: [kS][n_pad][m_pad] (column-major, like A). Y = A X reads them
//     M-major (TMA box 128 rows x 64 columns, 128B swizzle), A^T Q K-major
//     (box 64 rows x 128 columns, 64B swizzle): one copy serves both passes.
//   thin operand digits: [kS][l_pad][K_pad]
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "rfgpu_internal.h"

namespace rfgpu {
namespace {

// balanced base-256 digits per operand: 7 for FP64 data, 4 for FP32 (template S)
constexpr int OBM = 128;       // tile rows (TMEM lanes)
constexpr int OBN = 64;        // tile columns per accumulator group
// K bytes per pipeline stage: BK = 64 (64B-swizzled K-major rows, 2 stages
// of 86 KB for 7 digits) or 32 (32B swizzle, 5 stages of 43 KB: more bytes in
// flight per SM at the same shared-memory footprint).
constexpr int BKQ = 64;  // K bytes per block in kb_split_fixed
constexpr int64_t kSplitK = 16384;  // int32 safety: S * K * 128^2 < 2^31
// K per split of the A^T Q pass (= the column-exponent chunk). Measured: 4096 / 2048 instead of 16384 make
// the pass 17 % / 70 % slower (more partial sums to write and reduce).
int64_t tn_split_k() { return kSplitK; }
// warp 0 TMA producer, warp 1 MMA issuer, warps 2..9 epilogue (two warps per
// TMEM lane quarter, alternating 16-column chunks)
constexpr int kThreads = 320;
constexpr int kEpiWarps = kThreads / 32 - 2;
// One digit set may serve both passes when the non-zero columns' exponents
// span at most this many bits (ozaki_col_exponents): A^T Q on the row-scaled
// digits then loses at most kSharedSpread + 2 bits against column-scaled
// digits (see ozaki_tn). Used only when the second set does not fit in HBM:
// the row-major column-scaled set makes A^T Q ~20% faster than the shared
// set read K-major.
constexpr int kSharedSpread = 2;

// Per digit count S: S accumulator groups of OBN TMEM columns; as many
// 2-digit-plane... stages as fit in shared memory.
template <int S, int BK>
struct Dig {
  static constexpr size_t stage_bytes = static_cast<size_t>(S) * (OBM + OBN) * BK;
  static constexpr int fit = static_cast<int>((225 * 1024 - 2048) / stage_bytes);
  static constexpr int stages = fit > 8 ? 8 : fit;
  static constexpr int tmem_cols = S * OBN <= 256 ? 256 : 512;
  static constexpr size_t smem = stages * stage_bytes + 1024 + 256;
};

__host__ __device__ inline int64_t roundup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// ---- operand preparation ---------------------------------------------------------
// High word of |v|: ordered like |v| to within the top 20 mantissa bits, so
// its maximum carries the exponent of the maximum.
__device__ __forceinline__ uint32_t abs_hi(double v) {
  return static_cast<uint32_t>(static_cast<unsigned long long>(__double_as_longlong(fabs(v))) >> 32);
}
// Exponent e with |v| < 2^e from a high word (0 for zero).
__device__ __forceinline__ int hi_exp(uint32_t h) {
  const int E = static_cast<int>((h >> 20) & 0x7FF);
  return h == 0 ? 0 : (E == 0 ? -1021 : E - 1022);
}

// Rows [r0, r1) (r0 a multiple of 256) x one column chunk per blockIdx.y:
// row maxima (high words, atomicMax into rowhi), ||A||_F^2 partials (one per
// CTA) and per-CTA column maxima colpart[blk][j], blk = r0 / 256 +
// blockIdx.x. One thread per row, columns in sub-chunks of 256: warp maxima
// by redux, CTA maxima through shared memory. The column chunks keep the grid
// at >= 4 CTAs per SM for short (square) matrices.
template <class T>
__global__ void __launch_bounds__(256) stats_kernel(const T* __restrict__ A, int64_t r0, int64_t r1, int64_t n,
                                                    int64_t lda, int64_t n_pad, int64_t chunk,
                                                    uint32_t* __restrict__ rowhi, uint32_t* __restrict__ colpart,
                                                    double* __restrict__ ssq_part) {
  __shared__ double red[32];
  __shared__ uint32_t wmax[8][257];
  const int64_t i = r0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const bool ok = i < r1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t blk = r0 / 256 + blockIdx.x;
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * chunk, c1 = lmin(n, c0 + chunk);
  uint32_t rmax = 0;
  double s0 = 0.0, s1 = 0.0;
  for (int64_t j0 = c0; j0 < c1; j0 += 256) {
    const int jn = static_cast<int>(lmin(256, c1 - j0));
    int jj = 0;
    for (; jj + 4 <= jn; jj += 4) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = ok ? static_cast<double>(A[(j0 + jj + u) * lda + i]) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t h = abs_hi(v[u]);
        rmax = max(rmax, h);
        if (u & 1) s1 = fma(v[u], v[u], s1);
        else s0 = fma(v[u], v[u], s0);
        const uint32_t w = __reduce_max_sync(0xffffffffu, h);
        if (lane == 0) wmax[warp][jj + u] = w;
      }
    }
    for (; jj < jn; ++jj) {
      const double v = ok ? static_cast<double>(A[(j0 + jj) * lda + i]) : 0.0;
      const uint32_t h = abs_hi(v);
      rmax = max(rmax, h);
      s0 = fma(v, v, s0);
      const uint32_t w = __reduce_max_sync(0xffffffffu, h);
      if (lane == 0) wmax[warp][jj] = w;
    }
    __syncthreads();
    if (threadIdx.x < jn) {
      uint32_t mx = 0;
#pragma unroll
      for (int w = 0; w < 8; ++w) mx = max(mx, wmax[w][threadIdx.x]);
      colpart[blk * n_pad + j0 + threadIdx.x] = mx;
    }
    __syncthreads();
  }
  if (ok) {
    if (gridDim.y == 1) rowhi[i] = rmax;
    else atomicMax(&rowhi[i], rmax);
  }
  const double s = block_sum(s0 + s1, red);
  if (threadIdx.x == 0 && ssq_part) ssq_part[static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x] = s;
}

__global__ void rowexp_kernel(const uint32_t* __restrict__ rowhi, int64_t r0, int64_t r1, int* __restrict__ rowexp) {
  for (int64_t i = r0 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < r1;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    rowexp[i] = hi_exp(rowhi[i]);
}

// Column exponents of the column-scaled digit set, per row chunk (the A^T Q
// K-splits: chunk c = rows [c chunk_rows, (c+1) chunk_rows), 256-row blocks
// per chunk = bpc): colexp[c][j] from the per-block column maxima colpart.
// Chunks [c0, c1) only (the streamed upload computes them panel by panel).
// ext[0] = max and ext[1] = -min exponent over the non-zero columns of those
// chunks (both pre-set very negative), for the shared-set fallback test.
// Block (32, 32): 32 columns, the chunks strided over threadIdx.y (each warp
// reads 128 contiguous bytes per row block).
__global__ void __launch_bounds__(1024) colexp_kernel(const uint32_t* __restrict__ colpart, int64_t nblk, int64_t bpc,
                                                      int64_t c0, int64_t c1, int64_t n, int64_t n_pad,
                                                      int* __restrict__ colexp, int* __restrict__ ext) {
  __shared__ uint32_t red[32][33];
  const int64_t j = static_cast<int64_t>(blockIdx.x) * 32 + threadIdx.x;
  uint32_t gmx = 0;
  for (int64_t ch = c0 + threadIdx.y; ch < c1; ch += 32) {
    uint32_t mx = 0;
    if (j < n)
      for (int64_t b = ch * bpc; b < min(nblk, (ch + 1) * bpc); ++b) mx = max(mx, colpart[b * n_pad + j]);
    if (j < n_pad) colexp[ch * n_pad + j] = hi_exp(mx);
    gmx = max(gmx, mx);
  }
  red[threadIdx.y][threadIdx.x] = gmx;
  __syncthreads();
  if (threadIdx.y == 0) {
    for (int y = 1; y < 32; ++y) gmx = max(gmx, red[y][threadIdx.x]);
    int emax = INT_MIN, nmin = INT_MIN;
    if (gmx != 0) {
      emax = hi_exp(gmx);
      nmin = -emax;
    }
    emax = __reduce_max_sync(0xffffffffu, emax);
    nmin = __reduce_max_sync(0xffffffffu, nmin);
    if (threadIdx.x == 0 && emax != INT_MIN) {
      atomicMax(&ext[0], emax);
      atomicMax(&ext[1], nmin);
    }
  }
}

// S digits: X' = trunc(v 2^(8S-2-e)) + (0x80 in each of the S low bytes) for
// |v| < 2^e; byte k of X', minus 0x80, is the balanced base-256 digit d_k of
// trunc(v 2^(8S-2-e)) (|X| < 2^(8S-2) keeps the top byte in range). Built
// from v's bits (new exponent E + 8S-2 - e, then a truncating conversion);
// zero, subnormal and negligible (< 2^-(8S-2) relative) inputs give all-zero
// digits (X' bytes 0x80).
template <int S>
__device__ __forceinline__ uint64_t balanced(double v, int e) {
  constexpr uint64_t bias = S == 7 ? 0x0080808080808080ull : 0x0000000080808080ull;
  static_assert(S == 7 || S == 4, "digit counts: 7 (FP64) or 4 (FP32)");
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(v));
  const int E = static_cast<int>((bits >> 52) & 0x7FF);
  const int En = E + (8 * S - 2) - e;
  int64_t X = 0;
  if (E != 0 && En > 0)
    X = static_cast<int64_t>(__longlong_as_double(static_cast<long long>((bits & ~(uint64_t(0x7FF) << 52)) |
                                                                          (static_cast<uint64_t>(En) << 52))));
  return static_cast<uint64_t>(X) + bias;
}

// Digits of A for rows [r0, r1) (r0 a multiple of 4), column-major planes
// [kS][n_pad][m_pad]: rs <- A(i,j) 2^-e_i (row exponents, for A X), cs <-
// A(i,j) 2^-f_j (column exponents, for A^T Q); either may be null. Padding
// rows / columns get zero digits. One thread: 4 consecutive rows of one
// column (32 B read, 4 B per plane written), a warp 128 rows: coalesced.
// Four elements' packed digits (p[b] = digits of element b) -> per-digit words
// (word s = digit s of elements 0..3 in bytes 0..3): a 4x4 byte transpose.
__device__ __forceinline__ void transpose4(const uint32_t* p, uint32_t* w) {
  const uint32_t a = __byte_perm(p[0], p[1], 0x5140), b = __byte_perm(p[0], p[1], 0x7362);
  const uint32_t c = __byte_perm(p[2], p[3], 0x5140), d = __byte_perm(p[2], p[3], 0x7362);
  w[0] = __byte_perm(a, c, 0x5410);
  w[1] = __byte_perm(a, c, 0x7632);
  w[2] = __byte_perm(b, d, 0x5410);
  w[3] = __byte_perm(b, d, 0x7632);
}

template <class T, int S>
__global__ void __launch_bounds__(256) slice_a_kernel(const T* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                      int64_t r0, int64_t r1, const int* __restrict__ rowexp,
                                                      const int* __restrict__ colexp, int64_t chunk_rows,
                                                      int8_t* __restrict__ rs, int8_t* __restrict__ cs, int64_t m_pad,
                                                      int64_t n_pad) {
  const int64_t quads = (r1 - r0 + 3) / 4;
  const int64_t total = quads * n_pad;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = e / quads, i0 = r0 + (e - j * quads) * 4;
    uint32_t wr[S] = {}, wc[S] = {};
    if (j < n) {
      const int fj = cs ? colexp[(i0 / chunk_rows) * n_pad + j] : 0;  // 4-row quads never straddle a chunk
      double v[4];
      int er[4];
      if (i0 + 3 < m && sizeof(T) == 8 && ((j * lda + i0) & 1) == 0) {
        const double2 p0 = *reinterpret_cast<const double2*>(A + j * lda + i0);
        const double2 p1 = *reinterpret_cast<const double2*>(A + j * lda + i0 + 2);
        v[0] = p0.x, v[1] = p0.y, v[2] = p1.x, v[3] = p1.y;
        if (rs) {
          const int4 q = *reinterpret_cast<const int4*>(rowexp + i0);
          er[0] = q.x, er[1] = q.y, er[2] = q.z, er[3] = q.w;
        }
      } else {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const bool in = i0 + b < m;
          v[b] = in ? static_cast<double>(A[j * lda + i0 + b]) : 0.0;
          er[b] = (in && rs) ? rowexp[i0 + b] : 0;
        }
      }
      // words of X' per element: lo = bytes 0-3, hi = bytes 4-6 (+0)
      uint32_t hr[4], lr[4], hc[4], lc[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (rs) {
          const uint64_t x = balanced<S>(v[b], er[b]);
          lr[b] = static_cast<uint32_t>(x) ^ 0x80808080u;
          hr[b] = static_cast<uint32_t>(x >> 32) ^ 0x80808080u;
        }
        if (cs) {
          const uint64_t x = balanced<S>(v[b], fj);
          lc[b] = static_cast<uint32_t>(x) ^ 0x80808080u;
          hc[b] = static_cast<uint32_t>(x >> 32) ^ 0x80808080u;
        }
      }
      // transpose: t[k] = byte k of the four elements; plane s = byte 6 - s
      if (rs) {
        uint32_t t[8];
        transpose4(lr, t);
        transpose4(hr, t + 4);
#pragma unroll
        for (int q = 0; q < S; ++q) wr[q] = t[S - 1 - q];
      }
      if (cs) {
        uint32_t t[8];
        transpose4(lc, t);
        transpose4(hc, t + 4);
#pragma unroll
        for (int q = 0; q < S; ++q) wc[q] = t[S - 1 - q];
      }
    } else {
      // padding columns: zero digits
    }
    const int64_t off = j * m_pad + i0;
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int64_t o = static_cast<int64_t>(s) * n_pad * m_pad + off;
      if (rs) *reinterpret_cast<uint32_t*>(rs + o) = wr[s];
      if (cs) *reinterpret_cast<uint32_t*>(cs + o) = wc[s];
    }
  }
}

// Digits of A for rows [0, m_pad) with the column-scaled set ROW-major:
// cs planes [kS][m_pad][n_pad] (row i contiguous over j), so that A^T Q reads
// them M-major with a 128B swizzle exactly like A X reads rs (K-major 64-byte
// rows of A's columns were measured ~30% slower on the tensor cores). rs
// (optional) is written column-major as in slice_a_kernel.
// Tile: 128 rows x 64 columns per CTA (column tile fastest, so neighbouring
// CTAs complete each other's 128-byte row segments in L2). Warp w reads
// columns w, w + 8, ... with 4 consecutive rows per lane (1 KB per column per
// warp), writes rs directly and stages the column-scaled words (4 rows of one
// column per word) in shared memory; then each lane byte-transposes 4 words
// (4 columns x 4 rows) and writes 4 rows x 4 bytes (16 lanes: 64 B of a row).
constexpr int kSliceTRows = 128, kSliceTCols = 64;

template <class T, int S>
__global__ void __launch_bounds__(256) slice_at_kernel(const T* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                       const int* __restrict__ rowexp, const int* __restrict__ colexp_all,
                                                       int64_t chunk_rows, int64_t row_start, int8_t* __restrict__ rs,
                                                       int8_t* __restrict__ cs, int64_t m_pad, int64_t n_pad) {
  extern __shared__ uint32_t W[];  // [S][kSliceTCols][33]
  const int64_t ntc = n_pad / kSliceTCols;
  const int64_t jt = blockIdx.x % ntc, it = blockIdx.x / ntc;
  const int64_t i0 = row_start + it * kSliceTRows, j0 = jt * kSliceTCols;
  const int* __restrict__ colexp = colexp_all + (i0 / chunk_rows) * n_pad;  // a tile never straddles a chunk
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ib = i0 + 4 * lane;
  const int64_t plane = m_pad * n_pad;  // bytes per digit plane (both sets)
  int er[4] = {0, 0, 0, 0};
  if (rs)
#pragma unroll
    for (int b = 0; b < 4; ++b) er[b] = ib + b < m ? rowexp[ib + b] : 0;
  // running pointers (columns j0 + cc, cc = warp, warp + 8, ...): no 64-bit
  // index products inside the loop
  const bool vec = sizeof(T) == 8 && ib + 3 < m && (lda & 1) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  const T* colp = A + (j0 + warp) * lda + ib;
  const int64_t col_step = 8 * lda;
  int8_t* rsp = rs ? rs + (j0 + warp) * m_pad + ib : nullptr;
  // 4 rows of one column (zeros outside A); the next column's loads are
  // issued before the current one is processed (two columns in flight per warp)
  auto load4 = [&](const T* cp, int64_t j, double* v) {
    if (j < n && vec) {
      const double2 p0 = reinterpret_cast<const double2*>(cp)[0];
      const double2 p1 = reinterpret_cast<const double2*>(cp)[1];
      v[0] = p0.x, v[1] = p0.y, v[2] = p1.x, v[3] = p1.y;
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b) v[b] = (j < n && ib + b < m) ? static_cast<double>(cp[b]) : 0.0;
    }
  };
  double vn[4];
  load4(colp, j0 + warp, vn);
  for (int cc = warp; cc < kSliceTCols; cc += 8, colp += col_step) {
    const int64_t j = j0 + cc;
    double v[4] = {vn[0], vn[1], vn[2], vn[3]};
    if (cc + 8 < kSliceTCols) load4(colp + col_step, j + 8, vn);
    uint32_t wr[S], wc[S];
#pragma unroll
    for (int q = 0; q < S; ++q) wr[q] = wc[q] = 0u;
    if (j < n) {
      const int fj = colexp[j];
      uint32_t lc[4], hc[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint64_t x = balanced<S>(v[b], fj);
        lc[b] = static_cast<uint32_t>(x) ^ 0x80808080u;
        hc[b] = static_cast<uint32_t>(x >> 32) ^ 0x80808080u;
      }
      uint32_t t[8];
      transpose4(lc, t);
      transpose4(hc, t + 4);
#pragma unroll
      for (int q = 0; q < S; ++q) wc[q] = t[S - 1 - q];
      if (rs) {
        uint32_t lr[4], hr[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint64_t x = balanced<S>(v[b], er[b]);
          lr[b] = static_cast<uint32_t>(x) ^ 0x80808080u;
          hr[b] = static_cast<uint32_t>(x >> 32) ^ 0x80808080u;
        }
        transpose4(lr, t);
        transpose4(hr, t + 4);
#pragma unroll
        for (int q = 0; q < S; ++q) wr[q] = t[S - 1 - q];
      }
    }
    if (rs) {
      int8_t* d = rsp;
#pragma unroll
      for (int q = 0; q < S; ++q, d += plane) *reinterpret_cast<uint32_t*>(d) = wr[q];
      rsp += 8 * m_pad;
    }
#pragma unroll
    for (int q = 0; q < S; ++q) W[(q * kSliceTCols + cc) * 33 + lane] = wc[q];
  }
  __syncthreads();
  const int cq = threadIdx.x & 15;  // column quad: columns 4 cq .. 4 cq + 3 of the tile
  for (int rg = threadIdx.x >> 4; rg < kSliceTRows / 4; rg += 16) {
    int8_t* dst = cs + (i0 + 4 * rg) * n_pad + j0 + 4 * cq;
#pragma unroll
    for (int q = 0; q < S; ++q, dst += plane) {
      uint32_t in[4], out[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) in[c] = W[(q * kSliceTCols + 4 * cq + c) * 33 + rg];
      transpose4(in, out);  // out[u]: row 4 rg + u, columns 4 cq .. 4 cq + 3
      int8_t* d = dst;
#pragma unroll
      for (int u = 0; u < 4; ++u, d += n_pad) *reinterpret_cast<uint32_t*>(d) = out[u];
    }
  }
}

// slice_at_kernel for A whose columns start 16-byte aligned (the device
// layout): the loads go through cp.async instead of registers, so each lane
// has all 8 of its columns (8 x 32 B, FP32: 8 x 16 B) in flight at once and a CTA 64 KB
// (the register-prefetch version above keeps 2 columns per warp in flight and
// reaches ~5.2 TB/s on 94 GB). Lane l loads rows 4l..4l+3 of its warp's
// columns into the tile's shared copy, one commit group per column, and
// processes column i after waiting for group i; once the warp has read a
// column, its column-scaled words overwrite that column's 1 KB of the copy
// (word q * 33 + ((lane + cc) & 31): the skew keeps the transpose reads below
// at most 2-way bank conflicted).
template <class T, int S>
__global__ void __launch_bounds__(256) slice_at_async_kernel(const T* __restrict__ A, int64_t m, int64_t n,
                                                             int64_t lda, const int* __restrict__ rowexp,
                                                             const int* __restrict__ colexp_all, int64_t chunk_rows,
                                                             int64_t row_start, int8_t* __restrict__ rs,
                                                             int8_t* __restrict__ cs, int64_t m_pad, int64_t n_pad) {
  extern __shared__ __align__(16) uint32_t Ws[];  // [kSliceTCols][256] words: A column (1 KB), then its W words
  const int64_t ntc = n_pad / kSliceTCols;
  const int64_t jt = blockIdx.x % ntc, it = blockIdx.x / ntc;
  const int64_t i0 = row_start + it * kSliceTRows, j0 = jt * kSliceTCols;
  const int* __restrict__ colexp = colexp_all + (i0 / chunk_rows) * n_pad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ib = i0 + 4 * lane;
  const int64_t plane = m_pad * n_pad;
  // bytes of this lane's 4 rows that exist (the rest is zero-filled): 32 (FP64) or 16 (FP32)
  constexpr int kLane = 4 * static_cast<int>(sizeof(T));
  const int valid = ib >= m ? 0 : (ib + 4 <= m ? kLane : static_cast<int>(m - ib) * static_cast<int>(sizeof(T)));
  const int v0 = valid >= 16 ? 16 : valid, v1 = valid >= 16 ? valid - 16 : 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int cc = warp + 8 * i;
    const int64_t j = j0 + cc;
    const bool in = j < n;
    const T* src = in ? A + j * lda + ib : A;
    const uint32_t dst = static_cast<uint32_t>(__cvta_generic_to_shared(Ws + cc * 256 + (kLane / 4) * lane));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(in ? v0 : 0)
                 : "memory");
    if (kLane == 32)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst + 16),
                   "l"(in && v0 == 16 ? src + 16 / sizeof(T) : src), "r"(in ? v1 : 0)
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  int er[4] = {0, 0, 0, 0};
  if (rs)
#pragma unroll
    for (int b = 0; b < 4; ++b) er[b] = ib + b < m ? rowexp[ib + b] : 0;
  int8_t* rsp = rs ? rs + (j0 + warp) * m_pad + ib : nullptr;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int cc = warp + 8 * i;
    const int64_t j = j0 + cc;
    switch (i) {  // wait_group takes an immediate: groups i+1..7 may stay in flight
      case 0: asm volatile("cp.async.wait_group 7;\n" ::: "memory"); break;
      case 1: asm volatile("cp.async.wait_group 6;\n" ::: "memory"); break;
      case 2: asm volatile("cp.async.wait_group 5;\n" ::: "memory"); break;
      case 3: asm volatile("cp.async.wait_group 4;\n" ::: "memory"); break;
      case 4: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
      case 5: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
      case 6: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
      default: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
    }
    uint32_t* col = Ws + cc * 256;
    double v[4];
    if constexpr (sizeof(T) == 8) {
      const double2 p0 = reinterpret_cast<const double2*>(col + 8 * lane)[0];
      const double2 p1 = reinterpret_cast<const double2*>(col + 8 * lane)[1];
      v[0] = p0.x, v[1] = p0.y, v[2] = p1.x, v[3] = p1.y;
    } else {
      const float4 p = reinterpret_cast<const float4*>(col + 4 * lane)[0];
      v[0] = p.x, v[1] = p.y, v[2] = p.z, v[3] = p.w;
    }
    __syncwarp();  // every lane has read the column before its words overwrite it
    uint32_t wr[S], wc[S];
#pragma unroll
    for (int q = 0; q < S; ++q) wr[q] = wc[q] = 0u;
    if (j < n) {
      const int fj = colexp[j];
      uint32_t lc[4], hc[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint64_t x = balanced<S>(v[b], fj);
        lc[b] = static_cast<uint32_t>(x) ^ 0x80808080u;
        hc[b] = static_cast<uint32_t>(x >> 32) ^ 0x80808080u;
      }
      uint32_t t[8];
      transpose4(lc, t);
      transpose4(hc, t + 4);
#pragma unroll
      for (int q = 0; q < S; ++q) wc[q] = t[S - 1 - q];
      if (rs) {
        uint32_t lr[4], hr[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint64_t x = balanced<S>(v[b], er[b]);
          lr[b] = static_cast<uint32_t>(x) ^ 0x80808080u;
          hr[b] = static_cast<uint32_t>(x >> 32) ^ 0x80808080u;
        }
        transpose4(lr, t);
        transpose4(hr, t + 4);
#pragma unroll
        for (int q = 0; q < S; ++q) wr[q] = t[S - 1 - q];
      }
    }
    if (rs) {
      int8_t* d = rsp;
#pragma unroll
      for (int q = 0; q < S; ++q, d += plane) *reinterpret_cast<uint32_t*>(d) = wr[q];
      rsp += 8 * m_pad;
    }
    const int sk = (lane + cc) & 31;
#pragma unroll
    for (int q = 0; q < S; ++q) col[q * 33 + sk] = wc[q];
  }
  __syncthreads();
  const int cq = threadIdx.x & 15;
  for (int rg = threadIdx.x >> 4; rg < kSliceTRows / 4; rg += 16) {
    int8_t* dst = cs + (i0 + 4 * rg) * n_pad + j0 + 4 * cq;
#pragma unroll
    for (int q = 0; q < S; ++q, dst += plane) {
      uint32_t in[4], out[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int cc = 4 * cq + c;
        in[c] = Ws[cc * 256 + q * 33 + ((rg + cc) & 31)];
      }
      transpose4(in, out);
      int8_t* d = dst;
#pragma unroll
      for (int u = 0; u < 4; ++u, d += n_pad) *reinterpret_cast<uint32_t*>(d) = out[u];
    }
  }
}

// Thin operand R (K x N, col-major ld), optionally pre-scaled by
// 2^(rowexp[i] - shift): per-column exponent f_c of max |R(i,c) 2^(e_i - shift)|.
// Grid (N, row chunks): each CTA reduces one chunk of one column and folds its
// exponent into colexp[c] (pre-set very negative; colexp_fix_kernel maps
// all-zero columns to 0).
__device__ __forceinline__ double thin_val(const double* __restrict__ R, int64_t c, int64_t ldr, int64_t i,
                                          const int* __restrict__ rowexp, int shift) {
  const double v = R[c * ldr + i];
  return rowexp ? ldexp(v, rowexp[i] - shift) : v;
}

__global__ void __launch_bounds__(256) col_exp_kernel(const double* __restrict__ R, int64_t K, int64_t ldr,
                                                      const int* __restrict__ rowexp, int shift, int64_t chunk,
                                                      int* __restrict__ colexp) {
  __shared__ uint32_t red[8];
  const int64_t c = blockIdx.x;
  const int64_t i0 = static_cast<int64_t>(blockIdx.y) * chunk, i1 = lmin(K, i0 + chunk);
  uint32_t mx = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) mx = max(mx, abs_hi(thin_val(R, c, ldr, i, rowexp, shift)));
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) mx = max(mx, red[w]);
    if (mx) atomicMax(&colexp[c], hi_exp(mx));
  }
}

__global__ void colexp_fix_kernel(int* __restrict__ colexp, int64_t N) {
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < N;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (colexp[c] < -100000) colexp[c] = 0;
}

// Digits of R(i,c) 2^(e_i - shift) 2^-f_c (row factor only with rowexp) into
// [kS][N_pad][K_pad] (4 rows per thread).
template <int S>
__global__ void slice_r_kernel(const double* __restrict__ R, int64_t K, int64_t N, int64_t ldr,
                               const int* __restrict__ rowexp, int shift, const int* __restrict__ colexp,
                               int8_t* __restrict__ out, int64_t K_pad, int64_t N_pad) {
  const int64_t quads = K_pad / 4;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < quads * N_pad;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / quads, i0 = (e - c * quads) * 4;
    uint32_t lo[4], hi[4];
    const int fc = c < N ? colexp[c] : 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t i = i0 + b;
      const double v = (i < K && c < N) ? thin_val(R, c, ldr, i, rowexp, shift) : 0.0;
      const uint64_t x = balanced<S>(v, fc);
      lo[b] = static_cast<uint32_t>(x) ^ 0x80808080u;
      hi[b] = static_cast<uint32_t>(x >> 32) ^ 0x80808080u;
    }
    uint32_t t[8];
    transpose4(lo, t);
    transpose4(hi, t + 4);
#pragma unroll
    for (int s = 0; s < S; ++s)
      *reinterpret_cast<uint32_t*>(out + (static_cast<int64_t>(s) * N_pad + c) * K_pad + i0) = t[S - 1 - s];
  }
}

// ---- the digit GEMM -------------------------------------------------------------
struct OzParams {
  int64_t L_rows;   // rows per digit plane of L (multiple of 128)
  int64_t R_rows;   // rows per digit plane of R (multiple of 64)
  int64_t kb_per_split;  // K blocks (64 B) per split
  int64_t kb_total;
  int ntn, mtn, splits;
  int64_t row0;      // first L row handled by this launch (panelled pass 1)
  double* C;         // output (col-major, ldc) or split workspace
  int64_t ldc;
  int64_t M_real, N_real;  // valid output extent
  int64_t c_row0;    // output row offset (row of C for L row row0)
  const int* rowexp;  // optional 2^e_row output scale (indexed by L row)
  const int* colexp;  // 2^f_col output scale
  int cshift;         // extra output exponent (the thin operand's row pre-scaling shift)
  int ws_mode;        // 1: C is [split][N_real][M_real]
  int cl;             // cluster size along N tiles: the A tile is TMA-multicast to all of them
  int64_t ngroups;    // tile groups (all tiles / cl); the kernel loops over groups when the grid is smaller
  int w_big, n_big;   // the first n_big n-tiles are w_big wide, the rest w_small (multiples of 16, <= OBN):
  int w_small;        // l's padding is not multiplied, and the tiles sharing an A tile stay close in speed
  int64_t rex_stride;      // rowexp is [split][rex_stride] (per K-chunk output-row exponents; 0: one vector)
  int tma3;                // 1: one 3-D TMA copy per operand and stage (no multicast)
  int64_t kb_split_fixed;  // K blocks per split when it must match the chunks (0: even split)
};

__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// 3-D box (all digit planes of a tile in one copy): coordinates {c0, c1, plane}.
__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Same tile into every CTA of the cluster in ctaMask (same smem offsets; each
// destination's mbarrier at `bar`'s offset receives the bytes).
__device__ __forceinline__ void tma2d_mc(void* dst, const CUtensorMap* tm, uint64_t* bar, int c0, int c1,
                                         uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, "
      "{%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(tm), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}

// K-major operand tile: rows of BK K-bytes, BK-byte swizzle (8-row atoms, SBO 8 BK).
template <int BK>
__device__ __forceinline__ uint64_t umma_desc(const void* p) {
  uint64_t d = 0;
  d |= (static_cast<uint64_t>(smem_u32(p)) >> 4) & 0x3FFF;  // start address
  d |= static_cast<uint64_t>(1) << 16;                       // LBO (unused: swizzled K-major)
  d |= static_cast<uint64_t>((8 * BK) >> 4) << 32;           // SBO: 8 rows x BK bytes
  d |= static_cast<uint64_t>(1) << 46;                       // sm100 descriptor version
  d |= static_cast<uint64_t>(BK == 64 ? 4 : 6) << 61;        // SWIZZLE_64B / SWIZZLE_32B
  return d;
}

// MN-major operand tile: K rows of 128 M-bytes, 128B swizzle (atoms of 8
// K-rows x 128 B, SBO 1024 B; a single atom along M).
template <int BK>
__device__ __forceinline__ uint64_t umma_desc_mn(const void* p) {
  uint64_t d = 0;
  d |= (static_cast<uint64_t>(smem_u32(p)) >> 4) & 0x3FFF;
  d |= static_cast<uint64_t>((BK * OBM) >> 4) << 16;         // LBO: next M atom (unused, M = 128)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;               // SBO: 8 K-rows x 128 B
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;                       // SWIZZLE_128B
  return d;
}

// L_MN: the L digit planes are read M-major (column-major A digits serving
// Y = A X), else K-major (A^T Q).
//
// Persistent over tile groups (one group = the cl CTAs of a cluster, each one
// (m, n, split) tile): cluster c takes groups c, c + #clusters, ... The TMA
// producer runs straight on into the next tile's K blocks while the epilogue
// drains the previous tile, and the MMA issuer waits only for the epilogue to
// release TMEM (tfree). With one group per cluster (grid = all tiles) this is
// the plain one-tile-per-CTA kernel.
struct TileCoord {
  int64_t lrow0, ncol0, kb0;
  int nk, split;
  int w;  // tile width: p.w_big or p.w_small
};

__device__ __forceinline__ TileCoord tile_coord(const OzParams& p, int64_t tile) {
  // n-tile fastest: the CTAs sharing an L tile run together (L2 reuse)
  TileCoord t;
  const int nt = static_cast<int>(tile % p.ntn);
  const int64_t rest = tile / p.ntn;
  const int mt = static_cast<int>(rest % p.mtn);
  t.split = static_cast<int>(rest / p.mtn);
  t.lrow0 = p.row0 + static_cast<int64_t>(mt) * OBM;
  t.w = nt < p.n_big ? p.w_big : p.w_small;
  t.ncol0 = nt < p.n_big ? static_cast<int64_t>(nt) * p.w_big
                         : static_cast<int64_t>(p.n_big) * p.w_big + static_cast<int64_t>(nt - p.n_big) * p.w_small;
  t.kb0 = t.split * p.kb_per_split;
  const int64_t kb1 = min(p.kb_total, t.kb0 + p.kb_per_split);
  t.nk = static_cast<int>(kb1 - t.kb0);
  return t;
}

template <bool L_MN, int S, int BK>
__global__ void __launch_bounds__(kThreads, 1) ozaki_gemm_kernel(const __grid_constant__ CUtensorMap tmL,
                                                                  const __grid_constant__ CUtensorMap tmR,
                                                                  const __grid_constant__ CUtensorMap tmR2,
                                                                  const __grid_constant__ CUtensorMap tmL3,
                                                                  const __grid_constant__ CUtensorMap tmR3,
                                                                  const __grid_constant__ CUtensorMap tmR23,
                                                                  const OzParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int kS = S, kStages = Dig<S, BK>::stages, kTmemCols = Dig<S, BK>::tmem_cols;
  constexpr int ASZ = kS * OBM * BK, BSZ = kS * OBN * BK;
  uint8_t* sA = smem;
  uint8_t* sB = sA + kStages * ASZ;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * BSZ);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint64_t* tfree = done + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfree + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cl = p.cl;
  const int crank = static_cast<int>(blockIdx.x % cl);  // rank in the cluster (consecutive n-tiles)
  const int64_t cid = blockIdx.x / cl, ncl = gridDim.x / cl;
  const uint16_t cmask = static_cast<uint16_t>((1u << cl) - 1u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], cl);  // every CTA of the cluster must release the (shared) A stage
    }
    mbar_init(done, 1);
    mbar_init(tfree, kEpiWarps);
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  if (cl > 1) {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0 && lane == 0) {
    uint32_t it = 0;  // K blocks issued over all of this CTA's tiles
    for (int64_t g = cid; g < p.ngroups; g += ncl) {
      const TileCoord tc = tile_coord(p, g * cl + crank);
      for (int kb = 0; kb < tc.nk; ++kb, ++it) {
        const int st = static_cast<int>(it % kStages);
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>(ASZ + kS * tc.w * BK));
        const CUtensorMap* tr = tc.w == p.w_big ? &tmR : &tmR2;  // box of w rows
        const int kx = static_cast<int>((tc.kb0 + kb) * BK);
        if (p.tma3) {  // all digit planes of each operand tile in one 3-D copy (2 TMA issues per stage)
          const int lc0 = L_MN ? static_cast<int>(tc.lrow0) : kx;
          const int lc1 = L_MN ? static_cast<int>((tc.kb0 + kb) * BK) : static_cast<int>(tc.lrow0);
          tma3d(sA + st * ASZ, &tmL3, &full[st], lc0, lc1, 0);
          tma3d(sB + st * BSZ, tc.w == p.w_big ? &tmR3 : &tmR23, &full[st], kx, static_cast<int>(tc.ncol0), 0);
          continue;
        }
#pragma unroll
        for (int s = 0; s < kS; ++s) {
          // A planes round-robin over the cluster, multicast to all of it
          // K-major L: box {BK K-bytes, 128 rows} at (k, plane row); M-major L
          // (planes [kS][K_rows][M]): box {128 M-bytes, BK K-rows} at (m, plane k)
          const int lc0 = L_MN ? static_cast<int>(tc.lrow0) : kx;
          const int lc1 = L_MN ? static_cast<int>(s * p.L_rows + (tc.kb0 + kb) * BK)
                               : static_cast<int>(s * p.L_rows + tc.lrow0);
          if (cl == 1)
            tma2d(sA + st * ASZ + s * OBM * BK, &tmL, &full[st], lc0, lc1);
          else if (s % cl == crank)
            tma2d_mc(sA + st * ASZ + s * OBM * BK, &tmL, &full[st], lc0, lc1, cmask);
          tma2d(sB + st * BSZ + s * tc.w * BK, tr, &full[st], kx, static_cast<int>(s * p.R_rows + tc.ncol0));
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // For a fixed A digit s the groups g = s + t of consecutive t are
    // consecutive 64-column TMEM blocks, and the B digit planes are
    // consecutive 64-row blocks in shared memory: one MMA with N = 64 x (up to
    // 4 digits of B) covers them. 10 MMAs per 32 K-bytes instead of 28, each
    // A tile read from shared memory once per 4 B digits.
    auto idesc_n = [](int n) {
      return (2u << 4) | (1u << 7) | (1u << 10) | (L_MN ? (1u << 15) : 0u) | (static_cast<uint32_t>(n >> 3) << 17) |
             (static_cast<uint32_t>(OBM >> 4) << 24);
    };
    uint32_t it = 0, tt = 0;
    for (int64_t g = cid; g < p.ngroups; g += ncl, ++tt) {
      const TileCoord tc = tile_coord(p, g * cl + crank);
      mbar_wait(tfree, (tt & 1) ^ 1);  // the epilogue has drained the previous tile
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      for (int kb = 0; kb < tc.nk; ++kb, ++it) {
        const int st = static_cast<int>(it % kStages);
        const uint32_t ph = (it / kStages) & 1;
        mbar_wait(&full[st], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < BK / 32; ++kk) {
#pragma unroll
          for (int s = 0; s < kS; ++s) {
#pragma unroll
            for (int t0 = 0; t0 < kS - s; t0 += 4) {
              const int cnt = (kS - s - t0) < 4 ? (kS - s - t0) : 4;
              // M-major: K advances by 32 K-rows = 4 swizzle atoms
              const uint64_t da = L_MN ? umma_desc_mn<BK>(sA + st * ASZ + s * OBM * BK + kk * 32 * OBM)
                                       : umma_desc<BK>(sA + st * ASZ + s * OBM * BK + kk * 32);
              const uint64_t db = umma_desc<BK>(sB + st * BSZ + t0 * tc.w * BK + kk * 32);
              // groups s + t0 .. s + t0 + cnt - 1; every group is first written by s = 0
              const uint32_t accum = (kb == 0 && kk == 0 && s == 0) ? 0u : 1u;
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem + (s + t0) * tc.w),
                  "l"(da), "l"(db), "r"(idesc_n(tc.w * cnt)), "r"(accum));
            }
          }
        }
        if (cl == 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty[st]))
                       : "memory");
        else  // release this stage in every CTA of the cluster
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&empty[st])),
              "h"(cmask)
              : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(done))
                   : "memory");
    }
  } else if (warp >= 2) {
    const int q = warp & 3;              // TMEM lane quarter of this warp
    const int half = (warp - 2) >> 2;    // its 16-column chunks: half, half + 2, ...
    constexpr int kHalves = kEpiWarps / 4;
    uint32_t tt = 0;
    for (int64_t g = cid; g < p.ngroups; g += ncl, ++tt) {
      const TileCoord tc = tile_coord(p, g * cl + crank);
      mbar_wait(done, tt & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const int64_t lrow = tc.lrow0 + q * 32 + lane;
      const int64_t orow = p.c_row0 + (lrow - p.row0);
      const int rex = (p.rowexp && tc.nk > 0) ? p.rowexp[tc.split * p.rex_stride + lrow] : 0;
      const bool row_ok = orow < p.M_real + p.c_row0 && lrow - p.row0 < p.M_real;
      if (half * 16 >= tc.w) {  // no chunk for this warp in a narrow tile
        __syncwarp();
        if (lane == 0) mbar_arrive(tfree);
      }
      for (int c = half * 16; c < tc.w; c += 16 * kHalves) {
        uint32_t r[kS][16];
        if (tc.nk > 0) {
#pragma unroll
          for (int gg = 0; gg < kS; ++gg) {
            const uint32_t ta = tmem + (static_cast<uint32_t>(q * 32) << 16) + gg * tc.w + c;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[gg][0]), "=r"(r[gg][1]), "=r"(r[gg][2]), "=r"(r[gg][3]), "=r"(r[gg][4]), "=r"(r[gg][5]),
                  "=r"(r[gg][6]), "=r"(r[gg][7]), "=r"(r[gg][8]), "=r"(r[gg][9]), "=r"(r[gg][10]), "=r"(r[gg][11]),
                  "=r"(r[gg][12]), "=r"(r[gg][13]), "=r"(r[gg][14]), "=r"(r[gg][15])
                : "r"(ta));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        }
        if (c + 16 * kHalves >= tc.w) {  // this warp's last chunk is in registers: release its share of TMEM
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(tfree);
        }
        // sum_g acc_g 2^-(12+8g) = 2^-36 (hi + 2^-24 lo), hi = sum_{g<4} acc_g 256^(3-g) and
        // lo = sum_{g>=4} acc_g 256^(6-g) exact in int64 (|acc_g| < 2^31): two conversions, not seven
        double acc[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = 0.0;
        if (tc.nk > 0) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            int64_t hi = static_cast<int32_t>(r[0][j]);
#pragma unroll
            for (int gg = 1; gg < 4 && gg < kS; ++gg) hi = hi * 256 + static_cast<int32_t>(r[gg][j]);
            double d = static_cast<double>(hi);
            if constexpr (kS > 4) {
              int64_t lo = static_cast<int32_t>(r[4][j]);
#pragma unroll
              for (int gg = 5; gg < kS; ++gg) lo = lo * 256 + static_cast<int32_t>(r[gg][j]);
              d = fma(static_cast<double>(lo), 0x1p-24, d);
            }
            acc[j] = d;
          }
        }
        if (row_ok) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int64_t col = tc.ncol0 + c + j;
            if (col < p.N_real) {
              const double v = ldexp(acc[j], rex + p.colexp[col] + p.cshift - 36);
              if (p.ws_mode)
                p.C[(static_cast<int64_t>(tc.split) * p.N_real + col) * p.M_real + (lrow - p.row0)] = v;
              else
                p.C[col * p.ldc + orow] = v;
            }
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // no CTA may leave while cluster peers can still write into its shared memory
  if (cl > 1)
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  else
    __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

__global__ void reduce_ws_kernel(const double* __restrict__ part, int64_t M, int64_t N, int S, double* __restrict__ C,
                                 int64_t ldc) {
  const int64_t total = M * N;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t n = e / M, m = e - n * M;
    double s = 0.0;
    for (int k = 0; k < S; ++k) s += part[k * total + e];
    C[n * ldc + m] = s;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// int8 digit planes: rows x inner bytes (row-major); box {box_inner, box_rows}.
bool digit_tmap(CUtensorMap* tm, const int8_t* base, int64_t rows, int64_t inner, int box_inner, int box_rows,
                CUtensorMapSwizzle sw) {
  auto fn = tmap_encoder();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D map over the digit planes: dims {inner, rows per plane, planes}; box
// {box_inner, box_rows, planes} lands in shared memory plane after plane.
bool digit_tmap3(CUtensorMap* tm, const int8_t* base, int64_t planes, int64_t rows, int64_t inner, int box_inner,
                 int box_rows, CUtensorMapSwizzle sw) {
  auto fn = tmap_encoder();
  if (!fn) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(planes)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(inner * rows)};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_rows),
                       static_cast<cuuint32_t>(planes)};
  cuuint32_t es[3] = {1, 1, 1};
  return fn(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// multicast: share each A tile across the CTAs of its N tiles (cluster).
// Measured at config 3: it pays for the split-K A^T Q pass (31.1 vs 39.1 ms)
// and costs the NN pass (30.3 vs 25.3 ms: four CTAs in lock step through a
// 2-stage ring), so the caller chooses.
// L_mn: L planes are [kS][K_pad][L_M] (M contiguous, L_rows = K_pad rows per
// plane, L_M = M extent), else [kS][L_rows][K_pad].

template <int S, int BK>
cudaError_t launch_digit_gemm_s(const int8_t* L, int64_t L_rows, bool L_mn, int64_t L_M, const int8_t* R,
                                int64_t R_rows, int64_t K_pad, int64_t row0, int64_t rows, int64_t N_real, int splits,
                                const OzParams& base, bool multicast, cudaStream_t st) {
  constexpr int kS = S;
  constexpr size_t kSmemBytes = Dig<S, BK>::smem;
  constexpr CUtensorMapSwizzle kSwK = BK == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B;
  static std::atomic<uint64_t> cfg{0};
  if (attr_pending(cfg)) {
    for (auto fn : {ozaki_gemm_kernel<true, S, BK>, ozaki_gemm_kernel<false, S, BK>}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes));
      if (e != cudaSuccess) return e;
    }
    attr_done(cfg);
  }
  CUtensorMap tl, tr;
  const bool okl = L_mn ? digit_tmap(&tl, L, kS * L_rows, L_M, OBM, BK, CU_TENSOR_MAP_SWIZZLE_128B)
                        : digit_tmap(&tl, L, kS * L_rows, K_pad, BK, OBM, kSwK);
  if (!okl) return cudaErrorInvalidValue;
  // n-tile widths: roundup(N_real, 16) split over the ntn tiles as evenly as 16-column units allow
  // (l = 220: 64 64 48 48); RFGPU_OZAKI_NARROW=0 pads every tile to 64, =1 keeps 64 ... 64 + a narrow last
  const int ntn = static_cast<int>(R_rows / OBN);
  const int units = static_cast<int>(std::min<int64_t>(4 * ntn, std::max<int64_t>(1, (N_real + 15) / 16)));
  // (measured: padding every tile to 64 columns costs 7 %, 64-column tiles and one narrow last tile 1-2 %)
  const int q = units / ntn, r = units % ntn;
  // (measured: equal 48-column tiles for the split-K A^T Q pass, so that the CTAs sharing an A tile run at
  // one speed, cut its DRAM reads 65 -> 41 GB but not its time: 21.9 vs 22.1 ms)
  const int w_small = 16 * q > 0 ? 16 * q : 16 * (q + 1), w_big = r ? 16 * (q + 1) : 16 * q;
  const int n_big = r ? r : ntn;
  CUtensorMap tr2;
  if (!digit_tmap(&tr, R, kS * R_rows, K_pad, BK, w_big, kSwK)) return cudaErrorInvalidValue;
  tr2 = tr;
  if (w_small != w_big && !digit_tmap(&tr2, R, kS * R_rows, K_pad, BK, w_small, kSwK)) return cudaErrorInvalidValue;
  CUtensorMap tl3 = tl, tr3 = tr, tr23 = tr2;
  bool tma3 = true;  // all digit planes of a tile in one 3-D copy (2 TMA issues per stage instead of 14)
  {
    tma3 = (L_mn ? digit_tmap3(&tl3, L, kS, L_rows, L_M, OBM, BK, CU_TENSOR_MAP_SWIZZLE_128B)
                 : digit_tmap3(&tl3, L, kS, L_rows, K_pad, BK, OBM, kSwK)) &&
           digit_tmap3(&tr3, R, kS, R_rows, K_pad, BK, w_big, kSwK) &&
           (w_small == w_big || digit_tmap3(&tr23, R, kS, R_rows, K_pad, BK, w_small, kSwK));
    if (w_small == w_big) tr23 = tr3;
  }
  OzParams p = base;
  p.L_rows = L_rows;
  p.R_rows = R_rows;
  p.kb_total = K_pad / BK;
  if (base.kb_split_fixed > 0) {  // chunk-aligned splits (given in 64-byte K blocks)
    p.kb_per_split = base.kb_split_fixed * 64 / BK;
    splits = static_cast<int>((p.kb_total + p.kb_per_split - 1) / p.kb_per_split);
  } else {
    p.kb_per_split = (p.kb_total + splits - 1) / splits;
  }
  p.splits = splits;
  p.ntn = ntn;
  p.w_big = w_big;
  p.n_big = n_big;
  p.w_small = w_small;
  p.mtn = static_cast<int>((rows + OBM - 1) / OBM);
  p.row0 = row0;
  p.M_real = rows;
  p.N_real = N_real;
  const int64_t grid = static_cast<int64_t>(p.ntn) * p.mtn * splits;
  if (grid <= 0) return cudaSuccess;
  p.cl = 1;
  // multicast of the A tile over the n-tiles of a cluster: the digit Grams (short K) use it; the passes do
  // not (measured at config 3: clusters of 4 cost 25-30 %, of 2 with equal-work pairs 0-13 %)
  if (multicast)
    for (int c : {8, 7, 6, 5, 4, 3, 2})
      if (p.ntn % c == 0) {
        p.cl = c;
        break;
      }
  p.ngroups = grid / p.cl;
  p.tma3 = (tma3 && p.cl == 1) ? 1 : 0;
  cudaLaunchConfig_t cfgl{};
  cfgl.gridDim = dim3(static_cast<unsigned>(grid));
  cfgl.blockDim = dim3(kThreads);
  cfgl.dynamicSmemBytes = kSmemBytes;
  cfgl.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(p.cl);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfgl.attrs = attr;
  cfgl.numAttrs = 1;
  cudaError_t e = L_mn ? cudaLaunchKernelEx(&cfgl, ozaki_gemm_kernel<true, S, BK>, tl, tr, tr2, tl3, tr3, tr23, p)
                       : cudaLaunchKernelEx(&cfgl, ozaki_gemm_kernel<false, S, BK>, tl, tr, tr2, tl3, tr3, tr23, p);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}


// 64 K-bytes per stage, 2 stages (measured: 32-byte stages, 5 deep, with a 32B swizzle are 30 % slower)
cudaError_t launch_digit_gemm(int S, const int8_t* L, int64_t L_rows, bool L_mn, int64_t L_M, const int8_t* R,
                              int64_t R_rows, int64_t K_pad, int64_t row0, int64_t rows, int64_t N_real, int splits,
                              const OzParams& base, bool multicast, cudaStream_t st) {
  if (S == 4)
    return launch_digit_gemm_s<4, 64>(L, L_rows, L_mn, L_M, R, R_rows, K_pad, row0, rows, N_real, splits, base,
                                      multicast, st);
  return launch_digit_gemm_s<7, 64>(L, L_rows, L_mn, L_M, R, R_rows, K_pad, row0, rows, N_real, splits, base,
                                    multicast, st);
}

// Column exponents (many CTAs per column) + digits of the thin operand R
// (K x N), rows optionally pre-scaled by 2^(rowexp[i] - shift).
cudaError_t slice_thin(int S, const double* R, int64_t K, int64_t N, int64_t ldr, const int* rowexp, int shift,
                       int* colexp, int8_t* out, int64_t K_pad, int64_t N_pad, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(colexp, 0x80, sizeof(int) * N, st);  // very negative
  if (e != cudaSuccess) return e;
  const int64_t chunk = 16384;
  if (N > 0 && K > 0)
    col_exp_kernel<<<dim3(static_cast<unsigned>(N), static_cast<unsigned>((K + chunk - 1) / chunk)), 256, 0, st>>>(
        R, K, ldr, rowexp, shift, chunk, colexp);
  colexp_fix_kernel<<<static_cast<unsigned>(std::max<int64_t>(1, (N + 255) / 256)), 256, 0, st>>>(colexp, N);
  if (S == 4)
    slice_r_kernel<4><<<1184, 256, 0, st>>>(R, K, N, ldr, rowexp, shift, colexp, out, K_pad, N_pad);
  else
    slice_r_kernel<7><<<1184, 256, 0, st>>>(R, K, N, ldr, rowexp, shift, colexp, out, K_pad, N_pad);
  count_launch(3);
  return cudaGetLastError();
}

template <class T>
void slice_a(int S, const T* A, int64_t m, int64_t n, int64_t lda, int64_t r0, int64_t r1, const int* rowexp,
             const int* colexp, int64_t chunk_rows, int8_t* rs, int8_t* cs, int64_t m_pad, int64_t n_pad,
             cudaStream_t st) {
  const int64_t items = (r1 - r0 + 3) / 4 * n_pad;
  if (items <= 0) return;
  const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((items + 255) / 256, 148 * 32));
  if (S == 4)
    slice_a_kernel<T, 4><<<blocks, 256, 0, st>>>(A, m, n, lda, r0, r1, rowexp, colexp, chunk_rows, rs, cs, m_pad,
                                                 n_pad);
  else
    slice_a_kernel<T, 7><<<blocks, 256, 0, st>>>(A, m, n, lda, r0, r1, rowexp, colexp, chunk_rows, rs, cs, m_pad,
                                                 n_pad);
}

}  // namespace

bool ozaki_enabled(int64_t m, int64_t n) {
  const char* e = std::getenv("RFGPU_OZAKI");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return true;
  return m * n >= (int64_t(1) << 26);  // large passes only: the digit planes cost 14 m n bytes
}

OzakiA ozaki_layout(int64_t m, int64_t n, int digits) {
  OzakiA a{};
  a.m = m;
  a.n = n;
  a.digits = digits;
  a.m_pad = roundup(std::max<int64_t>(m, 1), 256);
  a.n_pad = roundup(std::max<int64_t>(n, 1), OBM);
  a.chunk_rows = tn_split_k();  // the A^T Q K-splits: a multiple of 256
  a.nchunks = (a.m_pad + a.chunk_rows - 1) / a.chunk_rows;
  return a;
}

size_t ozaki_set_bytes(int64_t m, int64_t n, int digits) {
  const OzakiA a = ozaki_layout(m, n, digits);
  return static_cast<size_t>(digits) * a.m_pad * a.n_pad;
}

int64_t ozaki_chunk_rows() { return tn_split_k(); }

// The column-scaled set is row-major, read M-major by A^T Q (measured: the column-major set read K-major is
// ~30 % slower on the tensor cores); the K-major reader remains for the shared-set fallback.
bool ozaki_cs_rowmajor() { return true; }

size_t ozaki_a_bytes(int64_t m, int64_t n, int digits) {
  const OzakiA a = ozaki_layout(m, n, digits);
  return ozaki_set_bytes(m, n, digits) + sizeof(int) * (2 * a.m_pad + a.nchunks * a.n_pad + 8) +
         sizeof(uint32_t) * (a.m_pad / 256) * a.n_pad + 1024;
}

namespace {
// Column chunks of the stats pass: >= 4 CTAs per SM in total.
int64_t stats_chunks(int64_t rows, int64_t n) {
  const int64_t rb = std::max<int64_t>(1, (rows + 255) / 256), cb = std::max<int64_t>(1, (n + 255) / 256);
  return std::max<int64_t>(1, std::min<int64_t>(cb, (592 + rb - 1) / rb));
}
}  // namespace

int64_t ozaki_ssq_slots(int64_t rows, int64_t n) { return ((rows + 255) / 256) * stats_chunks(rows, n); }

void ozaki_bind(void* work, int64_t m, int64_t n, int digits, OzakiA* out) {
  *out = ozaki_layout(m, n, digits);
  const size_t planes = ozaki_set_bytes(m, n, digits);
  int8_t* base = static_cast<int8_t*>(work);
  out->rs = base;
  out->cs = nullptr;  // the caller binds the column-scaled set (OzPasses::init / columns)
  out->rowexp = reinterpret_cast<int*>(base + planes);
  out->colexp = out->rowexp + out->m_pad;
  out->ext = out->colexp + out->nchunks * out->n_pad;
  out->rowhi = reinterpret_cast<uint32_t*>(out->ext + 8);
  out->colpart = out->rowhi + out->m_pad;
}

template <class T>
cudaError_t prepare_rows_t(const T* A, int64_t lda, int64_t r0, int64_t r1, const OzakiA& a, double* ssq_part,
                           bool slice_rows, cudaStream_t st) {
  if (r1 == a.m && a.m_pad > a.m) {  // padding rows: exponent 0, zero column maxima
    cudaError_t e = cudaMemsetAsync(a.rowexp + a.m, 0, sizeof(int) * (a.m_pad - a.m), st);
    if (e != cudaSuccess) return e;
  }
  const int64_t rows = r1 - r0;
  const int64_t blocks = (rows + 255) / 256;
  const int64_t s1 = r1 == a.m ? a.m_pad : r1;
  if (rows > 0) {
    const int64_t chunks = stats_chunks(rows, a.n);
    const int64_t chunk = ((a.n + chunks - 1) / chunks + 255) / 256 * 256;
    uint32_t* rowhi = reinterpret_cast<uint32_t*>(a.rowhi);
    if (chunks > 1) {
      cudaError_t e = cudaMemsetAsync(rowhi + r0, 0, sizeof(uint32_t) * rows, st);
      if (e != cudaSuccess) return e;
    }
    dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>((a.n + chunk - 1) / chunk));
    stats_kernel<T><<<grid, 256, 0, st>>>(A, r0, r1, a.n, lda, a.n_pad, chunk, rowhi, a.colpart, ssq_part);
    rowexp_kernel<<<static_cast<unsigned>(std::min<int64_t>((rows + 255) / 256, 1184)), 256, 0, st>>>(rowhi, r0, r1,
                                                                                                       a.rowexp);
    count_launch(2);
  }
  if (slice_rows) {
    slice_a<T>(a.digits, A, a.m, a.n, lda, r0, s1, a.rowexp, nullptr, a.chunk_rows, a.rs, nullptr, a.m_pad, a.n_pad,
               st);
    count_launch();
  }
  return cudaGetLastError();
}

cudaError_t ozaki_prepare_rows(const void* A, bool f32, int64_t lda, int64_t r0, int64_t r1, const OzakiA& a,
                               double* ssq_part, bool slice_rows, cudaStream_t st) {
  return f32 ? prepare_rows_t(static_cast<const float*>(A), lda, r0, r1, a, ssq_part, slice_rows, st)
             : prepare_rows_t(static_cast<const double*>(A), lda, r0, r1, a, ssq_part, slice_rows, st);
}

namespace {
cudaError_t chunk_colexp(const OzakiA& a, int64_t c0, int64_t c1, cudaStream_t st) {
  if (c1 <= c0) return cudaSuccess;
  const int64_t nblk = (a.m + 255) / 256;
  colexp_kernel<<<static_cast<unsigned>((a.n_pad + 31) / 32), dim3(32, 32), 0, st>>>(
      a.colpart, nblk, a.chunk_rows / 256, c0, c1, a.n, a.n_pad, a.colexp, a.ext);
  count_launch();
  return cudaGetLastError();
}
}  // namespace

cudaError_t ozaki_col_exponents(OzakiA* a, cudaStream_t st, int* h_ext, bool decide) {
  cudaError_t e = cudaMemsetAsync(a->ext, 0x80, 2 * sizeof(int), st);  // very negative
  if (e != cudaSuccess) return e;
  if ((e = chunk_colexp(*a, 0, a->nchunks, st)) != cudaSuccess) return e;
  if (!decide) {  // the second digit set is already allocated: nothing to decide on the host, no sync
    a->shared = false;
    a->shared_ok = false;
    return cudaGetLastError();
  }
  if ((e = cudaMemcpyAsync(h_ext, a->ext, 2 * sizeof(int), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  const bool any = h_ext[0] > -100000;  // some non-zero column
  a->emax = any ? h_ext[0] : 0;
  const int spread = any ? h_ext[0] + h_ext[1] : 0;
  a->shared_ok = spread <= kSharedSpread;
  const char* v = std::getenv("RFGPU_OZAKI_SHARED");  // experiments / tests: 0 never, 1 always
  a->shared = v && v[0] == '1';
  return cudaGetLastError();
}

template <class T>
cudaError_t slice_sets_t(const T* A, int64_t lda, const OzakiA& a, bool rows, bool cols, int64_t r0, int64_t r1,
                         cudaStream_t st) {
  if (cols && a.cs_rowmajor) {
    const size_t smem = sizeof(uint32_t) * a.digits * kSliceTCols * 33;
    static std::atomic<uint64_t> cfg{0};
    if (attr_pending(cfg)) {
      for (auto fn : {slice_at_kernel<T, 7>, slice_at_kernel<T, 4>}) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sizeof(uint32_t) * 7 * kSliceTCols * 33));
        if (e != cudaSuccess) return e;
      }
      attr_done(cfg);
    }
    if (r1 <= r0) return cudaSuccess;
    const unsigned grid = static_cast<unsigned>(((r1 - r0) / kSliceTRows) * (a.n_pad / kSliceTCols));
    // cp.async loads (all 8 columns of a lane in flight) whenever the columns are 16-byte aligned; the
    // register-prefetch slicer otherwise (5.8 vs 5.2 TB/s at config 3)
    if ((lda * sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
      constexpr size_t smem_async = sizeof(uint32_t) * kSliceTCols * 256;
      static std::atomic<uint64_t> cfg_async{0};
      if (attr_pending(cfg_async)) {
        for (auto fn : {slice_at_async_kernel<T, 7>, slice_at_async_kernel<T, 4>}) {
          cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_async);
          if (e != cudaSuccess) return e;
        }
        attr_done(cfg_async);
      }
      if (a.digits == 4)
        slice_at_async_kernel<T, 4><<<grid, 256, smem_async, st>>>(A, a.m, a.n, lda, a.rowexp, a.colexp, a.chunk_rows,
                                                                r0, rows ? a.rs : nullptr, a.cs, a.m_pad, a.n_pad);
      else
        slice_at_async_kernel<T, 7><<<grid, 256, smem_async, st>>>(A, a.m, a.n, lda, a.rowexp, a.colexp, a.chunk_rows,
                                                                r0, rows ? a.rs : nullptr, a.cs, a.m_pad, a.n_pad);
      count_launch();
      return cudaGetLastError();
    }
    if (a.digits == 4)
      slice_at_kernel<T, 4><<<grid, 256, smem, st>>>(A, a.m, a.n, lda, a.rowexp, a.colexp, a.chunk_rows, r0,
                                                     rows ? a.rs : nullptr, a.cs, a.m_pad, a.n_pad);
    else
      slice_at_kernel<T, 7><<<grid, 256, smem, st>>>(A, a.m, a.n, lda, a.rowexp, a.colexp, a.chunk_rows, r0,
                                                     rows ? a.rs : nullptr, a.cs, a.m_pad, a.n_pad);
    count_launch();
    return cudaGetLastError();
  }
  slice_a<T>(a.digits, A, a.m, a.n, lda, r0, r1, a.rowexp, a.colexp, a.chunk_rows, rows ? a.rs : nullptr,
             cols ? a.cs : nullptr, a.m_pad, a.n_pad, st);
  count_launch();
  return cudaGetLastError();
}

cudaError_t ozaki_slice_sets(const void* A, bool f32, int64_t lda, const OzakiA& a, bool rows, bool cols,
                             cudaStream_t st) {
  if (!rows && !cols) return cudaSuccess;
  return f32 ? slice_sets_t(static_cast<const float*>(A), lda, a, rows, cols, 0, a.m_pad, st)
             : slice_sets_t(static_cast<const double*>(A), lda, a, rows, cols, 0, a.m_pad, st);
}

// Rows [r0, r1) of an uploaded panel (r0, r1 multiples of chunk_rows, or r1 =
// m): the column exponents of the chunks these rows complete, then their
// column-scaled digits (cs must be bound). Lets the streamed upload slice cs
// panel by panel instead of reading all of A again after the last panel.
cudaError_t ozaki_slice_cols_rows(const void* A, bool f32, int64_t lda, const OzakiA& a, int64_t r0, int64_t r1,
                                  cudaStream_t st) {
  const int64_t s1 = r1 >= a.m ? a.m_pad : r1;
  cudaError_t e = chunk_colexp(a, r0 / a.chunk_rows, (s1 + a.chunk_rows - 1) / a.chunk_rows, st);
  if (e != cudaSuccess) return e;
  return f32 ? slice_sets_t(static_cast<const float*>(A), lda, a, false, true, r0, s1, st)
             : slice_sets_t(static_cast<const double*>(A), lda, a, false, true, r0, s1, st);
}

size_t ozaki_nn_work_bytes(const OzakiA& a, int64_t rows, int64_t ell) {
  const int64_t lp = roundup(ell, OBN);
  const int splits = static_cast<int>((a.n_pad + kSplitK - 1) / kSplitK);
  return static_cast<size_t>(a.digits) * lp * a.n_pad + sizeof(int) * lp + 256 +
         (splits > 1 ? sizeof(double) * static_cast<size_t>(splits) * rows * ell : 0);
}

cudaError_t ozaki_nn(const OzakiA& a, int64_t r0, int64_t r1, const double* X, int64_t ldx, int64_t ell, double* Y,
                     int64_t ldy, void* work, cudaStream_t st) {
  const int64_t lp = roundup(ell, OBN), rows = r1 - r0;
  int8_t* xd = static_cast<int8_t*>(work);
  int* colexp = reinterpret_cast<int*>(xd + static_cast<size_t>(a.digits) * lp * a.n_pad);
  double* ws = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(colexp) + ((sizeof(int) * lp + 255) / 256) * 256);
  cudaError_t e = slice_thin(a.digits, X, a.n, ell, ldx, nullptr, 0, colexp, xd, a.n_pad, lp, st);
  if (e != cudaSuccess) return e;
  // K = n beyond kSplitK would overflow the int32 group sums: split K
  const int splits = static_cast<int>((a.n_pad + kSplitK - 1) / kSplitK);
  OzParams p{};
  p.C = splits > 1 ? ws : Y + r0;
  p.ldc = ldy;
  p.c_row0 = 0;
  p.rowexp = a.rowexp;
  p.colexp = colexp;
  p.ws_mode = splits > 1 ? 1 : 0;
  e = launch_digit_gemm(a.digits, a.rs, a.n_pad, true, a.m_pad, xd, lp, a.n_pad, r0, rows, ell, splits, p, false, st);
  if (e != cudaSuccess || splits == 1) return e;
  const int64_t total = rows * ell;
  reduce_ws_kernel<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16)), 256, 0, st>>>(
      ws, rows, ell, splits, Y + r0, ldy);
  count_launch();
  return cudaGetLastError();
}

size_t ozaki_tn_work_bytes(const OzakiA& a, int64_t ell) {
  const int64_t lp = roundup(ell, OBN);
  const int splits = static_cast<int>((a.m_pad + tn_split_k() - 1) / tn_split_k());
  return static_cast<size_t>(a.digits) * lp * a.m_pad + sizeof(int) * lp + 256 +
         sizeof(double) * static_cast<size_t>(splits) * a.n * ell;
}

cudaError_t ozaki_tn(const OzakiA& a, const double* Q, int64_t ldq, int64_t ell, double* Z, int64_t ldz, void* work,
                     cudaStream_t st, bool presliced) {
  const int64_t lp = roundup(ell, OBN);
  int8_t* qd = static_cast<int8_t*>(work);
  int* colexp = reinterpret_cast<int*>(qd + static_cast<size_t>(a.digits) * lp * a.m_pad);
  double* ws = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(colexp) + ((sizeof(int) * lp + 255) / 256) * 256);
  // Two ways to scale the summation index i (rows of A):
  //  * column-scaled digits of A (a.cs): Z(j, c) = 2^(f_j + g_c) sum_g 2^-(12+8g) acc_g;
  //  * shared (a.shared, one digit set for both passes): the row-scaled digits
  //    a'(i, j) = A(i, j) 2^-e_i with the row factors moved onto Q:
  //    Q'(i, c) = Q(i, c) 2^(e_i - emax) (exact, <= |Q|), sliced per column with
  //    2^-g_c; Z(j, c) = 2^(emax + g_c) sum_g 2^-(12+8g) acc_g. The truncation
  //    error per term is <= 2^-54 2^(emax) max|Q(:, c)| (x2), i.e. at most
  //    2^(emax - f_j + 2) times the column-scaled bound: ozaki_col_exponents
  //    only picks it when every non-zero column has f_j >= emax - kSharedSpread.
  // presliced: ozaki_slice_thin already left Q's column-scaled digits in work (orth's digit Gram)
  cudaError_t e = cudaSuccess;
  if (a.shared)
    e = slice_thin(a.digits, Q, a.m, ell, ldq, a.rowexp, a.emax, colexp, qd, a.m_pad, lp, st);
  else if (!presliced)
    e = slice_thin(a.digits, Q, a.m, ell, ldq, nullptr, 0, colexp, qd, a.m_pad, lp, st);
  if (e != cudaSuccess) return e;
  const int splits = static_cast<int>((a.m_pad + tn_split_k() - 1) / tn_split_k());
  OzParams p{};
  p.C = splits > 1 ? ws : Z;
  p.ldc = ldz;
  p.c_row0 = 0;
  p.rowexp = a.shared ? nullptr : a.colexp;  // output row j of A^T Q = column j of A (per K-split chunk)
  p.rex_stride = a.shared ? 0 : a.n_pad;
  p.kb_split_fixed = a.chunk_rows / BKQ;  // K-splits = the column-exponent chunks
  p.colexp = colexp;
  p.cshift = a.shared ? a.emax : 0;
  p.ws_mode = splits > 1 ? 1 : 0;
  // row-major cs: M-major L tiles (planes [kS][m_pad][n_pad]), like A X. Measured at config 3:
  // 21.9 ms per pass without multicast, 25.9 with the 4-CTA A multicast, 26.6 for the K-major
  // column-major set (which needs the multicast: 37 ms without).
  if (!a.shared && a.cs_rowmajor)
    e = launch_digit_gemm(a.digits, a.cs, a.m_pad, true, a.n_pad, qd, lp, a.m_pad, 0, a.n, ell, splits, p, false, st);
  else
    e = launch_digit_gemm(a.digits, a.shared ? a.rs : a.cs, a.n_pad, false, 0, qd, lp, a.m_pad, 0, a.n, ell, splits, p, true, st);
  if (e != cudaSuccess || splits == 1) return e;
  const int64_t total = a.n * ell;
  reduce_ws_kernel<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16)), 256, 0, st>>>(
      ws, a.n, ell, splits, Z, ldz);
  count_launch();
  return cudaGetLastError();
}

// ---- Gram matrices of tall thin matrices on the digit path -------------------------
// Column-scaled digits of R (K x ell, K = a.m rows) into `work` in ozaki_tn's
// layout (digits [7][lp][m_pad], then the column exponents), so that a
// following ozaki_tn(..., presliced = true) of the same R reuses them.
cudaError_t ozaki_slice_thin(const OzakiA& a, const double* R, int64_t ldr, int64_t ell, void* work, cudaStream_t st) {
  const int64_t lp = roundup(ell, OBN);
  int8_t* qd = static_cast<int8_t*>(work);
  int* colexp = reinterpret_cast<int*>(qd + static_cast<size_t>(a.digits) * lp * a.m_pad);
  return slice_thin(a.digits, R, a.m, ell, ldr, nullptr, 0, colexp, qd, a.m_pad, lp, st);
}

// G (ell x ell, ld ldg) = R^T R from the digits ozaki_slice_thin left in work:
// both operands K-major ([7][lp][m_pad]), split K in fixed order through the
// ozaki_tn workspace. G(i, j) = 2^(g_i + g_j) sum_g 2^-(12+8g) acc_g; the full
// square is computed (the Cholesky reads the upper triangle).
cudaError_t ozaki_gram_thin(const OzakiA& a, int64_t ell, void* work, double* G, int64_t ldg, cudaStream_t st) {
  const int64_t lp = roundup(ell, OBN);
  int8_t* qd = static_cast<int8_t*>(work);
  int* colexp = reinterpret_cast<int*>(qd + static_cast<size_t>(a.digits) * lp * a.m_pad);
  double* ws = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(colexp) + ((sizeof(int) * lp + 255) / 256) * 256);
  const int splits = static_cast<int>((a.m_pad + kSplitK - 1) / kSplitK);
  OzParams p{};
  p.C = splits > 1 ? ws : G;
  p.ldc = ldg;
  p.c_row0 = 0;
  p.rowexp = colexp;
  p.colexp = colexp;
  p.ws_mode = splits > 1 ? 1 : 0;
  cudaError_t e = launch_digit_gemm(a.digits, qd, lp, false, 0, qd, lp, a.m_pad, 0, ell, ell, splits, p, true, st);
  if (e != cudaSuccess || splits == 1) return e;
  const int64_t total = ell * ell;
  reduce_ws_kernel<<<static_cast<unsigned>(std::min<int64_t>((total + 255) / 256, 148 * 16)), 256, 0, st>>>(
      ws, ell, ell, splits, G, ldg);
  count_launch();
  return cudaGetLastError();
}

}  // namespace rfgpu
