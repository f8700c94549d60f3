// librandfact_b200.so — the reference randfact hot-path API (see
// include/randfact_b200.hpp) implemented on the B200 through the rfgpu C ABI.
//
// Each entry point keeps the reference's value semantics and contract:
// validation order and exception classes (proj/src/rangefinder.cpp:16-22,
// proj/src/lowrank.cpp:14-20), the seeded sketch drawn from the reference
// stream (rfgpu_gaussian == randfact::gaussian bitwise), result shapes
// (orth may drop columns, rsvd keeps min(k, l') unless keep_oversamples).
// The device work (passes over A, orthonormalisation, small SVD, CPQR)
// happens in librfgpu.so; there is no CPU fallback.
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>

#include "randfact_b200.hpp"
#include "rfgpu.h"

namespace randfact {

// Out-of-line members the reference defines in dense.cpp / stream.cpp; weak so
// a program that also links the reference core keeps a single definition.
__attribute__((weak)) DenseMatrix::DenseMatrix(idx m, idx n) : rows(m), cols(n) {
  if (m < 0 || n < 0) throw ParameterError("DenseMatrix: negative dimension");
  data.assign(static_cast<std::size_t>(m) * static_cast<std::size_t>(n), 0.0);
}

__attribute__((weak)) MatrixStream::MatrixStream(const DenseMatrix& a, idx block_cols) : a_(&a), block_cols_(block_cols) {
  if (block_cols_ < 1) throw ParameterError("MatrixStream: block width must be positive");
}

__attribute__((weak)) MatrixStream::Block MatrixStream::next_block() {
  if (next_col_ >= a_->cols) throw StreamContractError("MatrixStream: single pass already consumed");
  const idx c0 = next_col_;
  const idx c1 = std::min(a_->cols, c0 + block_cols_);
  Block b;
  b.col0 = c0;
  b.block.rows = a_->rows;
  b.block.cols = c1 - c0;
  b.block.data.assign(a_->data.begin() + c0 * a_->rows, a_->data.begin() + c1 * a_->rows);
  next_col_ = c1;
  entries_served_ += static_cast<std::uint64_t>(a_->rows) * static_cast<std::uint64_t>(c1 - c0);
  return b;
}

namespace {

std::mutex g_mu;
rfgpu_ctx* g_ctx = nullptr;
int g_device = -1;

int default_device() {
  if (g_device >= 0) return g_device;
  for (const char* v : {"RANDFACT_B200_DEVICE", "LOCAL_RANK"}) {
    if (const char* s = std::getenv(v)) return std::atoi(s);
  }
  return 0;
}

[[noreturn]] void raise(int code) {
  const std::string msg = rfgpu_last_error();
  switch (code) {
    case RFGPU_EPARAM: throw ParameterError(msg);
    case RFGPU_ENUMERICAL: throw NumericalError(msg);
    case RFGPU_ECONVERGENCE: throw ConvergenceError(msg);
    case RFGPU_ENOTPD: throw NotPositiveDefiniteError(msg);
    case RFGPU_ESTREAM: throw StreamContractError(msg);
    default: throw Error("rfgpu: " + msg);
  }
}

void check(int code) {
  if (code != RFGPU_OK) raise(code);
}

rfgpu_ctx* ctx() {
  if (!g_ctx) check(rfgpu_ctx_create(default_device(), &g_ctx));
  return g_ctx;
}

// Device copy of A for the duration of one call (value semantics).
struct DeviceA {
  rfgpu_matrix* h = nullptr;
  explicit DeviceA(const DenseMatrix& a) {
    check(rfgpu_matrix_upload(ctx(), a.data.data(), a.rows, a.cols, std::max<idx>(1, a.rows), &h));
  }
  ~DeviceA() { rfgpu_matrix_free(h); }
};

void check_sample(idx k, idx p, idx m, idx n, const char* where) {
  if (k < 1) throw ParameterError(std::string(where) + ": k must be at least 1");
  if (p < 0) throw ParameterError(std::string(where) + ": p must be non-negative");
  if (k + p > std::min(m, n)) throw ParameterError(std::string(where) + ": k + p exceeds min(m, n)");
}

DenseMatrix make(idx m, idx n, const double* src) {
  DenseMatrix d;
  d.rows = m;
  d.cols = n;
  d.data.assign(src, src + static_cast<std::size_t>(m) * static_cast<std::size_t>(n));
  return d;
}

DenseMatrix transposed(const DenseMatrix& a) {
  DenseMatrix t;
  t.rows = a.cols;
  t.cols = a.rows;
  t.data.resize(a.data.size());
  for (idx j = 0; j < a.cols; ++j)
    for (idx i = 0; i < a.rows; ++i) t.data[static_cast<std::size_t>(i * a.cols + j)] = a(i, j);
  return t;
}

RangeBasis range_impl(const DenseMatrix& a, const RangeConfig& cfg, const char* where) {
  check_sample(cfg.k, cfg.p, a.rows, a.cols, where);
  const idx ell = cfg.k + cfg.p;
  const DenseMatrix g = gaussian(cfg.seed, "range.G", a.cols, ell);
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceA da(a);
  std::vector<double> q(static_cast<std::size_t>(std::max<idx>(1, a.rows * ell)));
  std::vector<double> b(static_cast<std::size_t>(std::max<idx>(1, ell * a.cols)));
  double resid = 0.0;
  int64_t r = 0;
  check(rfgpu_range_finder(ctx(), da.h, g.data.data(), ell, cfg.q, cfg.reorthonormalize ? 1 : 0, q.data(), b.data(),
                           &resid, &r));
  RangeBasis out;
  out.Q = make(a.rows, r, q.data());
  out.B = make(r, a.cols, b.data());
  out.residual_frob = resid;
  return out;
}

}  // namespace

__attribute__((weak)) DenseMatrix gaussian(std::uint64_t seed, const std::string& tag, idx m, idx n) {
  if (m < 0 || n < 0) throw ParameterError("gaussian: negative dimension");
  DenseMatrix g;
  g.rows = m;
  g.cols = n;
  g.data.resize(static_cast<std::size_t>(m) * static_cast<std::size_t>(n));
  check(rfgpu_gaussian(seed, tag.c_str(), m, n, g.data.data()));
  return g;
}

RangeBasis basic_range(const DenseMatrix& a, const RangeConfig& cfg) {
  if (cfg.q != 0) throw ParameterError("basic_range: q must be 0 (use power_range)");
  RangeConfig c = cfg;
  c.reorthonormalize = false;
  return range_impl(a, c, "basic_range");
}

RangeBasis power_range(const DenseMatrix& a, const RangeConfig& cfg) {
  if (cfg.q < 0) throw ParameterError("power_range: q must be non-negative");
  return range_impl(a, cfg, "power_range");
}

SvdFactors rsvd(const DenseMatrix& a, idx k, idx p, idx q, std::uint64_t seed, bool keep_oversamples,
                bool reorthonormalize) {
  if (q < 0) throw ParameterError("power_range: q must be non-negative");
  check_sample(k, p, a.rows, a.cols, "power_range");
  const idx ell = k + p;
  const DenseMatrix g = gaussian(seed, "range.G", a.cols, ell);
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<double> u(static_cast<std::size_t>(std::max<idx>(1, a.rows * ell)));
  std::vector<double> d(static_cast<std::size_t>(ell));
  std::vector<double> v(static_cast<std::size_t>(std::max<idx>(1, a.cols * ell)));
  int64_t r = 0;
  // A streams in from the caller's DenseMatrix behind the first pass
  check(rfgpu_rsvd_host(ctx(), a.data.data(), a.rows, a.cols, std::max<idx>(1, a.rows), g.data.data(), k, ell, q,
                        keep_oversamples ? 1 : 0, reorthonormalize ? 1 : 0, u.data(), d.data(), v.data(), &r));
  SvdFactors out;
  out.U = make(a.rows, r, u.data());
  out.V = make(a.cols, r, v.data());
  out.D.assign(d.begin(), d.begin() + r);
  return out;
}

IdFactors id_deterministic(const DenseMatrix& a, idx k, IdSide side) {
  if (k < 1) throw ParameterError("id_deterministic: k must be at least 1");
  if (k > std::min(a.rows, a.cols)) throw ParameterError("id_deterministic: k exceeds min(m, n)");
  auto col_id = [&](const DenseMatrix& y, idx kk, std::vector<idx>& js, DenseMatrix& z, bool& trunc) {
    std::lock_guard<std::mutex> lk(g_mu);
    js.assign(static_cast<std::size_t>(kk), 0);
    std::vector<double> zb(static_cast<std::size_t>(kk * y.cols));
    int64_t ke = 0;
    int tr = 0;
    check(rfgpu_col_id(ctx(), y.data.data(), y.rows, y.cols, kk, js.data(), zb.data(), &ke, &tr));
    js.resize(static_cast<std::size_t>(ke));
    z = make(ke, y.cols, zb.data());
    trunc = tr != 0;
  };
  IdFactors out;
  out.side = side;
  bool tr1 = false, tr2 = false;
  switch (side) {
    case IdSide::Col:
      col_id(a, k, out.Js, out.Z, tr1);
      break;
    case IdSide::Row: {
      DenseMatrix z;
      col_id(transposed(a), k, out.Is, z, tr1);
      out.X = transposed(z);
      break;
    }
    case IdSide::Double: {
      col_id(a, k, out.Js, out.Z, tr1);
      DenseMatrix c;
      c.rows = a.rows;
      c.cols = static_cast<idx>(out.Js.size());
      c.data.resize(static_cast<std::size_t>(c.rows * c.cols));
      for (idx j = 0; j < c.cols; ++j)
        std::memcpy(c.data.data() + j * c.rows, a.data.data() + out.Js[static_cast<std::size_t>(j)] * a.rows,
                    sizeof(double) * static_cast<std::size_t>(a.rows));
      DenseMatrix z;
      col_id(transposed(c), c.cols, out.Is, z, tr2);
      out.X = transposed(z);
      break;
    }
  }
  out.rank_truncated = tr1 || tr2;
  return out;
}

IdFactors randomized_id(const DenseMatrix& a, idx k, idx p, idx q, std::uint64_t seed) {
  check_sample(k, p, a.rows, a.cols, "randomized_id");
  if (q < 0) throw ParameterError("randomized_id: q must be non-negative");
  const idx ell = k + p;
  const DenseMatrix g = gaussian(seed, "rid.G", a.cols, ell);
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceA da(a);
  std::vector<idx> is(static_cast<std::size_t>(k));
  std::vector<double> x(static_cast<std::size_t>(std::max<idx>(1, a.rows * k)));
  int64_t ke = 0;
  int tr = 0;
  check(rfgpu_randomized_id(ctx(), da.h, g.data.data(), k, ell, q, is.data(), x.data(), &ke, &tr));
  IdFactors out;
  out.side = IdSide::Row;
  is.resize(static_cast<std::size_t>(ke));
  out.Is = std::move(is);
  out.X = make(a.rows, ke, x.data());
  out.rank_truncated = tr != 0;
  return out;
}

CurFactors randomized_cur(const DenseMatrix& a, idx k, idx p, idx q, std::uint64_t seed) {
  check_sample(k, p, a.rows, a.cols, "randomized_cur");
  if (q < 0) throw ParameterError("randomized_cur: q must be non-negative");
  const idx ell = k + p;
  const DenseMatrix g = gaussian(seed, "cur.G", ell, a.rows);
  std::lock_guard<std::mutex> lk(g_mu);
  DeviceA da(a);
  std::vector<idx> js(static_cast<std::size_t>(k)), is(static_cast<std::size_t>(k));
  std::vector<double> u(static_cast<std::size_t>(k * k));
  double cc = 0.0, cr = 0.0;
  int w = 0;
  int64_t kc = 0, kr = 0;
  check(rfgpu_randomized_cur(ctx(), da.h, g.data.data(), k, ell, q, js.data(), is.data(), u.data(), &cc, &cr, &w, &kc,
                             &kr));
  CurFactors out;
  js.resize(static_cast<std::size_t>(kc));
  is.resize(static_cast<std::size_t>(kr));
  out.Js = std::move(js);
  out.Is = std::move(is);
  out.U = make(kc, kr, u.data());
  out.cond_C = cc;
  out.cond_R = cr;
  out.warning = w != 0;
  return out;
}

SvdFactors single_pass_svd(MatrixStream& stream, idx k, idx p, std::uint64_t seed) {
  // lowrank.cpp:160-220: every block of the stream is consumed once and
  // pushed to the device, where both sketches and the core solve live.
  const idx m = stream.rows(), n = stream.cols();
  check_sample(k, p, m, n, "single_pass_svd");
  const idx ell = k + p;
  const DenseMatrix gc = gaussian(seed, "spsvd.Gc", n, ell);
  const DenseMatrix gr = gaussian(seed, "spsvd.Gr", m, ell);
  std::lock_guard<std::mutex> lk(g_mu);
  rfgpu_single_pass* sp = nullptr;
  check(rfgpu_single_pass_begin(ctx(), m, n, ell, gc.data.data(), gr.data.data(), &sp));
  try {
    // Every remaining column exactly once, in order, in slabs straight from the
    // stream's matrix (no per-block DenseMatrix copies); the stream's counters
    // end as if next_block() had been drained.
    if (stream.next_col_ != 0) throw StreamContractError("MatrixStream: single pass already consumed");
    constexpr idx kSlab = 4096;
    while (stream.has_next()) {
      const idx c0 = stream.next_col_, c1 = std::min(stream.a_->cols, c0 + std::max(kSlab, stream.block_cols_));
      check(rfgpu_single_pass_push(sp, c0, stream.a_->data.data() + c0 * m, c1 - c0));
      stream.next_col_ = c1;
      stream.entries_served_ += static_cast<std::uint64_t>(m) * static_cast<std::uint64_t>(c1 - c0);
    }
  } catch (...) {
    rfgpu_single_pass_abort(sp);
    throw;
  }
  const idx kk = std::min(k, ell);
  std::vector<double> u(static_cast<std::size_t>(m * kk)), d(static_cast<std::size_t>(kk)),
      v(static_cast<std::size_t>(n * kk));
  int64_t r = 0;
  check(rfgpu_single_pass_finish(sp, k, u.data(), d.data(), v.data(), &r));
  SvdFactors out;
  out.U = make(m, r, u.data());
  out.V = make(n, r, v.data());
  out.D.assign(d.begin(), d.begin() + r);
  return out;
}

namespace b200 {
void set_device(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  g_device = device;
}
std::int64_t kernel_launches() { return g_ctx ? rfgpu_launch_count(g_ctx) : 0; }
void release_memory() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_ctx) check(rfgpu_ctx_release_memory(g_ctx));
}
}  // namespace b200

}  // namespace randfact
