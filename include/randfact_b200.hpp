// randfact_b200 — C++ drop-in for the hot path of the reference `randfact`
// library (arXiv 1607.01649 reference, /root/reference/proj/include/randfact).
//
// Declares, in namespace randfact and with the reference's type layouts and
// signatures, the entry points that librandfact_b200.so implements on the
// B200 through the C ABI in rfgpu.h:
//
//   gaussian        sketch.hpp:25        (host, bitwise the reference stream)
//   basic_range     rangefinder.hpp:50
//   power_range     rangefinder.hpp:55
//   rsvd            lowrank.hpp:15-16
//   single_pass_svd lowrank.hpp:41
//   id_deterministic lowrank.hpp:72      (column side on the device)
//   randomized_id   lowrank.hpp:78
//   randomized_cur  lowrank.hpp:102
//
// A program written against the reference headers links this library
// unchanged (the struct layouts and mangled names are the reference's;
// tests/test_dropin_cxx.py compiles a probe against the reference headers and
// links it here). Errors are the reference exception classes.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace randfact {

using idx = std::int64_t;

struct Error : std::runtime_error {
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
};
struct ParseError : Error {
  explicit ParseError(const std::string& msg) : Error(msg) {}
};
struct ParameterError : Error {
  explicit ParameterError(const std::string& msg) : Error(msg) {}
};
struct NumericalError : Error {
  explicit NumericalError(const std::string& msg) : Error(msg) {}
};
struct ConvergenceError : NumericalError {
  explicit ConvergenceError(const std::string& msg) : NumericalError(msg) {}
};
struct NotPositiveDefiniteError : NumericalError {
  explicit NotPositiveDefiniteError(const std::string& msg) : NumericalError(msg) {}
};
struct StreamContractError : Error {
  explicit StreamContractError(const std::string& msg) : Error(msg) {}
};

// Column-major FP64 matrix (layout of the reference DenseMatrix).
struct DenseMatrix {
  idx rows = 0;
  idx cols = 0;
  std::vector<double> data;

  DenseMatrix() = default;
  DenseMatrix(idx m, idx n);

  double& operator()(idx i, idx j) { return data[static_cast<std::size_t>(j * rows + i)]; }
  double operator()(idx i, idx j) const { return data[static_cast<std::size_t>(j * rows + i)]; }
  bool empty() const { return rows == 0 || cols == 0; }
};

struct SvdFactors {
  DenseMatrix U;
  std::vector<double> D;
  DenseMatrix V;
};

struct RangeConfig {
  idx k = 0;
  idx p = 10;
  idx q = 0;
  bool reorthonormalize = false;
  std::uint64_t seed = 0;
};

struct RangeBasis {
  DenseMatrix Q;
  std::optional<DenseMatrix> B;
  std::optional<double> residual_frob;
  std::vector<idx> picks;
};

enum class IdSide { Col, Row, Double };

struct IdFactors {
  IdSide side = IdSide::Col;
  std::vector<idx> Js;
  std::vector<idx> Is;
  DenseMatrix Z;
  DenseMatrix X;
  bool rank_truncated = false;
};

struct CurFactors {
  std::vector<idx> Js;
  std::vector<idx> Is;
  DenseMatrix U;
  double cond_C = 0.0;
  double cond_R = 0.0;
  bool warning = false;
};

// One-shot column-block view (layout of the reference MatrixStream).
class MatrixStream {
 public:
  struct Block {
    idx col0 = 0;
    DenseMatrix block;
  };
  explicit MatrixStream(const DenseMatrix& a, idx block_cols = 32);
  idx rows() const { return a_->rows; }
  idx cols() const { return a_->cols; }
  bool has_next() const { return next_col_ < a_->cols; }
  Block next_block();
  std::uint64_t entries_served() const { return entries_served_; }
  int passes_completed() const { return next_col_ >= a_->cols ? 1 : 0; }

 private:
  // the drop-in's single pass reads the matrix behind the stream directly, in
  // large column slabs, with the same observable effect as draining next_block()
  // (columns consumed once, in order; entries_served / passes_completed)
  friend SvdFactors single_pass_svd(MatrixStream& stream, idx k, idx p, std::uint64_t seed);
  const DenseMatrix* a_;
  idx block_cols_;
  idx next_col_ = 0;
  std::uint64_t entries_served_ = 0;
};

DenseMatrix gaussian(std::uint64_t seed, const std::string& tag, idx m, idx n);
RangeBasis basic_range(const DenseMatrix& a, const RangeConfig& cfg);
RangeBasis power_range(const DenseMatrix& a, const RangeConfig& cfg);
SvdFactors rsvd(const DenseMatrix& a, idx k, idx p, idx q, std::uint64_t seed, bool keep_oversamples = false,
                bool reorthonormalize = false);
SvdFactors single_pass_svd(MatrixStream& stream, idx k, idx p, std::uint64_t seed);
IdFactors id_deterministic(const DenseMatrix& a, idx k, IdSide side);
IdFactors randomized_id(const DenseMatrix& a, idx k, idx p, idx q, std::uint64_t seed);
CurFactors randomized_cur(const DenseMatrix& a, idx k, idx p, idx q, std::uint64_t seed);

// Matrix files (matrix_io.hpp:9-20): .mtx/.mm Matrix Market (array or
// coordinate; real, integer or pattern; general or symmetric) and .csv, by
// extension. ParseError on malformed input, ParameterError on an unknown
// extension; write_matrix commits atomically and refuses non-finite entries.
DenseMatrix read_matrix(const std::string& path);
void write_matrix(const std::string& path, const DenseMatrix& a);

namespace b200 {
// Device used by the drop-in (default: $RANDFACT_B200_DEVICE, else
// $LOCAL_RANK, else 0). Must be called before the first offloaded call.
void set_device(int device);
// Number of rfgpu kernels launched by the drop-in so far (telemetry).
std::int64_t kernel_launches();
// Returns the drop-in's cached device memory (the A buffer kept between
// calls, the context's memory pools) to the driver; the next call
// re-allocates.
void release_memory();
}  // namespace b200

}  // namespace randfact
