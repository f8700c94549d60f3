// Drop-in probe: compiled against the REFERENCE headers
// (/root/reference/proj/include/randfact) and linked ONLY against
// librandfact_b200.so. It proves that a program written for the reference
// API binds the B200 implementation unchanged (same types, same mangled
// entry points, same exception classes).
//
//   dropin_probe cpu                       -> expects randfact::Error without a GPU
//   dropin_probe rsvd A.bin m n k p q reorth out.bin
//   dropin_probe cur  A.bin m n k p out.bin
//   dropin_probe spsvd A.bin m n k p b out.bin -> single_pass_svd(MatrixStream(A, b)) + stream telemetry
//   dropin_probe io   FILE out.bin          -> randfact::read_matrix (matrix_io.hpp) from the drop-in
//   dropin_probe iow  A.bin m n FILE        -> randfact::write_matrix
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <vector>

#include "randfact/common.hpp"
#include "randfact/dense.hpp"
#include "randfact/lowrank.hpp"
#include "randfact/matrix_io.hpp"
#include "randfact/stream.hpp"
#include "randfact/rangefinder.hpp"
#include "randfact/sketch.hpp"

using namespace randfact;

static DenseMatrix read_matrix_bin(const char* path, idx m, idx n) {
  DenseMatrix a(m, n);
  std::ifstream f(path, std::ios::binary);
  f.read(reinterpret_cast<char*>(a.data.data()), static_cast<std::streamsize>(sizeof(double) * m * n));
  return a;
}

static void write_vec(const char* path, const std::vector<double>& v) {
  std::ofstream f(path, std::ios::binary);
  f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(sizeof(double) * v.size()));
}

int main(int argc, char** argv) {
  if (argc >= 2 && std::string(argv[1]) == "cpu") {
    DenseMatrix a = gaussian(1, "probe", 40, 30);
    try {
      SvdFactors f = rsvd(a, 5, 5, 1, 1, false, true);
      std::printf("OK %zu\n", f.D.size());
    } catch (const ParameterError& e) {
      std::printf("PARAM %s\n", e.what());
      return 1;
    } catch (const Error& e) {
      std::printf("DEVICE_ERROR %s\n", e.what());
    }
    try {
      rsvd(a, 0, 5, 1, 1);
    } catch (const ParameterError& e) {
      std::printf("VALIDATION_OK\n");
    }
    return 0;
  }
  if (argc >= 10 && std::string(argv[1]) == "rsvd") {
    const idx m = std::atoll(argv[3]), n = std::atoll(argv[4]);
    DenseMatrix a = read_matrix_bin(argv[2], m, n);
    SvdFactors f = rsvd(a, std::atoll(argv[5]), std::atoll(argv[6]), std::atoll(argv[7]), 1, false, std::atoi(argv[8]));
    std::vector<double> out(f.D);
    out.insert(out.end(), f.U.data.begin(), f.U.data.end());
    write_vec(argv[9], out);
    RangeConfig cfg;
    cfg.k = std::atoll(argv[5]);
    cfg.p = std::atoll(argv[6]);
    cfg.q = std::atoll(argv[7]);
    cfg.seed = 1;
    cfg.reorthonormalize = std::atoi(argv[8]) != 0;
    RangeBasis rb = power_range(a, cfg);
    std::printf("rank %zu Qcols %lld resid %.17g\n", f.D.size(), static_cast<long long>(rb.Q.cols), *rb.residual_frob);
    return 0;
  }
  if (argc >= 8 && std::string(argv[1]) == "cur") {
    const idx m = std::atoll(argv[3]), n = std::atoll(argv[4]);
    DenseMatrix a = read_matrix_bin(argv[2], m, n);
    CurFactors c = randomized_cur(a, std::atoll(argv[5]), std::atoll(argv[6]), 0, 1);
    std::vector<double> out;
    for (idx j : c.Js) out.push_back(static_cast<double>(j));
    for (idx i : c.Is) out.push_back(static_cast<double>(i));
    write_vec(argv[7], out);
    std::printf("kc %zu kr %zu condC %.6g condR %.6g\n", c.Js.size(), c.Is.size(), c.cond_C, c.cond_R);
    return 0;
  }
  if (argc >= 9 && std::string(argv[1]) == "spsvd") {
    const idx m = std::atoll(argv[3]), n = std::atoll(argv[4]);
    DenseMatrix a = read_matrix_bin(argv[2], m, n);
    MatrixStream stream(a, std::atoll(argv[7]));
    SvdFactors f = single_pass_svd(stream, std::atoll(argv[5]), std::atoll(argv[6]), 1);
    write_vec(argv[8], f.D);
    std::printf("rank %zu entries_served %llu passes_completed %d has_next %d\n", f.D.size(),
                static_cast<unsigned long long>(stream.entries_served()), stream.passes_completed(),
                stream.has_next() ? 1 : 0);
    try {
      single_pass_svd(stream, std::atoll(argv[5]), std::atoll(argv[6]), 1);
      std::printf("SECOND_PASS_ALLOWED\n");
    } catch (const StreamContractError&) {
      std::printf("STREAM_CONTRACT_OK\n");
    }
    return 0;
  }
  if (argc >= 4 && std::string(argv[1]) == "io") {
    try {
      DenseMatrix a = read_matrix(argv[2]);
      write_vec(argv[3], a.data);
      std::printf("OK %lld %lld\n", static_cast<long long>(a.rows), static_cast<long long>(a.cols));
    } catch (const ParseError& e) {
      std::printf("PARSE_ERROR %s\n", e.what());
    } catch (const ParameterError& e) {
      std::printf("PARAM_ERROR %s\n", e.what());
    } catch (const Error& e) {
      std::printf("ERROR %s\n", e.what());
    }
    return 0;
  }
  if (argc >= 6 && std::string(argv[1]) == "iow") {
    const idx m = std::atoll(argv[3]), n = std::atoll(argv[4]);
    DenseMatrix a = read_matrix_bin(argv[2], m, n);
    try {
      write_matrix(argv[5], a);
      std::printf("OK\n");
    } catch (const NumericalError& e) {
      std::printf("NUMERICAL_ERROR %s\n", e.what());
    } catch (const ParameterError& e) {
      std::printf("PARAM_ERROR %s\n", e.what());
    }
    return 0;
  }
  std::fprintf(stderr, "usage: dropin_probe cpu | rsvd ... | cur ...\n");
  return 2;
}
