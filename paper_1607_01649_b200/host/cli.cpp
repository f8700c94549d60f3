// randfact_b200 — command-line front end of the drop-in: the reference CLI's
// `factorize` and `bench` subcommands (proj/src/cli.cpp:268-343, run_algo
// :90-189, error/oracle blocks :191-230) for the algorithms on the B200 path
// (rsvd, spsvd, id, cur), reading Matrix Market / CSV input through
// randfact::read_matrix (host/matrix_io.cpp) and emitting the same
// "randfact/1" JSON report. The factorizations run through librandfact_b200.so
// (the drop-in entry points); the errors are recomputed from the returned
// factors on the device (rfgpu_lowrank_error: ||A - L R||_F and the 10
// Gaussian spectral probes of the reference's estimate_spectral_norm, with its
// probe stream), the exact-spectrum oracle block (inputs up to 320 on a side)
// from the device SVD.
//
// Exit codes follow the reference (cli.cpp:459-471): 0 ok, 2 ParseError
// (unreadable / malformed files), 3 ParameterError and bad command lines,
// 4 NumericalError and other library errors. The reference's other
// algorithms (spevd, nystrom, fastid, adaptive, blocked, hqrrp, randutv) are
// outside the B200 hot path and are rejected with exit code 3.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "randfact_b200.hpp"
#include "rfgpu.h"

namespace randfact {
namespace {

// ---- minimal JSON document (objects keep keys sorted, like the reference's nlohmann::json) ----
struct Json {
  enum Kind { Null, Bool, Int, Real, Str, Arr, Obj } kind = Null;
  bool b = false;
  long long i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> arr;
  std::map<std::string, Json> obj;

  Json() = default;
  Json(bool v) : kind(Bool), b(v) {}                        // NOLINT
  Json(int v) : kind(Int), i(v) {}                          // NOLINT
  Json(long long v) : kind(Int), i(v) {}                    // NOLINT
  Json(long v) : kind(Int), i(v) {}                         // NOLINT
  Json(unsigned long v) : kind(Int), i(static_cast<long long>(v)) {}  // NOLINT
  Json(unsigned long long v) : kind(Int), i(static_cast<long long>(v)) {}  // NOLINT
  Json(double v) : kind(Real), d(v) {}                      // NOLINT
  Json(const char* v) : kind(Str), s(v) {}                  // NOLINT
  Json(std::string v) : kind(Str), s(std::move(v)) {}       // NOLINT
  static Json array() {
    Json j;
    j.kind = Arr;
    return j;
  }
  static Json object() {
    Json j;
    j.kind = Obj;
    return j;
  }
  Json& operator[](const std::string& k) {
    if (kind != Obj) {
      kind = Obj;
      obj.clear();
    }
    return obj[k];
  }
  void push(Json v) {
    kind = Arr;
    arr.push_back(std::move(v));
  }
};

std::string real_text(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[40];
  for (int prec = 15; prec <= 17; ++prec) {  // shortest of these that reads back exactly
    std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
    if (std::strtod(buf, nullptr) == v) break;
  }
  std::string t = buf;
  if (t.find_first_of(".eEn") == std::string::npos) t += ".0";
  return t;
}

void quote(std::string& out, const std::string& s) {
  out.push_back('"');
  for (unsigned char ch : s) {
    switch (ch) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\t': out += "\\t"; break;
      case '\r': out += "\\r"; break;
      default:
        if (ch < 0x20) {
          char b[8];
          std::snprintf(b, sizeof(b), "\\u%04x", ch);
          out += b;
        } else {
          out.push_back(static_cast<char>(ch));
        }
    }
  }
  out.push_back('"');
}

void dump(const Json& j, std::string& out, int indent, int level) {
  const std::string pad(static_cast<std::size_t>(indent * (level + 1)), ' ');
  const std::string end(static_cast<std::size_t>(indent * level), ' ');
  switch (j.kind) {
    case Json::Null: out += "null"; break;
    case Json::Bool: out += j.b ? "true" : "false"; break;
    case Json::Int: out += std::to_string(j.i); break;
    case Json::Real: out += real_text(j.d); break;
    case Json::Str: quote(out, j.s); break;
    case Json::Arr:
      if (j.arr.empty()) {
        out += "[]";
        break;
      }
      out += "[\n";
      for (std::size_t k = 0; k < j.arr.size(); ++k) {
        out += pad;
        dump(j.arr[k], out, indent, level + 1);
        out += k + 1 < j.arr.size() ? ",\n" : "\n";
      }
      out += end + "]";
      break;
    case Json::Obj: {
      if (j.obj.empty()) {
        out += "{}";
        break;
      }
      out += "{\n";
      std::size_t k = 0;
      for (const auto& kv : j.obj) {
        out += pad;
        quote(out, kv.first);
        out += ": ";
        dump(kv.second, out, indent, level + 1);
        out += ++k < j.obj.size() ? ",\n" : "\n";
      }
      out += end + "}";
      break;
    }
  }
}

// ---- command line ------------------------------------------------------------------------
struct Knobs {
  idx k = 10, p = 10, q = 0, b = 32, r = 10;
  double eps = 1e-6;
  std::uint64_t seed = 0;
  bool keep_oversamples = false, reorthonormalize = false, p_given = false;
};

const std::set<std::string>& reference_algos() {  // the reference CLI's list (cli.cpp:31-35)
  static const std::set<std::string> names = {"rsvd", "spevd", "spsvd", "nystrom", "id", "fastid",
                                              "cur", "adaptive", "blocked", "hqrrp", "randutv"};
  return names;
}
const std::set<std::string>& device_algos() {
  static const std::set<std::string> names = {"rsvd", "spsvd", "id", "cur"};
  return names;
}

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

idx parse_idx(const std::string& opt, const std::string& v, idx lo) {
  char* end = nullptr;
  const long long x = std::strtoll(v.c_str(), &end, 10);
  if (v.empty() || *end != '\0') throw Usage(opt + ": '" + v + "' is not an integer");
  if (x < lo) throw Usage(opt + ": value " + v + (lo > 0 ? " is not positive" : " is negative"));
  return x;
}

struct Args {
  std::string cmd;
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;
};

Args parse_args(int argc, char** argv) {
  if (argc < 2) throw Usage("a subcommand is required: factorize | bench");
  Args a;
  a.cmd = argv[1];
  if (a.cmd != "factorize" && a.cmd != "bench") throw Usage("unknown subcommand '" + a.cmd + "'");
  static const std::set<std::string> flag_names = {"--keep-oversamples", "--reorth", "--deterministic"};
  static const std::set<std::string> value_names = {"--algo", "--algos", "--in", "--runs", "--k", "--p", "--q",
                                                    "--b", "--r", "--eps", "--seed", "--report"};
  for (int i = 2; i < argc; ++i) {
    std::string o = argv[i], v;
    const std::size_t eq = o.find('=');
    if (eq != std::string::npos) {
      v = o.substr(eq + 1);
      o = o.substr(0, eq);
    }
    if (flag_names.count(o)) {
      a.flags.insert(o);
    } else if (value_names.count(o)) {
      if (eq == std::string::npos) {
        if (i + 1 >= argc) throw Usage(o + " needs a value");
        v = argv[++i];
      }
      a.opt[o] = v;
    } else {
      throw Usage("unknown option '" + o + "'");
    }
  }
  return a;
}

Knobs knobs_of(const Args& a) {
  Knobs kb;
  auto get = [&](const char* name) -> const std::string* {
    auto it = a.opt.find(name);
    return it == a.opt.end() ? nullptr : &it->second;
  };
  if (auto v = get("--k")) kb.k = parse_idx("--k", *v, 1);
  if (auto v = get("--p")) {
    kb.p = parse_idx("--p", *v, 0);
    kb.p_given = true;
  }
  if (auto v = get("--q")) kb.q = parse_idx("--q", *v, 0);
  if (auto v = get("--b")) kb.b = parse_idx("--b", *v, 1);
  if (auto v = get("--r")) kb.r = parse_idx("--r", *v, 1);
  if (auto v = get("--eps")) kb.eps = std::strtod(v->c_str(), nullptr);
  if (auto v = get("--seed")) kb.seed = std::strtoull(v->c_str(), nullptr, 10);
  kb.keep_oversamples = a.flags.count("--keep-oversamples") > 0;
  kb.reorthonormalize = a.flags.count("--reorth") > 0;
  return kb;
}

// ---- factorizations through the drop-in --------------------------------------------------
struct Run {
  Json results = Json::object();
  std::vector<std::string> warnings;
  DenseMatrix L, R;  // approx = L R (L m x r, R r x n)
};

Json head(const std::vector<double>& v) {
  Json a = Json::array();
  for (std::size_t i = 0; i < v.size() && i < 10; ++i) a.push(v[i]);
  return a;
}
Json head(const std::vector<idx>& v) {
  Json a = Json::array();
  for (std::size_t i = 0; i < v.size() && i < 10; ++i) a.push(static_cast<long long>(v[i]));
  return a;
}

DenseMatrix rows_of(const DenseMatrix& a, const std::vector<idx>& is) {
  DenseMatrix r(static_cast<idx>(is.size()), a.cols);
  for (idx j = 0; j < a.cols; ++j)
    for (idx i = 0; i < r.rows; ++i) r.data[static_cast<std::size_t>(j * r.rows + i)] = a(is[static_cast<std::size_t>(i)], j);
  return r;
}

DenseMatrix transpose(const DenseMatrix& a) {
  DenseMatrix t(a.cols, a.rows);
  for (idx j = 0; j < a.cols; ++j)
    for (idx i = 0; i < a.rows; ++i) t.data[static_cast<std::size_t>(i * a.cols + j)] = a(i, j);
  return t;
}

void svd_factors(Run& out, const SvdFactors& f) {
  out.L = f.U;
  for (idx j = 0; j < out.L.cols; ++j)
    for (idx i = 0; i < out.L.rows; ++i) out.L.data[static_cast<std::size_t>(j * out.L.rows + i)] *= f.D[static_cast<std::size_t>(j)];
  out.R = transpose(f.V);
  out.results["rank"] = static_cast<long long>(f.D.size());
  out.results["singvals_head"] = head(f.D);
}

Run run_algo(const std::string& algo, const DenseMatrix& a, const Knobs& kb) {
  if (!reference_algos().count(algo)) throw ParameterError("unknown algorithm '" + algo + "'");
  if (!device_algos().count(algo))
    throw ParameterError("algorithm '" + algo + "' is outside the B200 hot path (rsvd, spsvd, id, cur)");
  Run out;
  const bool single_pass = algo == "spsvd";
  const idx p_eff = (single_pass && !kb.p_given) ? kb.k : kb.p;  // cli.cpp:94
  if (algo == "rsvd") {
    svd_factors(out, rsvd(a, kb.k, p_eff, kb.q, kb.seed, kb.keep_oversamples, kb.reorthonormalize));
  } else if (algo == "spsvd") {
    MatrixStream stream(a, kb.b);
    svd_factors(out, single_pass_svd(stream, kb.k, p_eff, kb.seed));
    out.results["p_used"] = static_cast<long long>(p_eff);
  } else if (algo == "id") {
    IdFactors f = randomized_id(a, kb.k, p_eff, kb.q, kb.seed);
    out.L = f.X;
    out.R = rows_of(a, f.Is);
    out.results["rank"] = static_cast<long long>(f.Is.size());
    out.results["rows_head"] = head(f.Is);
    if (f.rank_truncated) {
      out.results["rank_truncated"] = true;
      out.warnings.push_back("numerical rank is below the requested k; factors use the smaller rank");
    }
  } else {  // cur: approx = A(:, Js) U A(Is, :)
    CurFactors f = randomized_cur(a, kb.k, p_eff, kb.q, kb.seed);
    const idx kc = static_cast<idx>(f.Js.size()), kr = static_cast<idx>(f.Is.size());
    out.L = DenseMatrix(a.rows, kr);
    for (idx c = 0; c < kc; ++c) {
      const double* col = a.data.data() + f.Js[static_cast<std::size_t>(c)] * a.rows;
      for (idx j = 0; j < kr; ++j) {
        const double u = f.U(c, j);
        if (u == 0.0) continue;
        double* dst = out.L.data.data() + j * a.rows;
        for (idx i = 0; i < a.rows; ++i) dst[i] += col[i] * u;
      }
    }
    out.R = rows_of(a, f.Is);
    out.results["rank"] = static_cast<long long>(kc);
    out.results["cols_head"] = head(f.Js);
    out.results["rows_head"] = head(f.Is);
    out.results["cond_C"] = f.cond_C;
    out.results["cond_R"] = f.cond_R;
    if (f.warning) out.warnings.push_back("selected column or row panel is ill conditioned (above 1e8)");
  }
  return out;
}

// ---- device error recomputation ----------------------------------------------------------
struct Device {
  rfgpu_ctx* ctx = nullptr;
  rfgpu_matrix* a = nullptr;
  Device() {
    const char* dv = std::getenv("RANDFACT_B200_DEVICE");
    check(rfgpu_ctx_create(dv ? std::atoi(dv) : 0, &ctx));
  }
  ~Device() {
    rfgpu_matrix_free(a);
    rfgpu_ctx_destroy(ctx);
  }
  static void check(int code) {
    if (code == RFGPU_OK) return;
    const std::string msg = rfgpu_last_error();
    if (code == RFGPU_EPARAM) throw ParameterError(msg);
    if (code == RFGPU_ENUMERICAL || code == RFGPU_ECONVERGENCE || code == RFGPU_ENOTPD) throw NumericalError(msg);
    throw Error("rfgpu: " + msg);
  }
  void upload(const DenseMatrix& m) {
    rfgpu_matrix_free(a);
    a = nullptr;
    check(rfgpu_matrix_upload(ctx, m.data.data(), m.rows, m.cols, std::max<idx>(1, m.rows), &a));
  }
};

double frob(const DenseMatrix& a) {
  double s = 0.0;
  for (double v : a.data) s += v * v;
  return std::sqrt(s);
}

// errors of the run (cli.cpp:191-206): frob and the 10-probe spectral bound of the residual
Json error_block(Device& dev, const DenseMatrix& a, const Run& run, const Knobs& kb, double af, double* frob_abs) {
  constexpr idx kProbes = 10;
  constexpr double kAlpha = 0.1;
  const DenseMatrix g = gaussian(kb.seed ^ 0x9e3779b9ULL, "specnorm", a.cols, kProbes);
  std::vector<double> pn(kProbes);
  double fa = 0.0;
  Device::check(rfgpu_lowrank_error(dev.ctx, dev.a, run.L.data.data(), run.R.data.data(), run.L.cols, g.data.data(),
                                    kProbes, &fa, pn.data()));
  const double se = (1.0 / kAlpha) * std::sqrt(2.0 / M_PI) * *std::max_element(pn.begin(), pn.end());
  *frob_abs = fa;
  Json e = Json::object();
  e["frob_abs"] = fa;
  e["frob_rel"] = af > 0.0 ? fa / af : 0.0;
  e["spectral_probe_abs"] = se;
  e["spectral_probe_rel"] = af > 0.0 ? se / af : 0.0;
  e["spectral_probe_note"] =
      "probabilistic upper bound from 10 Gaussian probes; understates the true spectral norm with probability at "
      "most 1e-10";
  return e;
}

// exact-spectrum comparison for small inputs (cli.cpp:212-229), singular values from the device SVD
Json oracle_block(Device& dev, const DenseMatrix& a, double frob_abs, idx rank) {
  const bool wide = a.rows < a.cols;
  const DenseMatrix x = wide ? transpose(a) : a;
  const idx r = x.rows, c = x.cols;
  std::vector<double> u(static_cast<std::size_t>(r * c)), sv(static_cast<std::size_t>(c)),
      v(static_cast<std::size_t>(c * c));
  int sweeps = 0;
  Device::check(rfgpu_svd(dev.ctx, x.data.data(), r, c, u.data(), sv.data(), v.data(), &sweeps));
  double tail2 = 0.0;
  for (std::size_t j = static_cast<std::size_t>(std::max<idx>(rank, 0)); j < sv.size(); ++j) tail2 += sv[j] * sv[j];
  const double tail = std::sqrt(tail2);
  Json o = Json::object();
  o["sigma_head"] = head(sv);
  o["rank_compared"] = static_cast<long long>(rank);
  o["eckart_young_tail_at_rank"] = tail;
  o["frob_ratio_to_optimal"] = tail > 0.0 ? Json(frob_abs / tail) : Json();
  return o;
}

Json knob_json(const Knobs& kb, bool det) {
  Json j = Json::object();
  j["k"] = static_cast<long long>(kb.k);
  j["p"] = static_cast<long long>(kb.p);
  j["q"] = static_cast<long long>(kb.q);
  j["b"] = static_cast<long long>(kb.b);
  j["r"] = static_cast<long long>(kb.r);
  j["eps"] = kb.eps;
  j["seed"] = static_cast<unsigned long long>(kb.seed);
  j["keep_oversamples"] = kb.keep_oversamples;
  j["reorthonormalize"] = kb.reorthonormalize;
  j["deterministic"] = det;
  return j;
}

Json input_json(const std::string& path, const DenseMatrix& a, double af) {
  Json j = Json::object();
  j["path"] = path;
  j["rows"] = static_cast<long long>(a.rows);
  j["cols"] = static_cast<long long>(a.cols);
  j["frob"] = af;
  return j;
}

void emit(const Json& rep, const std::string& path) {
  std::string text;
  dump(rep, text, 2, 0);
  text += "\n";
  if (path.empty()) {
    std::cout << text;
    return;
  }
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    if (!out) throw ParseError("cannot open '" + tmp + "' for writing");
    out << text;
    out.flush();
    if (!out) throw ParseError("write to '" + tmp + "' failed");
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    throw ParseError("cannot move report into place at '" + path + "'");
  }
}

Json warnings_json(const std::vector<std::string>& w) {
  Json a = Json::array();
  for (const auto& s : w) a.push(s);
  return a;
}

double ms_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

int factorize(const Args& args) {
  const Knobs kb = knobs_of(args);
  auto get = [&](const char* o) { auto it = args.opt.find(o); return it == args.opt.end() ? std::string() : it->second; };
  const std::string algo = get("--algo"), in = get("--in");
  if (algo.empty()) throw Usage("--algo is required");
  if (in.empty()) throw Usage("--in is required");
  if (!reference_algos().count(algo)) throw Usage("--algo: '" + algo + "' not in {" + "rsvd, spevd, spsvd, nystrom, id, "
                                                                                       "fastid, cur, adaptive, blocked, hqrrp, randutv}");
  const bool det = args.flags.count("--deterministic") > 0;
  const DenseMatrix a = read_matrix(in);
  const double af = frob(a);
  const auto t0 = std::chrono::steady_clock::now();
  Run run = run_algo(algo, a, kb);
  const double wall = ms_since(t0);
  Device dev;
  dev.upload(a);
  Json rep = Json::object();
  rep["schema"] = "randfact/1";
  rep["mode"] = "factorize";
  rep["algo"] = algo;
  rep["input"] = input_json(in, a, af);
  rep["params"] = knob_json(kb, det);
  rep["wall_ms"] = wall;
  rep["results"] = run.results;
  double fa = 0.0;
  rep["errors"] = error_block(dev, a, run, kb, af, &fa);
  if (std::max(a.rows, a.cols) <= 320) rep["oracle"] = oracle_block(dev, a, fa, run.L.cols);
  rep["warnings"] = warnings_json(run.warnings);
  rep["device"] = "B200 (librandfact_b200 drop-in over librfgpu)";
  emit(rep, get("--report"));
  return 0;
}

double median(std::vector<double> v) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const std::size_t h = v.size() / 2;
  return v.size() % 2 ? v[h] : 0.5 * (v[h - 1] + v[h]);
}

int bench(const Args& args) {
  const Knobs kb = knobs_of(args);
  auto get = [&](const char* o) { auto it = args.opt.find(o); return it == args.opt.end() ? std::string() : it->second; };
  const std::string in = get("--in"), list = get("--algos");
  if (list.empty()) throw Usage("--algos is required");
  if (in.empty()) throw Usage("--in is required");
  const idx runs = args.opt.count("--runs") ? parse_idx("--runs", get("--runs"), 1) : 5;
  std::vector<std::string> algos;
  for (std::size_t s = 0; s <= list.size();) {
    std::size_t c = list.find(',', s);
    if (c == std::string::npos) c = list.size();
    if (c > s) algos.push_back(list.substr(s, c - s));
    s = c + 1;
  }
  if (algos.empty()) throw ParameterError("bench needs at least one algorithm in --algos");
  for (const auto& nm : algos)
    if (!reference_algos().count(nm)) throw ParameterError("unknown algorithm '" + nm + "' in --algos");
  const bool det = args.flags.count("--deterministic") > 0;
  const DenseMatrix a = read_matrix(in);
  const double af = frob(a);
  Device dev;
  dev.upload(a);
  Json rep = Json::object();
  rep["schema"] = "randfact/1";
  rep["mode"] = "bench";
  rep["input"] = input_json(in, a, af);
  rep["params"] = knob_json(kb, det);
  rep["runs_per_algo"] = static_cast<long long>(runs);
  Json rows = Json::array(), summary = Json::object();
  for (const auto& nm : algos) {
    std::vector<double> times, rels;
    for (idx i = 0; i < runs; ++i) {
      Knobs kbi = kb;
      kbi.seed = kb.seed + static_cast<std::uint64_t>(i);
      Json row = Json::object();
      row["algo"] = nm;
      row["seed"] = static_cast<unsigned long long>(kbi.seed);
      try {
        const auto t0 = std::chrono::steady_clock::now();
        Run run = run_algo(nm, a, kbi);
        const double ms = ms_since(t0);
        double fa = 0.0;
        Device::check(rfgpu_lowrank_error(dev.ctx, dev.a, run.L.data.data(), run.R.data.data(), run.L.cols, nullptr, 0,
                                          &fa, nullptr));
        const double rel = af > 0.0 ? fa / af : 0.0;
        row["wall_ms"] = ms;
        row["frob_rel"] = rel;
        row["warnings"] = warnings_json(run.warnings);
        times.push_back(ms);
        rels.push_back(rel);
      } catch (const Error& e) {  // a failed run is recorded and the sweep continues
        row["error"] = std::string(e.what());
      }
      rows.push(row);
    }
    Json s = Json::object();
    s["completed"] = static_cast<long long>(times.size());
    s["median_wall_ms"] = median(times);
    s["median_frob_rel"] = median(rels);
    summary[nm] = s;
  }
  rep["runs"] = rows;
  rep["summary"] = summary;
  rep["device"] = "B200 (librandfact_b200 drop-in over librfgpu)";
  emit(rep, get("--report"));
  return 0;
}

}  // namespace
}  // namespace randfact

int main(int argc, char** argv) {
  using namespace randfact;
  try {
    const Args args = parse_args(argc, argv);
    return args.cmd == "factorize" ? factorize(args) : bench(args);
  } catch (const Usage& e) {
    std::cerr << "error: " << e.what() << "\n"
              << "usage: randfact_b200 factorize --algo {rsvd,spsvd,id,cur} --in FILE [--k K] [--p P] [--q Q] [--b B]\n"
              << "                     [--seed S] [--keep-oversamples] [--reorth] [--deterministic] [--report PATH]\n"
              << "       randfact_b200 bench --algos A,B,... --in FILE [--runs N] [knobs as above] [--report PATH]\n";
    return 3;
  } catch (const ParseError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 2;
  } catch (const ParameterError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 3;
  } catch (const Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  }
}
