// Matrix files for the drop-in: randfact::read_matrix / write_matrix
// (reference proj/include/randfact/matrix_io.hpp, proj/src/matrix_io.cpp:93-252).
//
// Same contract as the reference: the extension picks the format (.mtx/.mm
// Matrix Market — array or coordinate, real/integer/pattern field, general or
// symmetric storage, densified column-major; .csv comma-separated rows);
// malformed content, unsupported qualifiers and non-finite values raise
// ParseError naming "path:line"; an unknown extension raises ParameterError;
// writes are %.17g round-trip text committed by an atomic rename, refusing
// non-finite entries with NumericalError.
//
// The file is read in one block and scanned in place (config-size inputs are
// tens of GB of text: no per-line stream extraction).
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "randfact_b200.hpp"

namespace randfact {
namespace {

std::string to_lower(std::string s) {
  for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
  return s;
}

std::string file_extension(const std::string& path) {
  const std::size_t dot = path.rfind('.');
  const std::size_t slash = path.rfind('/');
  if (dot == std::string::npos || (slash != std::string::npos && dot < slash)) return "";
  return to_lower(path.substr(dot));
}

bool is_space(char c) { return c == ' ' || c == '\t' || c == '\r' || c == '\n' || c == '\v' || c == '\f'; }

std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError("cannot open '" + path + "'");
  in.seekg(0, std::ios::end);
  const std::streamoff size = in.tellg();
  in.seekg(0, std::ios::beg);
  std::string buf(static_cast<std::size_t>(size > 0 ? size : 0), '\0');
  if (size > 0 && !in.read(&buf[0], size)) throw ParseError("cannot read '" + path + "'");
  return buf;
}

// Scanner over the whole file text. `line` is the 1-based number of the line
// the scanner is on; blank lines never count as content, '%' comment lines
// are skipped once `comments` is set (Matrix Market after the banner).
class Scanner {
 public:
  Scanner(const std::string& text, const std::string& path) : t_(text), path_(path) {}

  [[noreturn]] void fail(const std::string& what) const {
    throw ParseError(path_ + ":" + std::to_string(line_) + ": " + what);
  }

  // Advance to the next content line; its [begin, end) range in cur_/eol_.
  bool next_line() {
    while (next_ < t_.size()) {
      const std::size_t b = next_;
      std::size_t e = t_.find('\n', b);
      if (e == std::string::npos) e = t_.size();
      next_ = e + 1;
      ++line_;
      cur_ = b;
      eol_ = e;
      if (comments && e > b && t_[b] == '%') continue;
      std::size_t k = b;
      while (k < e && is_space(t_[k])) ++k;
      if (k == e) continue;
      return true;
    }
    cur_ = eol_ = t_.size();
    return false;
  }

  std::string rest_of_line() const { return t_.substr(cur_, eol_ - cur_); }
  void skip_line() { cur_ = eol_; }

  // Next whitespace-separated token, across line boundaries.
  bool token(const char** p, std::size_t* n) {
    for (;;) {
      while (cur_ < eol_ && is_space(t_[cur_])) ++cur_;
      if (cur_ < eol_) break;
      if (!next_line()) return false;
    }
    const std::size_t b = cur_;
    while (cur_ < eol_ && !is_space(t_[cur_])) ++cur_;
    *p = t_.data() + b;
    *n = cur_ - b;
    return true;
  }

  double real(const char* what) {
    const char* p;
    std::size_t n;
    if (!token(&p, &n)) fail(std::string("unexpected end of file, expected ") + what);
    return parse_real(p, n, what, true);
  }

  idx index(const char* what) {
    const char* p;
    std::size_t n;
    if (!token(&p, &n)) fail(std::string("unexpected end of file, expected ") + what);
    char buf[64];
    const std::string tok(p, n);
    if (n >= sizeof(buf)) fail("bad " + std::string(what) + " '" + tok + "'");
    std::memcpy(buf, p, n);
    buf[n] = '\0';
    char* end = nullptr;
    const long long v = std::strtoll(buf, &end, 10);
    if (end != buf + n || v < 0) fail("bad " + std::string(what) + " '" + tok + "'");
    return static_cast<idx>(v);
  }

  // strtod over exactly [p, p + n) (the whole token must parse; finite only)
  double parse_real(const char* p, std::size_t n, const char* what, bool token_msg) const {
    char small[128];
    std::string big;
    char* s = small;
    if (n >= sizeof(small)) {
      big.assign(p, n);
      s = &big[0];
    } else {
      std::memcpy(small, p, n);
      small[n] = '\0';
    }
    char* end = nullptr;
    const double v = std::strtod(s, &end);
    const std::string tok(p, n);
    if (end != s + n) fail((token_msg ? "bad " + std::string(what) + " '" : "bad value '") + tok + "'");
    if (!std::isfinite(v)) fail((token_msg ? std::string(what) + " '" : "value '") + tok + "' is not finite");
    return v;
  }

  bool comments = false;
  std::size_t cur_ = 0, eol_ = 0;

 private:
  const std::string& t_;
  const std::string& path_;
  std::size_t next_ = 0;
  long line_ = 0;
};

DenseMatrix parse_matrix_market(const std::string& text, const std::string& path) {
  Scanner sc(text, path);
  if (!sc.next_line()) sc.fail("empty file");
  std::vector<std::string> words;
  {
    const std::string head = sc.rest_of_line();
    std::size_t i = 0;
    while (words.size() < 5) {
      while (i < head.size() && is_space(head[i])) ++i;
      if (i >= head.size()) break;
      std::size_t j = i;
      while (j < head.size() && !is_space(head[j])) ++j;
      words.push_back(head.substr(i, j - i));
      i = j;
    }
    words.resize(5);
  }
  const std::string banner = to_lower(words[0]), object = to_lower(words[1]), format = to_lower(words[2]),
                    field = to_lower(words[3]), symmetry = to_lower(words[4]);
  if (banner != "%%matrixmarket") sc.fail("missing %%MatrixMarket banner");
  if (object != "matrix") sc.fail("unsupported object '" + words[1] + "'");
  if (format != "array" && format != "coordinate") sc.fail("unsupported format '" + format + "'");
  if (field == "complex") sc.fail("complex matrices are not supported");
  if (field != "real" && field != "integer" && field != "pattern") sc.fail("unsupported field '" + field + "'");
  if (symmetry == "hermitian" || symmetry == "skew-symmetric") sc.fail("unsupported symmetry '" + symmetry + "'");
  if (symmetry != "general" && symmetry != "symmetric") sc.fail("unsupported symmetry '" + symmetry + "'");
  if (format == "array" && field == "pattern") sc.fail("array format cannot carry a pattern field");
  sc.skip_line();
  sc.comments = true;
  const bool sym = symmetry == "symmetric";
  const idx m = sc.index("row count");
  const idx n = sc.index("column count");
  if (m <= 0 || n <= 0) sc.fail("matrix dimensions must be positive");
  if (sym && m != n) sc.fail("symmetric storage requires a square matrix");
  DenseMatrix a(m, n);
  double* d = a.data.data();
  if (format == "array") {  // column-major; symmetric storage lists the lower triangle only
    for (idx j = 0; j < n; ++j) {
      for (idx i = sym ? j : 0; i < m; ++i) {
        const double v = sc.real("matrix entry");
        d[j * m + i] = v;
        if (sym && i != j) d[i * m + j] = v;
      }
    }
  } else {
    const idx nnz = sc.index("entry count");
    const bool pattern = field == "pattern";
    for (idx e = 0; e < nnz; ++e) {
      const idx i = sc.index("row index") - 1;
      const idx j = sc.index("column index") - 1;
      if (i < 0 || i >= m || j < 0 || j >= n) sc.fail("entry index out of range");
      const double v = pattern ? 1.0 : sc.real("matrix entry");
      d[j * m + i] += v;  // duplicates accumulate
      if (sym && i != j) d[i * m + j] += v;
    }
  }
  const char* p;
  std::size_t len;
  if (sc.token(&p, &len)) sc.fail("trailing content '" + std::string(p, len) + "' after matrix data");
  return a;
}

DenseMatrix parse_csv(const std::string& text, const std::string& path) {
  Scanner sc(text, path);
  std::vector<double> vals;  // row-major while reading
  std::size_t width = 0, rows = 0;
  while (sc.next_line()) {
    const std::size_t b = sc.cur_, e = sc.eol_;
    std::size_t count = 0, s = b;
    for (;;) {
      std::size_t c = text.find(',', s);
      if (c == std::string::npos || c > e) c = e;
      std::size_t lo = s, hi = c;
      while (lo < hi && (text[lo] == ' ' || text[lo] == '\t' || text[lo] == '\r')) ++lo;
      while (hi > lo && (text[hi - 1] == ' ' || text[hi - 1] == '\t' || text[hi - 1] == '\r')) --hi;
      if (lo == hi) sc.fail("empty cell");
      vals.push_back(sc.parse_real(text.data() + lo, hi - lo, "value", false));
      ++count;
      if (c == e) break;
      s = c + 1;
    }
    if (rows > 0 && count != width)
      sc.fail("row has " + std::to_string(count) + " cells, expected " + std::to_string(width));
    width = count;
    ++rows;
    sc.skip_line();
  }
  if (rows == 0) throw ParseError(path + ": no data rows");
  DenseMatrix a(static_cast<idx>(rows), static_cast<idx>(width));
  for (std::size_t i = 0; i < rows; ++i)
    for (std::size_t j = 0; j < width; ++j) a.data[j * rows + i] = vals[i * width + j];
  return a;
}

void commit_atomically(const std::string& path, const std::string& body) {
  const std::string tmp = path + ".tmp";
  {
    std::ofstream out(tmp, std::ios::binary | std::ios::trunc);
    if (!out) throw ParseError("cannot open '" + tmp + "' for writing");
    out.write(body.data(), static_cast<std::streamsize>(body.size()));
    out.flush();
    if (!out) throw ParseError("write to '" + tmp + "' failed");
  }
  if (std::rename(tmp.c_str(), path.c_str()) != 0) {
    std::remove(tmp.c_str());
    throw ParseError("cannot move '" + tmp + "' into place at '" + path + "'");
  }
}

void append_value(std::string& out, double v) {
  char buf[40];
  const int n = std::snprintf(buf, sizeof(buf), "%.17g", v);
  out.append(buf, static_cast<std::size_t>(n));
}

}  // namespace

DenseMatrix read_matrix(const std::string& path) {
  const std::string ext = file_extension(path);
  if (ext != ".mtx" && ext != ".mm" && ext != ".csv")
    throw ParameterError("unknown matrix file extension '" + ext + "' in '" + path + "'");
  const std::string text = slurp(path);
  return ext == ".csv" ? parse_csv(text, path) : parse_matrix_market(text, path);
}

void write_matrix(const std::string& path, const DenseMatrix& a) {
  const std::string ext = file_extension(path);
  if (ext != ".mtx" && ext != ".mm" && ext != ".csv")
    throw ParameterError("unknown matrix file extension '" + ext + "' in '" + path + "'");
  if (a.rows <= 0 || a.cols <= 0) throw ParameterError("refusing to write an empty matrix");
  for (idx j = 0; j < a.cols; ++j)
    for (idx i = 0; i < a.rows; ++i)
      if (!std::isfinite(a.data[static_cast<std::size_t>(j * a.rows + i)]))
        throw NumericalError("refusing to write non-finite entry at (" + std::to_string(i) + ", " +
                             std::to_string(j) + ") to " + path);
  std::string body;
  body.reserve(static_cast<std::size_t>(a.rows * a.cols) * 24 + 64);
  if (ext == ".csv") {
    for (idx i = 0; i < a.rows; ++i) {
      for (idx j = 0; j < a.cols; ++j) {
        if (j) body.push_back(',');
        append_value(body, a.data[static_cast<std::size_t>(j * a.rows + i)]);
      }
      body.push_back('\n');
    }
  } else {
    body += "%%MatrixMarket matrix array real general\n";
    body += std::to_string(a.rows) + " " + std::to_string(a.cols) + "\n";
    for (double v : a.data) {
      append_value(body, v);
      body.push_back('\n');
    }
  }
  commit_atomically(path, body);
}

}  // namespace randfact
