// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// extern "C" shim over the UNMODIFIED reference library (randfact, built from
// /root/reference/proj/src by oracle/Makefile with -Drandfact=randfact_ref so
// its symbols cannot collide with the drop-in). Python tests, smoke() and the
// bench.py cpu_baseline / --impl reference legs load oracle/_ref/librfref.so
// through oracle/oracle.py; nothing else may.
//
// Every entry point wraps one reference call and maps the reference exception
// tree (proj/include/randfact/common.hpp:11-44) to the status codes of
// include/rfgpu.h so the two sides of every parity test report failures the
// same way.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "randfact/common.hpp"
#include "randfact/dense.hpp"
#include "randfact/diagnostics.hpp"
#include "randfact/lowrank.hpp"
#include "randfact/matrix_io.hpp"
#include "randfact/rangefinder.hpp"
#include "randfact/rng.hpp"
#include "randfact/sketch.hpp"
#include "randfact/stream.hpp"

namespace rf = randfact;  // expands to randfact_ref under -Drandfact=randfact_ref

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const rf::ConvergenceError& e) {
        g_err = e.what();
        return 5;
    } catch (const rf::NotPositiveDefiniteError& e) {
        g_err = e.what();
        return 6;
    } catch (const rf::NumericalError& e) {
        g_err = e.what();
        return 4;
    } catch (const rf::ParameterError& e) {
        g_err = e.what();
        return 3;
    } catch (const rf::StreamContractError& e) {
        g_err = e.what();
        return 8;
    } catch (const rf::ParseError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

rf::DenseMatrix wrap(const double* a, int64_t m, int64_t n) {
    rf::DenseMatrix x;
    x.rows = m;
    x.cols = n;
    x.data.assign(a, a + static_cast<std::size_t>(m) * static_cast<std::size_t>(n));
    return x;
}

void put(const rf::DenseMatrix& x, double* out) {
    if (out && !x.data.empty()) std::memcpy(out, x.data.data(), x.data.size() * sizeof(double));
}

void put_idx(const std::vector<rf::idx>& v, int64_t* out) {
    for (std::size_t i = 0; i < v.size(); ++i) out[i] = v[i];
}

}  // namespace

extern "C" {

const char* rfref_last_error() { return g_err.c_str(); }

void rfref_set_threads(int n) { rf::set_max_threads(n); }
int rfref_threads() { return rf::max_threads(); }

// rng.cpp:12-56 / sketch.cpp:56-62
int rfref_gaussian(uint64_t seed, const char* tag, int64_t m, int64_t n, double* out) {
    return guard([&] { put(rf::gaussian(seed, tag, m, n), out); });
}

uint64_t rfref_splitmix_mix(uint64_t z) { return rf::splitmix_mix(z); }
uint64_t rfref_fnv1a64(const char* s) { return rf::fnv1a64(s); }

// diagnostics.cpp:124-136
int rfref_planted(int64_t m, int64_t n, const double* sigma, int64_t r, uint64_t seed, double* a_out) {
    return guard([&] {
        std::vector<double> s(sigma, sigma + r);
        put(rf::planted_matrix(m, n, s, seed).A, a_out);
    });
}

// dense.cpp:155-187
int rfref_multiply(const double* a, int64_t am, int64_t an, const double* b, int64_t bm, int64_t bn,
                   int ta, int tb, double* c) {
    return guard([&] { put(rf::multiply(wrap(a, am, an), wrap(b, bm, bn), ta != 0, tb != 0), c); });
}

// dense.cpp:402-431. q_out must hold m*n; *cols_out receives the kept count.
int rfref_orth(const double* x, int64_t m, int64_t n, double* q_out, int64_t* cols_out) {
    return guard([&] {
        rf::DenseMatrix q = rf::orth(wrap(x, m, n));
        *cols_out = q.cols;
        put(q, q_out);
    });
}

// dense.cpp:690-701. U m x r, D r, V n x r with r = min(m, n).
int rfref_svd(const double* a, int64_t m, int64_t n, double* u, double* d, double* v) {
    return guard([&] {
        rf::SvdFactors f = rf::svd_dense(wrap(a, m, n));
        put(f.U, u);
        if (d) std::memcpy(d, f.D.data(), f.D.size() * sizeof(double));
        put(f.V, v);
    });
}

// dense.cpp:763-786
int rfref_cholesky(const double* b, int64_t n, double* c) {
    return guard([&] { put(rf::cholesky(wrap(b, n, n)), c); });
}

// dense.cpp:453-552, Rank stop. R is rank x n (ld = rank), Q m x rank.
int rfref_cpqr_rank(const double* a, int64_t m, int64_t n, int64_t k, int64_t* perm, double* r_out,
                    double* q_out, int64_t* rank_out, double* resid_out) {
    return guard([&] {
        rf::PivotedQr f = rf::cpqr(wrap(a, m, n), rf::CpqrStop::rank(k));
        put_idx(f.perm, perm);
        put(f.R, r_out);
        put(f.Q, q_out);
        *rank_out = f.stopped_rank;
        if (resid_out) *resid_out = f.residual_frob;
    });
}

// rangefinder.cpp:56-80 (+ finish_with_projection :24-30). Q m x ell', B ell' x n.
int rfref_power_range(const double* a, int64_t m, int64_t n, int64_t k, int64_t p, int64_t q, int reorth,
                      uint64_t seed, int basic, double* q_out, double* b_out, double* resid_out,
                      int64_t* ell_out) {
    return guard([&] {
        rf::RangeConfig cfg;
        cfg.k = k;
        cfg.p = p;
        cfg.q = q;
        cfg.reorthonormalize = reorth != 0;
        cfg.seed = seed;
        const rf::DenseMatrix am = wrap(a, m, n);
        rf::RangeBasis rb = basic ? rf::basic_range(am, cfg) : rf::power_range(am, cfg);
        *ell_out = rb.Q.cols;
        put(rb.Q, q_out);
        if (rb.B) put(*rb.B, b_out);
        if (resid_out) *resid_out = rb.residual_frob.value_or(-1.0);
    });
}

// lowrank.cpp:74-96. U m x r, D r, V n x r; *rank_out = r.
int rfref_rsvd(const double* a, int64_t m, int64_t n, int64_t k, int64_t p, int64_t q, uint64_t seed,
               int keep, int reorth, double* u, double* d, double* v, int64_t* rank_out) {
    return guard([&] {
        rf::SvdFactors f = rf::rsvd(wrap(a, m, n), k, p, q, seed, keep != 0, reorth != 0);
        *rank_out = static_cast<int64_t>(f.D.size());
        put(f.U, u);
        if (d && !f.D.empty()) std::memcpy(d, f.D.data(), f.D.size() * sizeof(double));
        put(f.V, v);
    });
}

// lowrank.cpp:273-310, Col side. Js ke, Z ke x n.
int rfref_id_col(const double* a, int64_t m, int64_t n, int64_t k, int64_t* js, double* z,
                 int64_t* rank_out, int* truncated) {
    return guard([&] {
        rf::IdFactors f = rf::id_deterministic(wrap(a, m, n), k, rf::IdSide::Col);
        *rank_out = static_cast<int64_t>(f.Js.size());
        put_idx(f.Js, js);
        put(f.Z, z);
        *truncated = f.rank_truncated ? 1 : 0;
    });
}

// lowrank.cpp:312-329. Is ke, X m x ke.
int rfref_randomized_id(const double* a, int64_t m, int64_t n, int64_t k, int64_t p, int64_t q,
                        uint64_t seed, int64_t* is, double* x, int64_t* rank_out, int* truncated) {
    return guard([&] {
        rf::IdFactors f = rf::randomized_id(wrap(a, m, n), k, p, q, seed);
        *rank_out = static_cast<int64_t>(f.Is.size());
        put_idx(f.Is, is);
        put(f.X, x);
        *truncated = f.rank_truncated ? 1 : 0;
    });
}

// lowrank.cpp:348-372. Js kc, Is kr, U kc x kr.
int rfref_randomized_cur(const double* a, int64_t m, int64_t n, int64_t k, int64_t p, int64_t q,
                         uint64_t seed, int64_t* js, int64_t* is, double* u, double* cond_c,
                         double* cond_r, int* warning, int64_t* kc_out, int64_t* kr_out) {
    return guard([&] {
        rf::CurFactors f = rf::randomized_cur(wrap(a, m, n), k, p, q, seed);
        *kc_out = static_cast<int64_t>(f.Js.size());
        *kr_out = static_cast<int64_t>(f.Is.size());
        put_idx(f.Js, js);
        put_idx(f.Is, is);
        put(f.U, u);
        *cond_c = f.cond_C;
        *cond_r = f.cond_R;
        *warning = f.warning ? 1 : 0;
    });
}

// lowrank.cpp:160-220 through stream.cpp:7-24. Feasible only at small k
// (stacked (2 k ell) x k^2 least squares).
int rfref_single_pass_svd(const double* a, int64_t m, int64_t n, int64_t k, int64_t p, uint64_t seed,
                          int64_t block, double* u, double* d, double* v, int64_t* rank_out,
                          uint64_t* entries_served, int* passes) {
    return guard([&] {
        const rf::DenseMatrix am = wrap(a, m, n);
        rf::MatrixStream s(am, block);
        rf::SvdFactors f = rf::single_pass_svd(s, k, p, seed);
        *rank_out = static_cast<int64_t>(f.D.size());
        put(f.U, u);
        if (d && !f.D.empty()) std::memcpy(d, f.D.data(), f.D.size() * sizeof(double));
        put(f.V, v);
        if (entries_served) *entries_served = s.entries_served();
        if (passes) *passes = s.passes_completed();
    });
}

// rangefinder.cpp:45-54
int rfref_frob_residual(double a_frob, const double* b, int64_t m, int64_t n, double* out) {
    return guard([&] { *out = rf::frob_residual(a_frob, wrap(b, m, n)); });
}

// tests/test_support.hpp:37-46 (the reference suite's planted(): Haar factors from the "planted.u" /
// "planted.v" streams), for re-expressing the reference's own tests on their own data
int rfref_test_planted(int64_t m, int64_t n, const double* sigma, int64_t r, uint64_t seed, double* a_out) {
    return guard([&] {
        rf::DenseMatrix u = rf::householder_qr(rf::gaussian(seed, "planted.u", m, r)).first;
        rf::DenseMatrix v = rf::householder_qr(rf::gaussian(seed, "planted.v", n, r)).first;
        for (int64_t j = 0; j < r; ++j)
            for (int64_t i = 0; i < m; ++i) u(i, j) *= sigma[j];
        put(rf::multiply(u, v, false, true), a_out);
    });
}

// matrix_io.cpp:224-233: the reference reader (rows/cols out; data into a
// buffer the caller frees with rfref_free)
int rfref_read_matrix(const char* path, int64_t* rows, int64_t* cols, double** data) {
    return guard([&] {
        rf::DenseMatrix a = rf::read_matrix(path);
        *rows = a.rows;
        *cols = a.cols;
        *data = new double[a.data.size() ? a.data.size() : 1];
        put(a, *data);
    });
}

int rfref_write_matrix(const char* path, const double* a, int64_t m, int64_t n) {
    return guard([&] { rf::write_matrix(path, wrap(a, m, n)); });
}

void rfref_free(double* p) { delete[] p; }

}  // extern "C"
