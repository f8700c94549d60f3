/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the randomized range-finder
 * hot path. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it (through oracle/oracle.py), and only as the checker.
 *
 * A plain-C restatement of the reference algorithms on the north-star path,
 * written to reproduce the reference's floating-point operation ORDER so that,
 * built like the reference (g++/gcc -O3, no -march, hence no FMA contraction
 * on x86-64), its outputs are bitwise identical to the compiled reference
 * (pinned in tests/test_oracle_pin.py against oracle/_ref and against the
 * committed fixtures in tests/golden/).
 *
 *   rng / gaussian ........ proj/src/rng.cpp:12-56, proj/src/sketch.cpp:56-62
 *   multiply nn/tn/nt ..... proj/src/dense.cpp:102-138 (fixed per-entry order)
 *   frob / vec norms ...... proj/src/dense.cpp:232-248
 *   orth (MGS x2, drop) ... proj/src/dense.cpp:402-431
 *   reflectors, HQR ....... proj/src/dense.cpp:328-400
 *   cpqr (rank stop) ...... proj/src/dense.cpp:453-552
 *   svd_tall / svd_dense .. proj/src/dense.cpp:560-701
 *   solve_upper ........... proj/src/dense.cpp:788-804
 *   least_squares ......... proj/src/dense.cpp:825-837
 *   power/basic range ..... proj/src/rangefinder.cpp:16-80
 *   rsvd .................. proj/src/lowrank.cpp:74-96
 *   col_id_core / ID / CUR  proj/src/lowrank.cpp:37-70, 312-372
 *   planted_matrix ........ proj/src/diagnostics.cpp:124-136
 *   single_pass_svd ....... proj/src/lowrank.cpp:160-220, core restated as the
 *                           normal-equation Sylvester solve:
 *                           the reference's stacked (2 k l) x k^2 design is
 *                           infeasible at config-4 size; pinned against the
 *                           reference at small k in tests/test_oracle_pin.py.
 *
 * Status codes match include/rfgpu.h: 0 ok, 3 parameter, 4 numerical,
 * 5 convergence, 6 not positive definite, 9 out of memory.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t i64;

enum { OK = 0, E_PARAM = 3, E_NUM = 4, E_CONV = 5, E_NOTPD = 6, E_NOMEM = 9 };

static __thread char g_err[256];
static int fail(int code, const char *msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char *rfo_last_error(void) { return g_err; }

#define AT(p, ld, i, j) ((p)[(size_t)(j) * (size_t)(ld) + (size_t)(i)])

static double *dalloc(i64 n) {
    return (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
}

static int g_threads = 0;
void rfo_set_threads(int n) { g_threads = n; }
static int nthreads(void) {
#ifdef _OPENMP
    return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---------------------------------------------------------------- rng --- */

uint64_t rfo_mix(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

uint64_t rfo_fnv1a64(const char *s) {
    uint64_t h = 0xCBF29CE484222325ULL;
    for (const unsigned char *c = (const unsigned char *)s; *c; ++c) {
        h ^= *c;
        h *= 0x100000001B3ULL;
    }
    return h;
}

static double u01_at(uint64_t key, uint64_t counter) {
    const uint64_t x = rfo_mix(key + 0x9E3779B97F4A7C15ULL * counter) >> 11;
    return ((double)x + 0.5) * 0x1.0p-53;
}

/* Elements [e0, e0+count) of the column-major gaussian(seed, tag, ., .):
 * element e is Box-Muller over draws 2*floor(e/2)+1 and +2; cos for even e,
 * sin for odd e (the reference caches the sin variate). */
int rfo_gaussian_range(uint64_t seed, const char *tag, i64 e0, i64 count, double *out) {
    if (e0 < 0 || count < 0) return fail(E_PARAM, "gaussian: negative range");
    const uint64_t key = rfo_mix(seed ^ rfo_fnv1a64(tag));
    const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static) num_threads(nthreads())
    for (i64 t = 0; t < count; ++t) {
        const i64 e = e0 + t;
        const uint64_t pair = (uint64_t)(e / 2);
        const double u1 = u01_at(key, 2 * pair + 1);
        const double u2 = u01_at(key, 2 * pair + 2);
        const double r = sqrt(-2.0 * log(u1));
        out[t] = (e % 2 == 0) ? r * cos(two_pi * u2) : r * sin(two_pi * u2);
    }
    return OK;
}

int rfo_gaussian(uint64_t seed, const char *tag, i64 m, i64 n, double *out) {
    if (m < 0 || n < 0) return fail(E_PARAM, "gaussian: negative dimension");
    return rfo_gaussian_range(seed, tag, 0, m * n, out);
}

/* ------------------------------------------------------------ products --- */

/* C (m x n) = A (m x kk) * B (kk x n); dense.cpp:102-113 order. */
static void mm_nn(const double *a, i64 m, i64 kk, const double *b, i64 n, double *c) {
    memset(c, 0, sizeof(double) * (size_t)(m * n));
#pragma omp parallel for schedule(static) num_threads(nthreads()) if (2.0 * m * n * kk > 4e6)
    for (i64 j = 0; j < n; ++j) {
        double *cj = c + j * m;
        for (i64 l = 0; l < kk; ++l) {
            const double blj = AT(b, kk, l, j);
            if (blj == 0.0) continue;
            const double *al = a + l * m;
            for (i64 i = 0; i < m; ++i) cj[i] += blj * al[i];
        }
    }
}

/* C (m x n) = A^T * B with A kk x m, B kk x n; dense.cpp:115-126 order. */
static void mm_tn(const double *a, i64 kk, i64 m, const double *b, i64 n, double *c) {
#pragma omp parallel for schedule(static) num_threads(nthreads()) if (2.0 * m * n * kk > 4e6)
    for (i64 j = 0; j < n; ++j) {
        const double *bj = b + j * kk;
        for (i64 i = 0; i < m; ++i) {
            const double *ai = a + i * kk;
            double s = 0.0;
            for (i64 l = 0; l < kk; ++l) s += ai[l] * bj[l];
            AT(c, m, i, j) = s;
        }
    }
}

/* C (m x n) = A * B^T with A m x kk, B n x kk; dense.cpp:128-138 order. */
static void mm_nt(const double *a, i64 m, i64 kk, const double *b, i64 n, double *c) {
    memset(c, 0, sizeof(double) * (size_t)(m * n));
    /* loop order l-outer, j-inner per column block; each c(:,j) still sees
     * l ascending, so partitioning j across threads keeps the bits. */
#pragma omp parallel num_threads(nthreads()) if (2.0 * m * n * kk > 4e6)
    {
        i64 j0 = 0, j1 = n;
#ifdef _OPENMP
        const int nt = omp_get_num_threads(), t = omp_get_thread_num();
        j0 = n * t / nt;
        j1 = n * (t + 1) / nt;
#endif
        for (i64 l = 0; l < kk; ++l) {
            const double *al = a + l * m;
            for (i64 j = j0; j < j1; ++j) {
                const double bjl = AT(b, n, j, l);
                if (bjl == 0.0) continue;
                double *cj = c + j * m;
                for (i64 i = 0; i < m; ++i) cj[i] += bjl * al[i];
            }
        }
    }
}

int rfo_multiply(const double *a, i64 am, i64 an, const double *b, i64 bm, i64 bn, int ta, int tb,
                 double *c) {
    const i64 m = ta ? an : am, ak = ta ? am : an, bk = tb ? bn : bm, n = tb ? bm : bn;
    if (ak != bk) return fail(E_PARAM, "multiply: inner dimensions disagree");
    if (m == 0 || n == 0) return OK;
    if (ak == 0) {
        memset(c, 0, sizeof(double) * (size_t)(m * n));
        return OK;
    }
    if (!ta && !tb) mm_nn(a, m, ak, b, n, c);
    else if (ta && !tb) mm_tn(a, ak, m, b, n, c);
    else if (!ta && tb) mm_nt(a, m, ak, b, n, c);
    else return fail(E_PARAM, "multiply: tt mode not restated");
    return OK;
}

static double sumsq(const double *x, i64 n) {
    double s = 0.0;
    for (i64 i = 0; i < n; ++i) s += x[i] * x[i];
    return s;
}

double rfo_frob(const double *a, i64 count) { return sqrt(sumsq(a, count)); }

static void transpose(const double *a, i64 m, i64 n, double *t) {
    for (i64 j = 0; j < n; ++j)
        for (i64 i = 0; i < m; ++i) AT(t, n, j, i) = AT(a, m, i, j);
}

/* -------------------------------------------------------------- orth --- */

/* Two-pass MGS with column dropping at 1e-13 ||X||_F (dense.cpp:402-431).
 * q must hold m*n; returns kept column count through *r_out. */
int rfo_orth(const double *x, i64 m, i64 n, double *q, i64 *r_out) {
    const double drop = 1e-13 * rfo_frob(x, m * n);
    double *v = dalloc(m);
    if (!v) return fail(E_NOMEM, "orth: allocation");
    i64 r = 0;
    for (i64 j = 0; j < n; ++j) {
        memcpy(v, x + j * m, sizeof(double) * (size_t)m);
        for (int pass = 0; pass < 2; ++pass) {
            for (i64 c = 0; c < r; ++c) {
                const double *qc = q + c * m;
                double dot = 0.0;
                for (i64 i = 0; i < m; ++i) dot += qc[i] * v[i];
                for (i64 i = 0; i < m; ++i) v[i] -= dot * qc[i];
            }
        }
        const double nrm = sqrt(sumsq(v, m));
        if (nrm > drop && nrm > 0.0) {
            double *qr = q + r * m;
            for (i64 i = 0; i < m; ++i) qr[i] = v[i] / nrm;
            ++r;
        }
    }
    free(v);
    *r_out = r;
    return OK;
}

/* --------------------------------------------------------- reflectors --- */

typedef struct {
    double beta, result;
} refl_t;

/* make_reflector (dense.cpp:328-357): tail written to tail[0..len-1). */
static refl_t make_refl(const double *x, i64 len, double *tail) {
    refl_t h = {0.0, 0.0};
    if (len == 0) return h;
    const double alpha = x[0];
    double sigma = 0.0;
    for (i64 i = 1; i < len; ++i) sigma += x[i] * x[i];
    for (i64 i = 0; i + 1 < len; ++i) tail[i] = 0.0;
    if (sigma == 0.0) {
        if (alpha >= 0.0) {
            h.beta = 0.0;
            h.result = alpha;
        } else {
            h.beta = 2.0;
            h.result = -alpha;
        }
        return h;
    }
    const double mu = sqrt(alpha * alpha + sigma);
    const double v0 = (alpha <= 0.0) ? alpha - mu : -sigma / (alpha + mu);
    h.beta = 2.0 * v0 * v0 / (sigma + v0 * v0);
    for (i64 i = 1; i < len; ++i) tail[i - 1] = x[i] / v0;
    h.result = mu;
    return h;
}

/* apply_reflector (dense.cpp:359-371) to columns [c0,c1) of W (ld = ldw). */
static void apply_refl(double *w, i64 ldw, i64 r0, i64 len, i64 c0, i64 c1, const double *tail,
                       double beta) {
    if (beta == 0.0) return;
    for (i64 j = c0; j < c1; ++j) {
        double *col = w + j * ldw + r0;
        double dot = col[0];
        for (i64 i = 1; i < len; ++i) dot += tail[i - 1] * col[i];
        const double bd = beta * dot;
        col[0] -= bd;
        for (i64 i = 1; i < len; ++i) col[i] -= bd * tail[i - 1];
    }
}

/* Q factor (m x min(m,n)) of householder_qr (dense.cpp:375-400). */
static int hqr_q(const double *a, i64 m, i64 n, double *q) {
    const i64 r = m < n ? m : n;
    double *w = dalloc(m * n), *tails = dalloc(r * m), *betas = dalloc(r);
    if (!w || !tails || !betas) return fail(E_NOMEM, "householder_qr: allocation");
    memcpy(w, a, sizeof(double) * (size_t)(m * n));
    for (i64 j = 0; j < r; ++j) {
        double *tail = tails + j * m;
        refl_t h = make_refl(w + j * m + j, m - j, tail);
        apply_refl(w, m, j, m - j, j + 1, n, tail, h.beta);
        AT(w, m, j, j) = h.result;
        for (i64 i = j + 1; i < m; ++i) AT(w, m, i, j) = 0.0;
        betas[j] = h.beta;
    }
    memset(q, 0, sizeof(double) * (size_t)(m * r));
    for (i64 i = 0; i < r; ++i) AT(q, m, i, i) = 1.0;
    for (i64 j = r - 1; j >= 0; --j) apply_refl(q, m, j, m - j, 0, r, tails + j * m, betas[j]);
    free(w);
    free(tails);
    free(betas);
    return OK;
}

/* planted_matrix (diagnostics.cpp:124-136): A = (U diag(s)) V^T. */
int rfo_planted(i64 m, i64 n, const double *sigma, i64 r, uint64_t seed, double *a) {
    if (r > (m < n ? m : n)) return fail(E_PARAM, "planted_matrix: spectrum longer than min(m,n)");
    double *g = dalloc((m > n ? m : n) * r), *u = dalloc(m * r), *v = dalloc(n * r);
    if (!g || !u || !v) return fail(E_NOMEM, "planted: allocation");
    rfo_gaussian(seed, "testmat.u", m, r, g);
    int st = hqr_q(g, m, r, u);
    if (st == OK) {
        rfo_gaussian(seed, "testmat.v", n, r, g);
        st = hqr_q(g, n, r, v);
    }
    if (st == OK) {
        for (i64 j = 0; j < r; ++j)
            for (i64 i = 0; i < m; ++i) AT(u, m, i, j) *= sigma[j];
        mm_nt(u, m, r, v, n, a);
    }
    free(g);
    free(u);
    free(v);
    return st;
}

/* ---------------------------------------------------------------- cpqr --- */

/* cpqr with CpqrStop::rank(k) (dense.cpp:453-552). perm n, R rank x n
 * (ld = k, caller allocates k*n), *rank_out = stopped rank. */
int rfo_cpqr_rank(const double *a, i64 m, i64 n, i64 k, i64 *perm, double *r_out, i64 *rank_out) {
    const i64 rmax = m < n ? m : n;
    if (k < 0 || k > rmax) return fail(E_PARAM, "cpqr: rank target out of range");
    double *w = dalloc(m * n), *nrm = dalloc(n), *nrm0 = dalloc(n), *tail = dalloc(m);
    if (!w || !nrm || !nrm0 || !tail) return fail(E_NOMEM, "cpqr: allocation");
    memcpy(w, a, sizeof(double) * (size_t)(m * n));
    for (i64 j = 0; j < n; ++j) {
        perm[j] = j;
        double s = 0.0;
        for (i64 i = 0; i < m; ++i) s += AT(w, m, i, j) * AT(w, m, i, j);
        nrm[j] = s;
        nrm0[j] = s;
    }
    const double halt = 1e-14 * rfo_frob(a, m * n);
    i64 r = 0;
    while (r < rmax && r < k) {
        i64 piv = r;
        double best = -1.0;
        for (i64 c = r; c < n; ++c)
            if (nrm[c] > best) {
                best = nrm[c];
                piv = c;
            }
        if (best <= 0.0 || best < 1e-8 * nrm0[piv]) {
            for (i64 c = r; c < n; ++c) {
                double s = 0.0;
                for (i64 i = r; i < m; ++i) s += AT(w, m, i, c) * AT(w, m, i, c);
                nrm[c] = s;
            }
            piv = r;
            best = -1.0;
            for (i64 c = r; c < n; ++c)
                if (nrm[c] > best) {
                    best = nrm[c];
                    piv = c;
                }
        }
        if (sqrt(best > 0.0 ? best : 0.0) < halt) break;
        if (piv != r) {
            for (i64 i = 0; i < m; ++i) {
                const double t = AT(w, m, i, r);
                AT(w, m, i, r) = AT(w, m, i, piv);
                AT(w, m, i, piv) = t;
            }
            i64 tp = perm[r];
            perm[r] = perm[piv];
            perm[piv] = tp;
            double t = nrm[r];
            nrm[r] = nrm[piv];
            nrm[piv] = t;
            t = nrm0[r];
            nrm0[r] = nrm0[piv];
            nrm0[piv] = t;
        }
        refl_t h = make_refl(w + r * m + r, m - r, tail);
        apply_refl(w, m, r, m - r, r + 1, n, tail, h.beta);
        AT(w, m, r, r) = h.result;
        for (i64 i = r + 1; i < m; ++i) AT(w, m, i, r) = 0.0;
        for (i64 c = r + 1; c < n; ++c) nrm[c] -= AT(w, m, r, c) * AT(w, m, r, c);
        ++r;
    }
    for (i64 j = 0; j < n; ++j)
        for (i64 i = 0; i < k; ++i) AT(r_out, k, i, j) = (i < r && i <= j) ? AT(w, m, i, j) : 0.0;
    *rank_out = r;
    free(w);
    free(nrm);
    free(nrm0);
    free(tail);
    return OK;
}

/* --------------------------------------------------------------- svd --- */

static int cmp_desc_stable_keys(const double *key, i64 x, i64 y) {
    /* strict "key[x] > key[y]" comparator used by std::stable_sort */
    return key[x] > key[y];
}

/* stable merge sort of idx[0..n) by descending key (std::stable_sort with
 * comparator key[x] > key[y]). */
static void stable_sort_desc(i64 *idx, i64 n, const double *key, i64 *tmp) {
    for (i64 width = 1; width < n; width *= 2) {
        for (i64 lo = 0; lo < n; lo += 2 * width) {
            i64 mid = lo + width < n ? lo + width : n, hi = lo + 2 * width < n ? lo + 2 * width : n;
            i64 i = lo, j = mid, o = lo;
            while (i < mid && j < hi) {
                if (cmp_desc_stable_keys(key, idx[j], idx[i])) tmp[o++] = idx[j++];
                else tmp[o++] = idx[i++];
            }
            while (i < mid) tmp[o++] = idx[i++];
            while (j < hi) tmp[o++] = idx[j++];
        }
        memcpy(idx, tmp, sizeof(i64) * (size_t)n);
    }
}

/* fill_orthonormal_completion (dense.cpp:560-583). */
static void complete_cols(double *u, i64 m, i64 have, i64 want) {
    double *v = dalloc(m), *best = dalloc(m);
    for (i64 next = have; next < want; ++next) {
        double best_norm = -1.0;
        for (i64 cand = 0; cand < m; ++cand) {
            memset(v, 0, sizeof(double) * (size_t)m);
            v[cand] = 1.0;
            for (int pass = 0; pass < 2; ++pass)
                for (i64 c = 0; c < next; ++c) {
                    double dot = 0.0;
                    for (i64 i = 0; i < m; ++i) dot += AT(u, m, i, c) * v[i];
                    for (i64 i = 0; i < m; ++i) v[i] -= dot * AT(u, m, i, c);
                }
            const double nv = sqrt(sumsq(v, m));
            if (nv > best_norm) {
                best_norm = nv;
                memcpy(best, v, sizeof(double) * (size_t)m);
            }
        }
        for (i64 i = 0; i < m; ++i) AT(u, m, i, next) = best[i] / best_norm;
    }
    free(v);
    free(best);
}

/* svd_tall (dense.cpp:585-686): one-sided Jacobi on m x n (m >= n).
 * U m x n, D n, V n x n. */
static int svd_tall(const double *a, i64 m, i64 n, double *U, double *D, double *V) {
    double *w = dalloc(m * n), *v = dalloc(n * n), *w2 = dalloc(m * n), *v2 = dalloc(n * n);
    double *key = dalloc(n);
    i64 *ord = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    i64 *tmp = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    if (!w || !v || !w2 || !v2 || !key || !ord || !tmp) return fail(E_NOMEM, "svd: allocation");
    memcpy(w, a, sizeof(double) * (size_t)(m * n));
    for (i64 i = 0; i < n; ++i) AT(v, n, i, i) = 1.0;
    const double tol = 1e-15;
    int converged = (n <= 1);
    for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
        for (i64 j = 0; j < n; ++j) {
            key[j] = sumsq(w + j * m, m);
            ord[j] = j;
        }
        stable_sort_desc(ord, n, key, tmp);
        for (i64 j = 0; j < n; ++j) {
            memcpy(w2 + j * m, w + ord[j] * m, sizeof(double) * (size_t)m);
            memcpy(v2 + j * n, v + ord[j] * n, sizeof(double) * (size_t)n);
        }
        double *t = w;
        w = w2;
        w2 = t;
        t = v;
        v = v2;
        v2 = t;
        converged = 1;
        for (i64 p = 0; p + 1 < n; ++p) {
            for (i64 q = p + 1; q < n; ++q) {
                double *wp = w + p * m, *wq = w + q * m;
                double app = 0.0, aqq = 0.0, apq = 0.0;
                for (i64 i = 0; i < m; ++i) {
                    app += wp[i] * wp[i];
                    aqq += wq[i] * wq[i];
                    apq += wp[i] * wq[i];
                }
                if (app == 0.0 || aqq == 0.0) continue;
                if (fabs(apq) <= tol * sqrt(app * aqq)) continue;
                converged = 0;
                const double zeta = (aqq - app) / (2.0 * apq);
                const double tt = (zeta < 0.0 ? -1.0 : 1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + tt * tt);
                const double sn = cs * tt;
                for (i64 i = 0; i < m; ++i) {
                    const double xp = wp[i], xq = wq[i];
                    wp[i] = cs * xp - sn * xq;
                    wq[i] = sn * xp + cs * xq;
                }
                double *vp = v + p * n, *vq = v + q * n;
                for (i64 i = 0; i < n; ++i) {
                    const double xp = vp[i], xq = vq[i];
                    vp[i] = cs * xp - sn * xq;
                    vq[i] = sn * xp + cs * xq;
                }
            }
        }
    }
    int st = OK;
    if (!converged) {
        st = fail(E_CONV, "svd_dense: Jacobi sweeps did not converge");
    } else {
        for (i64 j = 0; j < n; ++j) {
            key[j] = sqrt(sumsq(w + j * m, m));
            ord[j] = j;
        }
        stable_sort_desc(ord, n, key, tmp);
        memset(U, 0, sizeof(double) * (size_t)(m * n));
        const double smax = key[ord[0]];
        i64 filled = 0;
        for (i64 j = 0; j < n; ++j) {
            const i64 src = ord[j];
            const double s = key[src];
            D[j] = s;
            memcpy(V + j * n, v + src * n, sizeof(double) * (size_t)n);
            if (s > 0.0 && s > smax * 1e-250) {
                for (i64 i = 0; i < m; ++i) AT(U, m, i, j) = AT(w, m, i, src) / s;
                filled = j + 1;
            } else {
                D[j] = 0.0;
            }
        }
        if (filled < n) complete_cols(U, m, filled, n);
    }
    free(w);
    free(v);
    free(w2);
    free(v2);
    free(key);
    free(ord);
    free(tmp);
    return st;
}

/* svd_dense (dense.cpp:690-701): U m x r, D r, V n x r, r = min(m, n). */
int rfo_svd(const double *a, i64 m, i64 n, double *U, double *D, double *V) {
    if (m == 0 || n == 0) return OK;
    if (m >= n) return svd_tall(a, m, n, U, D, V);
    double *t = dalloc(m * n);
    if (!t) return fail(E_NOMEM, "svd: allocation");
    transpose(a, m, n, t);
    const int st = svd_tall(t, n, m, V, D, U); /* swap roles: U <-> V */
    free(t);
    return st;
}

/* solve_upper (dense.cpp:788-804): X = R^-1 B, R n x n (ld ldr), B n x nb. */
static int solve_upper(const double *r, i64 ldr, i64 n, const double *b, i64 nb, double *x) {
    for (i64 i = 0; i < n; ++i)
        if (AT(r, ldr, i, i) == 0.0) return fail(E_NUM, "solve_upper: singular triangular factor");
    memcpy(x, b, sizeof(double) * (size_t)(n * nb));
#pragma omp parallel for schedule(static) num_threads(nthreads()) if (n * n * nb > 4000000)
    for (i64 col = 0; col < nb; ++col) {
        double *xc = x + col * n;
        for (i64 i = n - 1; i >= 0; --i) {
            double s = xc[i];
            for (i64 j = i + 1; j < n; ++j) s -= AT(r, ldr, i, j) * xc[j];
            xc[i] = s / AT(r, ldr, i, i);
        }
    }
    return OK;
}

/* least_squares (dense.cpp:825-837): X (n x nb) = pinv(M) B, M m x n. */
static int least_squares(const double *mm, i64 m, i64 n, const double *b, i64 nb, double *x) {
    const i64 r = m < n ? m : n;
    double *U = dalloc(m * r), *D = dalloc(r), *V = dalloc(n * r), *ub = dalloc(r * nb);
    if (!U || !D || !V || !ub) return fail(E_NOMEM, "least_squares: allocation");
    int st = rfo_svd(mm, m, n, U, D, V);
    if (st == OK) {
        const double cutoff = (r > 0 ? D[0] : 0.0) * 1e-12;
        mm_tn(U, m, r, b, nb, ub);
        for (i64 i = 0; i < r; ++i) {
            const double d = D[i];
            const double inv = (d > cutoff && d > 0.0) ? 1.0 / d : 0.0;
            for (i64 j = 0; j < nb; ++j) AT(ub, r, i, j) *= inv;
        }
        mm_nn(V, n, r, ub, nb, x);
    }
    free(U);
    free(D);
    free(V);
    free(ub);
    return st;
}

/* -------------------------------------------------------- range finder --- */

static int check_sample(i64 m, i64 n, i64 k, i64 p) {
    if (k < 1) return fail(E_PARAM, "k must be at least 1");
    if (p < 0) return fail(E_PARAM, "p must be non-negative");
    if (k + p > (m < n ? m : n)) return fail(E_PARAM, "k + p exceeds min(m, n)");
    return OK;
}

/* frob_residual (rangefinder.cpp:45-54). */
int rfo_frob_residual(double a_frob, const double *b, i64 count, double *out) {
    if (!(a_frob >= 0.0)) return fail(E_PARAM, "frob_residual: norm must be non-negative");
    const double bn = rfo_frob(b, count);
    if (bn > a_frob * (1.0 + 1e-8))
        return fail(E_NUM, "frob_residual: projection exceeds the total norm");
    const double diff = a_frob * a_frob - bn * bn;
    *out = sqrt(diff > 0.0 ? diff : 0.0);
    return OK;
}

/* power_range / basic_range (rangefinder.cpp:56-80). Q m x ell' (caller
 * allocates m*(k+p)), B ell' x n (caller allocates (k+p)*n). */
int rfo_power_range(const double *a, i64 m, i64 n, i64 k, i64 p, i64 q, int reorth, uint64_t seed,
                    int basic, double *Q, double *B, double *resid, i64 *ell_out) {
    if (basic && q != 0) return fail(E_PARAM, "basic_range: q must be 0 (use power_range)");
    if (q < 0) return fail(E_PARAM, "power_range: q must be non-negative");
    int st = check_sample(m, n, k, p);
    if (st) return st;
    const i64 ell = k + p;
    double *g = dalloc(n * ell), *y = dalloc(m * ell), *z = dalloc(n * ell), *w = dalloc(n * ell);
    if (!g || !y || !z || !w) return fail(E_NOMEM, "power_range: allocation");
    rfo_gaussian(seed, "range.G", n, ell, g);
    i64 r = 0;
    if (!reorth) {
        mm_nn(a, m, n, g, ell, y);
        for (i64 j = 0; j < q; ++j) {
            mm_tn(a, m, n, y, ell, z);
            mm_nn(a, m, n, z, ell, y);
        }
        st = rfo_orth(y, m, ell, Q, &r);
    } else {
        mm_nn(a, m, n, g, ell, y);
        st = rfo_orth(y, m, ell, Q, &r);
        for (i64 j = 0; j < q && st == OK; ++j) {
            i64 rw = 0;
            mm_tn(a, m, n, Q, r, z);
            st = rfo_orth(z, n, r, w, &rw);
            if (st) break;
            mm_nn(a, m, n, w, rw, y);
            st = rfo_orth(y, m, rw, Q, &r);
        }
    }
    if (st == OK) {
        /* finish_with_projection: B = Q^T A (kernel_tn, r x n) */
        mm_tn(Q, m, r, a, n, B);
        st = rfo_frob_residual(rfo_frob(a, m * n), B, r * n, resid);
        *ell_out = r;
    }
    free(g);
    free(y);
    free(z);
    free(w);
    return st;
}

/* rsvd (lowrank.cpp:74-96). U m x keep, D keep, V n x keep (caller allocates
 * with keep <= k+p). */
int rfo_rsvd(const double *a, i64 m, i64 n, i64 k, i64 p, i64 q, uint64_t seed, int keep_over,
             int reorth, double *U, double *D, double *V, i64 *rank_out) {
    int st = check_sample(m, n, k, p);
    if (st) return st;
    if (q < 0) return fail(E_PARAM, "power_range: q must be non-negative");
    const i64 ell = k + p;
    double *Q = dalloc(m * ell), *B = dalloc(ell * n);
    double resid = 0.0;
    i64 r = 0;
    if (!Q || !B) return fail(E_NOMEM, "rsvd: allocation");
    st = rfo_power_range(a, m, n, k, p, q, reorth, seed, 0, Q, B, &resid, &r);
    *rank_out = 0;
    if (st == OK && r > 0) {
        /* svd_dense(B), B r x n with r <= n: via svd_tall(B^T) */
        const i64 rr = r < n ? r : n;
        double *su = dalloc(r * rr), *sd = dalloc(rr), *sv = dalloc(n * rr);
        st = rfo_svd(B, r, n, su, sd, sv);
        if (st == OK) {
            const i64 keep = keep_over ? rr : (k < rr ? k : rr);
            mm_nn(Q, m, r, su, keep, U); /* U = Q * small.U(:, :keep) */
            memcpy(V, sv, sizeof(double) * (size_t)(n * keep));
            memcpy(D, sd, sizeof(double) * (size_t)keep);
            *rank_out = keep;
        }
        free(su);
        free(sd);
        free(sv);
    }
    free(Q);
    free(B);
    return st;
}

/* ------------------------------------------------------------------ ID --- */

/* col_id_core (lowrank.cpp:51-70): Js ke, Z ke x n (caller allocates k*n). */
int rfo_col_id(const double *a, i64 m, i64 n, i64 k, i64 *js, double *z, i64 *rank_out,
               int *truncated) {
    i64 *perm = (i64 *)malloc(sizeof(i64) * (size_t)(n > 0 ? n : 1));
    double *R = dalloc(k * n);
    if (!perm || !R) return fail(E_NOMEM, "col_id: allocation");
    i64 r = 0;
    int st = rfo_cpqr_rank(a, m, n, k, perm, R, &r);
    if (st == OK) {
        const i64 ke = k < r ? k : r;
        *truncated = ke < k;
        *rank_out = ke;
        for (i64 j = 0; j < ke; ++j) js[j] = perm[j];
        memset(z, 0, sizeof(double) * (size_t)(ke * n));
        for (i64 j = 0; j < ke; ++j) AT(z, ke, j, perm[j]) = 1.0;
        if (ke > 0 && n > ke) {
            double *s12 = dalloc(ke * (n - ke)), *t = dalloc(ke * (n - ke)), *s11 = dalloc(ke * ke);
            for (i64 j = 0; j < ke; ++j)
                for (i64 i = 0; i < ke; ++i) AT(s11, ke, i, j) = AT(R, k, i, j);
            for (i64 j = 0; j < n - ke; ++j)
                for (i64 i = 0; i < ke; ++i) AT(s12, ke, i, j) = AT(R, k, i, ke + j);
            st = solve_upper(s11, ke, ke, s12, n - ke, t);
            if (st == OK)
                for (i64 j = 0; j < n - ke; ++j)
                    for (i64 i = 0; i < ke; ++i) AT(z, ke, i, perm[ke + j]) = AT(t, ke, i, j);
            free(s12);
            free(t);
            free(s11);
        }
    }
    free(perm);
    free(R);
    return st;
}

/* randomized_id (lowrank.cpp:312-329): Is ke, X m x ke. */
int rfo_randomized_id(const double *a, i64 m, i64 n, i64 k, i64 p, i64 q, uint64_t seed, i64 *is,
                      double *x, i64 *rank_out, int *truncated) {
    int st = check_sample(m, n, k, p);
    if (st) return st;
    if (q < 0) return fail(E_PARAM, "randomized_id: q must be non-negative");
    const i64 ell = k + p;
    double *g = dalloc(n * ell), *y = dalloc(m * ell), *zz = dalloc(n * ell), *yt = dalloc(m * ell);
    double *z = dalloc(k * m);
    rfo_gaussian(seed, "rid.G", n, ell, g);
    mm_nn(a, m, n, g, ell, y);
    for (i64 t = 0; t < q; ++t) {
        mm_tn(a, m, n, y, ell, zz);
        mm_nn(a, m, n, zz, ell, y);
    }
    transpose(y, m, ell, yt);
    i64 ke = 0;
    st = rfo_col_id(yt, ell, m, k, is, z, &ke, truncated);
    if (st == OK) {
        transpose(z, ke, m, x);
        *rank_out = ke;
    }
    free(g);
    free(y);
    free(zz);
    free(yt);
    free(z);
    return st;
}

/* Column-ID part of randomized_cur (lowrank.cpp:351-357): Y = G A with
 * G = gaussian(seed, "cur.G", k+p, m), then col_id_core(Y, k).
 * Y_out (optional) receives the (k+p) x n sketch. */
int rfo_cur_col_id(const double *a, i64 m, i64 n, i64 k, i64 p, uint64_t seed, i64 *js, double *z,
                   i64 *rank_out, int *truncated, double *y_out) {
    int st = check_sample(m, n, k, p);
    if (st) return st;
    const i64 ell = k + p;
    double *g = dalloc(ell * m), *y = dalloc(ell * n);
    rfo_gaussian(seed, "cur.G", ell, m, g);
    mm_nn(g, ell, m, a, n, y);
    if (y_out) memcpy(y_out, y, sizeof(double) * (size_t)(ell * n));
    st = rfo_col_id(y, ell, n, k, js, z, rank_out, truncated);
    free(g);
    free(y);
    return st;
}

static double cond_number(const double *a, i64 m, i64 n) {
    const i64 r = m < n ? m : n;
    double *U = dalloc(m * r), *D = dalloc(r), *V = dalloc(n * r);
    double c = INFINITY;
    if (rfo_svd(a, m, n, U, D, V) == OK && r > 0 && D[r - 1] > 0.0) c = D[0] / D[r - 1];
    free(U);
    free(D);
    free(V);
    return c;
}

/* randomized_cur (lowrank.cpp:348-372), q = 0 only. U kc x kr. */
int rfo_randomized_cur(const double *a, i64 m, i64 n, i64 k, i64 p, uint64_t seed, i64 *js, i64 *is,
                       double *u, double *cond_c, double *cond_r, int *warning, i64 *kc_out,
                       i64 *kr_out) {
    double *z = dalloc(k * n);
    i64 kc = 0;
    int trunc = 0;
    int st = rfo_cur_col_id(a, m, n, k, p, seed, js, z, &kc, &trunc, NULL);
    if (st) {
        free(z);
        return st;
    }
    double *c = dalloc(m * kc), *ct = dalloc(kc * m), *zr = dalloc(kc * m);
    for (i64 j = 0; j < kc; ++j) memcpy(c + j * m, a + js[j] * m, sizeof(double) * (size_t)m);
    transpose(c, m, kc, ct);
    i64 kr = 0;
    st = rfo_col_id(ct, kc, m, kc, is, zr, &kr, &trunc);
    if (st == OK) {
        /* R = A(Is, :) kr x n; U = (lsq(R^T, Z^T))^T */
        double *rr = dalloc(kr * n), *rt = dalloc(n * kr), *zt = dalloc(n * kc), *x = dalloc(kr * kc);
        for (i64 i = 0; i < kr; ++i)
            for (i64 j = 0; j < n; ++j) AT(rr, kr, i, j) = AT(a, m, is[i], j);
        transpose(rr, kr, n, rt);
        transpose(z, kc, n, zt);
        st = least_squares(rt, n, kr, zt, kc, x);
        if (st == OK) {
            transpose(x, kr, kc, u);
            *cond_c = cond_number(c, m, kc);
            *cond_r = cond_number(rr, kr, n);
            *warning = *cond_c > 1e8 || *cond_r > 1e8;
            *kc_out = kc;
            *kr_out = kr;
        }
        free(rr);
        free(rt);
        free(zt);
        free(x);
    }
    free(z);
    free(c);
    free(ct);
    free(zr);
    return st;
}

/* ---------------------------------------------------------- single pass --- */

/* Cyclic two-sided Jacobi eigendecomposition of a symmetric n x n matrix
 * (restated from dense.cpp:703-761 without the final sort). */
static int eig_sym(double *s, i64 n, double *v, double *lam) {
    memset(v, 0, sizeof(double) * (size_t)(n * n));
    for (i64 i = 0; i < n; ++i) AT(v, n, i, i) = 1.0;
    const double scale = rfo_frob(s, n * n);
    int converged = (n <= 1) || scale == 0.0;
    for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
        converged = 1;
        for (i64 p = 0; p + 1 < n; ++p)
            for (i64 q = p + 1; q < n; ++q) {
                const double spq = AT(s, n, p, q);
                if (fabs(spq) <= 1e-15 * scale) continue;
                converged = 0;
                const double tau = (AT(s, n, q, q) - AT(s, n, p, p)) / (2.0 * spq);
                const double t = (tau < 0.0 ? -1.0 : 1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                const double c = 1.0 / sqrt(1.0 + t * t), sn = t * c;
                for (i64 i = 0; i < n; ++i) {
                    const double xp = AT(s, n, i, p), xq = AT(s, n, i, q);
                    AT(s, n, i, p) = c * xp - sn * xq;
                    AT(s, n, i, q) = sn * xp + c * xq;
                }
                for (i64 i = 0; i < n; ++i) {
                    const double xp = AT(s, n, p, i), xq = AT(s, n, q, i);
                    AT(s, n, p, i) = c * xp - sn * xq;
                    AT(s, n, q, i) = sn * xp + c * xq;
                }
                AT(s, n, p, q) = 0.0;
                AT(s, n, q, p) = 0.0;
                for (i64 i = 0; i < n; ++i) {
                    const double xp = AT(v, n, i, p), xq = AT(v, n, i, q);
                    AT(v, n, i, p) = c * xp - sn * xq;
                    AT(v, n, i, q) = sn * xp + c * xq;
                }
            }
    }
    for (i64 i = 0; i < n; ++i) lam[i] = AT(s, n, i, i);
    return converged ? OK : fail(E_CONV, "eig_sym: Jacobi sweeps did not converge");
}

/* The dual sketch of single_pass_svd (lowrank.cpp:170-176) with stream block
 * width b: Yc = sum over blocks of (A_blk Gc_blk) accumulated by add(), and
 * Yr(blk rows) = A_blk^T Gr. */
int rfo_dual_sketch(const double *a, i64 m, i64 n, const double *gc, const double *gr, i64 ell,
                    i64 b, double *yc, double *yr) {
    if (b < 1) return fail(E_PARAM, "MatrixStream: block width must be positive");
    double *prod = dalloc(m * ell), *gpart = dalloc(b * ell), *tr = dalloc(b * ell);
    memset(yc, 0, sizeof(double) * (size_t)(m * ell));
    for (i64 c0 = 0; c0 < n; c0 += b) {
        const i64 w = (c0 + b <= n) ? b : n - c0;
        for (i64 j = 0; j < ell; ++j)
            for (i64 i = 0; i < w; ++i) AT(gpart, w, i, j) = AT(gc, n, c0 + i, j);
        mm_nn(a + c0 * m, m, w, gpart, ell, prod);
        for (i64 t = 0; t < m * ell; ++t) yc[t] = yc[t] + prod[t];
        mm_tn(a + c0 * m, m, w, gr, ell, tr); /* w x ell */
        for (i64 j = 0; j < ell; ++j)
            for (i64 i = 0; i < w; ++i) AT(yr, n, c0 + i, j) = AT(tr, w, i, j);
    }
    free(prod);
    free(gpart);
    free(tr);
    return OK;
}

/* single_pass_svd restated: reference sketch + dominant_left + the
 * normal-equation (Sylvester) core P^T P C + C W W^T = P^T E + F W^T solved in
 * the eigenbases of P^T P and W W^T, then svd_dense(C) and the lift.
 * U m x kk, D kk, V n x kk. */
int rfo_single_pass_svd(const double *a, i64 m, i64 n, i64 k, i64 p, uint64_t seed, i64 block,
                        double *U, double *D, double *V, i64 *rank_out) {
    int st = check_sample(m, n, k, p);
    if (st) return st;
    const i64 ell = k + p;
    double *gc = dalloc(n * ell), *gr = dalloc(m * ell), *yc = dalloc(m * ell), *yr = dalloc(n * ell);
    rfo_gaussian(seed, "spsvd.Gc", n, ell, gc);
    rfo_gaussian(seed, "spsvd.Gr", m, ell, gr);
    st = rfo_dual_sketch(a, m, n, gc, gr, ell, block, yc, yr);
    double *uc = dalloc(m * ell), *dc = dalloc(ell), *vc = dalloc(ell * ell);
    double *ur = dalloc(n * ell), *dr = dalloc(ell), *vr = dalloc(ell * ell);
    if (st == OK) st = rfo_svd(yc, m, ell, uc, dc, vc);
    if (st == OK) st = rfo_svd(yr, n, ell, ur, dr, vr);
    if (st == OK) {
        const i64 kk = k < ell ? k : ell; /* dominant_left keeps min(k, ell) */
        /* qck = uc(:, :kk), qrk = ur(:, :kk) (leading columns, contiguous) */
        double *P = dalloc(ell * kk), *E = dalloc(ell * kk), *W = dalloc(kk * ell), *F = dalloc(kk * ell);
        mm_tn(gr, m, ell, uc, kk, P);   /* ell x kk */
        mm_tn(yr, n, ell, ur, kk, E);   /* ell x kk */
        mm_tn(ur, n, kk, gc, ell, W);   /* kk x ell */
        mm_tn(uc, m, kk, yc, ell, F);   /* kk x ell */
        double *ptp = dalloc(kk * kk), *wwt = dalloc(kk * kk), *rhs = dalloc(kk * kk), *tmp = dalloc(kk * kk);
        double *wt = dalloc(ell * kk);
        mm_tn(P, ell, kk, P, kk, ptp);
        transpose(W, kk, ell, wt);
        mm_tn(wt, ell, kk, wt, kk, wwt);
        mm_tn(P, ell, kk, E, kk, rhs);
        mm_nn(F, kk, ell, wt, kk, tmp);
        for (i64 t = 0; t < kk * kk; ++t) rhs[t] += tmp[t];
        double *u1 = dalloc(kk * kk), *l1 = dalloc(kk), *u2 = dalloc(kk * kk), *l2 = dalloc(kk);
        st = eig_sym(ptp, kk, u1, l1);
        if (st == OK) st = eig_sym(wwt, kk, u2, l2);
        if (st == OK) {
            double *c = dalloc(kk * kk);
            mm_tn(u1, kk, kk, rhs, kk, tmp);    /* U1^T RHS */
            mm_nn(tmp, kk, kk, u2, kk, c);      /* (U1^T RHS) U2 */
            for (i64 j = 0; j < kk; ++j)
                for (i64 i = 0; i < kk; ++i) AT(c, kk, i, j) /= (l1[i] + l2[j]);
            mm_nn(u1, kk, kk, c, kk, tmp);      /* U1 Ct */
            mm_nt(tmp, kk, kk, u2, kk, c);      /* (U1 Ct) U2^T */
            double *cu = dalloc(kk * kk), *cv = dalloc(kk * kk);
            st = rfo_svd(c, kk, kk, cu, D, cv);
            if (st == OK) {
                mm_nn(uc, m, kk, cu, kk, U);
                mm_nn(ur, n, kk, cv, kk, V);
                *rank_out = kk;
            }
            free(c);
            free(cu);
            free(cv);
        }
        free(P);
        free(E);
        free(W);
        free(F);
        free(ptp);
        free(wwt);
        free(rhs);
        free(tmp);
        free(wt);
        free(u1);
        free(l1);
        free(u2);
        free(l2);
    }
    free(gc);
    free(gr);
    free(yc);
    free(yr);
    free(uc);
    free(dc);
    free(vc);
    free(ur);
    free(dr);
    free(vr);
    return st;
}
