/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot-path arithmetic (iluamg, the
 * CPU code under /root/reference/proj), used by tests/ and by bench.py's
 * cpu_baseline leg as the checker. The product (paper_2111_09512_b200/) never
 * links, loads or calls this file.
 *
 * Pinning: every function here is checked in tests/test_oracle.py against
 *   (a) the reference itself, compiled unmodified into oracle/_ref (bitwise:
 *       same operation order, no FMA — x86-64 baseline gcc emits none), and
 *   (b) the golden known-answer vectors restated from the reference tests
 *       (tests/golden/, see tests/golden/make_golden.py).
 *
 * Conventions follow include/iluamg/sparse.hpp:14-51: CSR with int64 row
 * starts / column indices (strictly increasing per row) and fp64 values;
 * accumulation is in ascending column order starting from 0.0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t idx;

/* src/sparse.cpp:162-174 spmv_into: y_i = sum_k a_ik x_k, ascending k, from 0.0 */
void orc_spmv(idx n, const idx* rp, const idx* ci, const double* v, const double* x, double* y) {
    for (idx i = 0; i < n; ++i) {
        double s = 0.0;
        for (idx k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

/* src/sparse.cpp:327-332 residual: r = b - spmv(A, x) */
void orc_residual(idx n, const idx* rp, const idx* ci, const double* v, const double* x,
                  const double* b, double* r) {
    for (idx i = 0; i < n; ++i) {
        double s = 0.0;
        for (idx k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        r[i] = b[i] - s;
    }
}

/* src/trisolve.cpp:94-104 richardson_lower: y0 = 0, y <- b - L_s y, m times */
void orc_richardson_lower(idx n, const idx* rp, const idx* ci, const double* v, const double* b,
                          idx m, double* y) {
    double* t = (double*)malloc((size_t)n * sizeof(double));
    for (idx i = 0; i < n; ++i) y[i] = 0.0;
    for (idx s = 0; s < m; ++s) {
        orc_spmv(n, rp, ci, v, y, t);
        for (idx i = 0; i < n; ++i) y[i] = b[i] - t[i];
    }
    free(t);
}

/* Strict part of a row (skip j == i), the split_triangular view used by
 * strict_upper_of (src/trisolve.cpp:123-128, src/sparse.cpp:302-325). */
static void strict_spmv(idx n, const idx* rp, const idx* ci, const double* v, const double* x,
                        double* y) {
    for (idx i = 0; i < n; ++i) {
        double s = 0.0;
        for (idx k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] != i) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

/* src/trisolve.cpp:110-147 richardson_upper_scaled: bs = b / rs (division),
 * x0 = 0, x <- bs - U_s x (m times) on the stored unit-diagonal U, then
 * x /= cs when a column scale is present. U holds its diagonal (ignored). */
void orc_richardson_upper_scaled(idx n, const idx* rp, const idx* ci, const double* v,
                                 const double* rs, const double* cs, const double* b, idx m,
                                 double* x) {
    double* bs = (double*)malloc((size_t)n * sizeof(double));
    double* t = (double*)malloc((size_t)n * sizeof(double));
    for (idx i = 0; i < n; ++i) bs[i] = b[i] / rs[i];
    for (idx i = 0; i < n; ++i) x[i] = 0.0;
    for (idx s = 0; s < m; ++s) {
        strict_spmv(n, rp, ci, v, x, t);
        for (idx i = 0; i < n; ++i) x[i] = bs[i] - t[i];
    }
    if (cs)
        for (idx i = 0; i < n; ++i) x[i] /= cs[i];
    free(bs);
    free(t);
}

/* North-star deviation a11b(i): Jacobi on the UNSCALED U,
 * x0 = 0, x <- D^-1 (b - N x), N = strict upper, D = diag(U). Same iteration
 * matrix as richardson_upper_scaled with row scaling; pinned to it at 1e-12. */
void orc_jacobi_upper(idx n, const idx* rp, const idx* ci, const double* v, const double* b, idx m,
                      double* x) {
    double* d = (double*)malloc((size_t)n * sizeof(double));
    double* t = (double*)malloc((size_t)n * sizeof(double));
    for (idx i = 0; i < n; ++i) {
        d[i] = 0.0;
        for (idx k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) d[i] = v[k];
        x[i] = 0.0;
    }
    for (idx s = 0; s < m; ++s) {
        strict_spmv(n, rp, ci, v, x, t);
        for (idx i = 0; i < n; ++i) x[i] = (b[i] - t[i]) / d[i];
    }
    free(d);
    free(t);
}

/* src/ilu.cpp:271-295 row_scale: d = diag(U); diag -> 1.0 exactly; off-diag *= 1.0/d.
 * Returns the first row with a zero diagonal, or -1. */
idx orc_row_scale(idx n, const idx* rp, const idx* ci, const double* v, double* vout, double* d) {
    for (idx i = 0; i < n; ++i) {
        d[i] = 0.0;
        for (idx k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) {
                d[i] = v[k];
                break;
            }
        if (d[i] == 0.0) return i;
    }
    for (idx i = 0; i < n; ++i) {
        const double inv = 1.0 / d[i];
        for (idx k = rp[i]; k < rp[i + 1]; ++k) vout[k] = ci[k] == i ? 1.0 : v[k] * inv;
    }
    return -1;
}

/* src/ilu.cpp:297-333 row_col_scale: root = sqrt|d|, dr = sign/root, dc = 1/root;
 * off-diag *= dr_i * dc_j; stores rs = sign*root, cs = root. */
idx orc_row_col_scale(idx n, const idx* rp, const idx* ci, const double* v, double* vout,
                      double* rs, double* cs) {
    double* dr = (double*)malloc((size_t)n * sizeof(double));
    double* dc = (double*)malloc((size_t)n * sizeof(double));
    for (idx i = 0; i < n; ++i) {
        double d = 0.0;
        for (idx k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) {
                d = v[k];
                break;
            }
        if (d == 0.0) {
            free(dr);
            free(dc);
            return i;
        }
        const double root = sqrt(fabs(d));
        const double sign = d < 0.0 ? -1.0 : 1.0;
        dc[i] = 1.0 / root;
        dr[i] = sign / root;
        cs[i] = root;
        rs[i] = sign * root;
    }
    for (idx i = 0; i < n; ++i)
        for (idx k = rp[i]; k < rp[i + 1]; ++k)
            vout[k] = ci[k] == i ? 1.0 : v[k] * (dr[i] * dc[ci[k]]);
    free(dr);
    free(dc);
    return -1;
}

/* src/trisolve.cpp:20-33 solve_lower_direct (unit lower, strict storage) */
void orc_solve_lower_direct(idx n, const idx* rp, const idx* ci, const double* v, const double* b,
                            double* x) {
    for (idx i = 0; i < n; ++i) {
        double s = b[i];
        for (idx k = rp[i]; k < rp[i + 1]; ++k) s -= v[k] * x[ci[k]];
        x[i] = s;
    }
}

/* src/trisolve.cpp:35-55 solve_upper_direct (stored diagonal; divide at the end).
 * Returns the first zero-diagonal row, or -1. */
idx orc_solve_upper_direct(idx n, const idx* rp, const idx* ci, const double* v, const double* b,
                           double* x) {
    for (idx i = n; i-- > 0;) {
        double s = b[i], d = 0.0;
        for (idx k = rp[i]; k < rp[i + 1]; ++k) {
            if (ci[k] == i)
                d = v[k];
            else
                s -= v[k] * x[ci[k]];
        }
        if (d == 0.0) return i;
        x[i] = s / d;
    }
    return -1;
}

/* src/smoother.cpp:113-132 gauss_seidel_sweep: x_i = (b_i - sum_{j!=i} a_ij x_j) / a_ii */
idx orc_gauss_seidel_sweep(idx n, const idx* rp, const idx* ci, const double* v, const double* b,
                           double* x) {
    for (idx i = 0; i < n; ++i) {
        double s = b[i], d = 0.0;
        for (idx k = rp[i]; k < rp[i + 1]; ++k) {
            if (ci[k] == i)
                d = v[k];
            else
                s -= v[k] * x[ci[k]];
        }
        if (d == 0.0) return i;
        x[i] = s / d;
    }
    return -1;
}

/* src/smoother.cpp:143-159 ilu_smooth_sweep, Richardson mode on scaled factors:
 * r = b - Ax; y = richardson_lower(L, r, mL); z = richardson_upper_scaled(U, y, mU); x += z.
 * direct != 0 selects solve_lower_direct + solve_upper_scaled_direct (:147-149). */
void orc_ilu_smooth_sweep(idx n, const idx* arp, const idx* aci, const double* av,
                          const idx* lrp, const idx* lci, const double* lv, const idx* urp,
                          const idx* uci, const double* uv, const double* rs, const double* cs,
                          int direct, idx mL, idx mU, const double* b, double* x) {
    double* r = (double*)malloc((size_t)n * sizeof(double));
    double* y = (double*)malloc((size_t)n * sizeof(double));
    double* z = (double*)malloc((size_t)n * sizeof(double));
    orc_residual(n, arp, aci, av, x, b, r);
    if (direct) {
        orc_solve_lower_direct(n, lrp, lci, lv, r, y);
        for (idx i = 0; i < n; ++i) r[i] = y[i] / rs[i];
        orc_solve_upper_direct(n, urp, uci, uv, r, z);
        if (cs)
            for (idx i = 0; i < n; ++i) z[i] /= cs[i];
    } else {
        orc_richardson_lower(n, lrp, lci, lv, r, mL, y);
        orc_richardson_upper_scaled(n, urp, uci, uv, rs, cs, y, mU, z);
    }
    for (idx i = 0; i < n; ++i) x[i] += z[i];
    free(r);
    free(y);
    free(z);
}

/* src/dense.cpp:8-38 DenseLu: row-major, partial pivoting (first max wins). Returns
 * the singular column or -1. */
idx orc_dense_lu(idx n, double* lu, idx* piv) {
    for (idx k = 0; k < n; ++k) {
        idx p = k;
        for (idx i = k + 1; i < n; ++i)
            if (fabs(lu[i * n + k]) > fabs(lu[p * n + k])) p = i;
        if (lu[p * n + k] == 0.0) return k;
        piv[k] = p;
        if (p != k)
            for (idx j = 0; j < n; ++j) {
                const double t = lu[p * n + j];
                lu[p * n + j] = lu[k * n + j];
                lu[k * n + j] = t;
            }
        const double pivot = lu[k * n + k];
        for (idx i = k + 1; i < n; ++i) {
            const double mlt = lu[i * n + k] / pivot;
            lu[i * n + k] = mlt;
            for (idx j = k + 1; j < n; ++j) lu[i * n + j] -= mlt * lu[k * n + j];
        }
    }
    return -1;
}

/* src/dense.cpp:40-55 DenseLu::solve */
void orc_dense_lu_solve(idx n, const double* lu, const idx* piv, const double* b, double* x) {
    for (idx i = 0; i < n; ++i) x[i] = b[i];
    for (idx k = 0; k < n; ++k) {
        const idx p = piv[k];
        if (p != k) {
            const double t = x[p];
            x[p] = x[k];
            x[k] = t;
        }
        for (idx i = k + 1; i < n; ++i) x[i] -= lu[i * n + k] * x[k];
    }
    for (idx i = n; i-- > 0;) {
        double s = x[i];
        for (idx j = i + 1; j < n; ++j) s -= lu[i * n + j] * x[j];
        x[i] = s / lu[i * n + i];
    }
}

/* Henrici departure of a triangular T: sqrt of the off-diagonal square sum
 * (src/ilu.cpp:351-366). */
double orc_departure(idx n, const idx* rp, const idx* ci, const double* v) {
    double s = 0.0;
    for (idx i = 0; i < n; ++i)
        for (idx k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] != i) s += v[k] * v[k];
    return sqrt(s);
}

/* splitmix64 hash_mix / hash_unit (include/iluamg/rng.hpp:16-27) */
static uint64_t hash_mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
double orc_hash_unit(uint64_t seed, uint64_t i) {
    const uint64_t h = hash_mix(seed ^ hash_mix(i));
    return (double)(h >> 11) * 0x1.0p-53;
}
