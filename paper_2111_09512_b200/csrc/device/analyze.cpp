// run_analyze (reference: src/driver.cpp:92-163): factor diagnostics for the
// drop-in ABI. Not a hot path (SURVEY.md §2 row 2 marks the diagnostics out of
// scope) but every reference entry point must work: the factors come from the
// host setup, the scalings from the K1 kernel, the triangular solves of the
// Hager/Higham condition estimate from the K5 level-scheduled kernels; the
// scalar reductions run on the host in the reference's order, so every
// reported number is bitwise the reference's.
#include "driver.hpp"

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <limits>

namespace ilug {

namespace {

// Henrici departure of a triangular matrix: off-diagonal square sum (src/ilu.cpp:351-366).
double departure(const Csr& T) {
    double s = 0.0;
    for (i64 i = 0; i < T.nrows; ++i)
        for (i64 k = T.rp[i]; k < T.rp[i + 1]; ++k)
            if (T.ci[k] != i) s += T.v[k] * T.v[k];
    return std::sqrt(s);
}

enum class Shape { unit_lower, upper };

// Hager/Higham 1-norm condition estimate (src/ilu.cpp:368-442) with the
// forward and adjoint triangular solves on the device.
double condition_estimate(const Csr& T, Shape shape, cudaStream_t st) {
    const i64 n = T.nrows;
    if (n == 0) return 1.0;
    if (shape == Shape::upper) {
        const Vec d = csr_diag(T);
        for (i64 i = 0; i < n; ++i)
            if (d[i] == 0.0) fail_numeric("condition_estimate: singular diagonal at row " + std::to_string(i));
    }
    const Csr Tt = csr_transpose(T);
    LevelPlan fwd, adj;
    if (shape == Shape::unit_lower) {
        fwd.build(T, LevelPlan::Kind::lower_unit, st);   // solve_lower_direct
        adj.build(Tt, LevelPlan::Kind::upper, st);       // solve_upper_unit (x = s / 1.0)
    } else {
        fwd.build(T, LevelPlan::Kind::upper, st);        // solve_upper_direct
        adj.build(Tt, LevelPlan::Kind::gauss_seidel, st); // solve_lower_explicit (no j > i entries)
    }
    DBuf<double> db(n), dx(n);
    auto solve = [&](const LevelPlan& P, const Vec& b) {
        Vec out(static_cast<size_t>(n));
        db.upload(b.data(), n, st);
        P.solve(db.p, dx.p, db.p, st);
        dx.download(out.data(), st);
        ILUG_CUDA(cudaStreamSynchronize(st));
        return out;
    };
    Vec x(static_cast<size_t>(n), 1.0 / static_cast<double>(n));
    double est = 0.0;
    i64 last_j = -1;
    for (int iter = 0; iter < 8; ++iter) {
        const Vec y = solve(fwd, x);
        double est_new = 0.0;
        for (double v : y) est_new += std::abs(v);
        if (iter > 0 && est_new <= est) break;
        est = est_new;
        Vec xi(y.size());
        for (size_t i = 0; i < y.size(); ++i) xi[i] = y[i] < 0.0 ? -1.0 : 1.0;
        const Vec z = solve(adj, xi);
        i64 j = 0;
        double zmax = -1.0, ztx = 0.0;
        for (i64 i = 0; i < n; ++i) {
            ztx += z[i] * x[i];
            const double a = std::abs(z[i]);
            if (a > zmax) zmax = a, j = i;
        }
        if (zmax <= ztx || j == last_j) break;
        last_j = j;
        std::fill(x.begin(), x.end(), 0.0);
        x[j] = 1.0;
    }
    std::vector<double> colsum(static_cast<size_t>(n), 0.0);
    for (i64 i = 0; i < n; ++i)
        for (i64 k = T.rp[i]; k < T.rp[i + 1]; ++k) colsum[T.ci[k]] += std::abs(T.v[k]);
    if (shape == Shape::unit_lower)
        for (double& c : colsum) c += 1.0;
    double t_one = 0.0;
    for (double c : colsum) t_one = std::max(t_one, c);
    return t_one * est;
}

struct Striping {
    std::vector<std::array<double, 4>> cols; // col, max, median, ratio
    i64 flagged = 0;
};

// striping_report (src/ilu.cpp:444-474): per-column max / lower median of |L|+|U| incl. L's unit diagonal.
Striping striping(const Csr& L, const Csr& U, double threshold) {
    const i64 n = U.ncols;
    std::vector<std::vector<double>> cols(static_cast<size_t>(n));
    for (const Csr* M : {&L, &U})
        for (i64 k = 0; k < M->nnz(); ++k) cols[M->ci[k]].push_back(std::abs(M->v[k]));
    for (i64 i = 0; i < L.nrows; ++i) cols[i].push_back(1.0);
    Striping s;
    for (i64 j = 0; j < n; ++j) {
        auto& v = cols[j];
        if (v.empty()) continue;
        std::sort(v.begin(), v.end());
        const double mx = v.back(), med = v[(v.size() - 1) / 2];
        const double ratio = med > 0.0 ? mx / med : (mx > 0.0 ? std::numeric_limits<double>::infinity() : 0.0);
        if (ratio > threshold) ++s.flagged;
        s.cols.push_back({static_cast<double>(j), mx, med, ratio});
    }
    return s;
}

} // namespace

Report run_analyze(const Csr& A, const Config& cfg, const std::string& label) {
    const auto t0 = std::chrono::steady_clock::now();
    const IluParams ip = ilu_params_from(cfg);
    const HostFactors f = factorize(A, ip, nullptr);
    const double factor_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    DeviceContext ctx(cfg);
    cudaStream_t st = ctx.stream;

    const double dep_l = departure(f.L), dep_u = departure(f.U);
    DeviceIlu row, rowcol;
    row.build(f, ScalingKind::row, UpperIteration::scaled, false, st);
    rowcol.build(f, ScalingKind::row_col, UpperIteration::scaled, false, st);
    const Csr U_row = row.scaled_upper_host(), U_rowcol = rowcol.scaled_upper_host();
    const double dep_u_row = departure(U_row), dep_u_rowcol = departure(U_rowcol);

    const ScalingKind target = scaling_from(cfg);
    const Csr& U_diag = target == ScalingKind::none ? f.U : (target == ScalingKind::row ? U_row : U_rowcol);
    const double cond_l = condition_estimate(f.L, Shape::unit_lower, st);
    const double cond_u = condition_estimate(U_diag, Shape::upper, st);
    const double thr = cfg.get_double("striping.threshold");
    const Striping sp = striping(f.L, U_diag, thr);

    const char* variant = ip.variant == IluVariant::ilu0 ? "ilu0" : "ilut";
    const i64 nnz_l = f.L.nnz() + A.nrows, nnz_u = f.U.nnz();
    Report r;
    r.add("matrix", label);
    r.add("n", A.nrows);
    r.add("nnz", A.nnz());
    r.add("variant", variant);
    r.add("droptol", ip.droptol);
    r.add("lfill", ip.lfill);
    r.add("nnz_L", nnz_l);
    r.add("nnz_U", nnz_u);
    r.add("dep_L", dep_l);
    r.add("dep_U", dep_u);
    r.add("dep_U_row", dep_u_row);
    r.add("dep_U_rowcol", dep_u_rowcol);
    r.add("cond_L", cond_l);
    r.add("cond_U", cond_u);
    r.add("cond_scaling", target == ScalingKind::none ? "none" : (target == ScalingKind::row ? "row" : "row_col"));
    r.add("striping_threshold", thr);
    r.add("striping_flagged", sp.flagged);
    r.add("factor_seconds", factor_seconds);
    ReportTable t;
    t.name = "analyze";
    t.columns = {"matrix", "variant", "droptol", "lfill", "nnzL", "nnzU", "depL", "depU", "depUrow", "depUrowcol",
                 "cond_est"};
    t.rows.push_back({label, variant, format_num(ip.droptol), std::to_string(ip.lfill), std::to_string(nnz_l),
                      std::to_string(nnz_u), format_num(dep_l), format_num(dep_u), format_num(dep_u_row),
                      format_num(dep_u_rowcol), format_num(cond_u)});
    r.tables.push_back(std::move(t));
    if (sp.flagged > 0) {
        ReportTable s;
        s.name = "striping";
        s.columns = {"col", "max_abs", "median_abs", "ratio"};
        for (const auto& c : sp.cols) {
            if (c[3] <= thr) continue;
            s.rows.push_back({std::to_string(static_cast<i64>(c[0])), format_num(c[1]), format_num(c[2]),
                              format_num(c[3])});
            if (s.rows.size() >= 200) break;
        }
        r.tables.push_back(std::move(s));
    }
    return r;
}

} // namespace ilug
