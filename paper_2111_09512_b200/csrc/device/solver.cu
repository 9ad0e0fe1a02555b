// Device ILU factors, smoothers and the V-cycle (see solver.hpp).
#include "solver.hpp"
#include "../kernels/spgemm.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace ilug {

// ============================================================ DeviceMatrix
void DeviceMatrix::build(const Csr& host, cudaStream_t st) {
    n = host.nrows;
    sell_from_host(A, host, Part::all, st);
}

void DeviceMatrix::build(const Csr& host, const i64* rp, const i32* ci, const double* v, cudaStream_t st) {
    n = host.nrows;
    sell_from_device_rows(A, host.nrows, host.ncols, host.rp, 0, rp, ci, v, Part::all, st);
}

void DeviceMatrix::residual(const double* x, const double* b, double* r, cudaStream_t st) const {
    if (!halo) return ilug::residual(A, x, b, r, st);
    halo->begin(x, st); // the local-only rows run while the halo is in flight
    const HaloWait w = halo->waiter();
    residual_split(A, x, halo->halo.p, halo->nloc, b, r, st, &w);
}

void DeviceMatrix::spmv(const double* x, double* y, cudaStream_t st) const {
    if (!halo) return ilug::spmv(A, x, y, st);
    halo->begin(x, st);
    const HaloWait w = halo->waiter();
    spmv_split(A, x, halo->halo.p, halo->nloc, y, st, &w);
}

// ============================================================ DeviceIlu (K1-K5)
void DeviceIlu::build(const HostFactors& f, ScalingKind scaling, UpperIteration upper,
                      bool direct_plans, cudaStream_t st) {
    DevFactors df = DevFactors::upload(f, st);
    finish(df, &f, scaling, upper, direct_plans, st);
}

void DeviceIlu::build(DevFactors&& df, ScalingKind scaling, UpperIteration upper, bool direct_plans,
                      cudaStream_t st) {
    DevFactors own = std::move(df);
    finish(own, nullptr, scaling, upper, direct_plans, st);
}

void DeviceIlu::finish(DevFactors& df, const HostFactors* host, ScalingKind scaling, UpperIteration upper,
                       bool direct_plans, cudaStream_t st) {
    n_ = df.n;
    scaling_ = scaling;
    upper_ = upper;
    // host patterns are needed only by the wavefront and level-set plans, and by
    // factors whose U rows do not all start with the diagonal
    HostFactors pulled;
    const bool need_host = !host && (wave_enabled(n_) || direct_plans || !df.diag_first);
    if (need_host) pulled = df.to_host(st);
    const HostFactors* hp = host ? host : (need_host ? &pulled : nullptr);
    sell_from_device_rows(Ls_, n_, n_, df.Lrp_h, 0, df.Lrp.p, df.Lci.p, df.Lv.p, Part::all, st);
    const i64* rp = df.Urp.p;
    const i32* ci = df.Uci.p;
    double* v = df.Uv.p;

    const bool scale = upper == UpperIteration::scaled && scaling != ScalingKind::none;
    if (!scale) {
        // Unscaled factor: keep D for the Jacobi iteration / direct division.
        d_.alloc(n_);
        const i64 bad = extract_diag(n_, rp, ci, v, d_.p, st);
        if (bad >= 0 && (upper == UpperIteration::jacobi || direct_plans))
            fail_numeric("ilu factors: zero diagonal entry in U at row " + std::to_string(bad));
    } else {
        rs_.alloc(n_);
        DBuf<double> dr, dc;
        if (scaling == ScalingKind::row_col) {
            cs_.alloc(n_);
            dr.alloc(n_);
            dc.alloc(n_);
        }
        const i64 bad = scale_upper(n_, rp, ci, v, scaling == ScalingKind::row ? 1 : 2, rs_.p, cs_.p, dr.p, dc.p, st);
        if (bad >= 0)
            fail_numeric(std::string(scaling == ScalingKind::row ? "row_scale" : "row_col_scale") +
                         ": zero diagonal entry in U at row " + std::to_string(bad));
    }
    if (df.diag_first)
        sell_from_device_rows(Us_, n_, n_, df.Urp_h, 1, rp, ci, v, Part::strict_upper, st);
    else
        sell_from_device_csr(Us_, hp->U, rp, ci, v, Part::strict_upper, {}, st);
    if (wave_enabled(n_)) {
        wave_build(wave_L_, hp->L, Ls_, false, st);
        wave_build(wave_U_, hp->U, Us_, true, st);
    }
    if (direct_plans) {
        lower_plan_.build(hp->L, LevelPlan::Kind::lower_unit, st);
        upper_plan_.build(hp->U, LevelPlan::Kind::upper, st, v);
        if (direct_uses_cusparse()) {
            cs_lower_ = std::make_unique<CusparseTri>();
            cs_lower_->build(n_, df.Lrp.p, df.Lci.p, df.Lv.p, df.Lv.n, true, st);
            cs_upper_ = std::make_unique<CusparseTri>();
            cs_upper_->build(n_, df.Urp.p, df.Uci.p, v, df.Uv.n, false, st);
        }
    }
    ILUG_CUDA(cudaStreamSynchronize(st));
}

void DeviceIlu::refactor(DevFactors&& dfin, cudaStream_t st) {
    DevFactors df = std::move(dfin);
    if (df.n != n_) fail_invalid("ilu refactor: dimension mismatch");
    if (wave_L_.ready() || wave_U_.ready())
        fail_invalid("ilu refactor: the wavefront plans (ILUG_WAVEFRONT) are not refilled");
    sell_refill(Ls_, df.Lrp.p, df.Lci.p, df.Lv.p, Part::all, st);
    const i64* rp = df.Urp.p;
    const i32* ci = df.Uci.p;
    double* v = df.Uv.p;
    const bool direct_plans = lower_plan_.levels() > 0;
    const bool scale = upper_ == UpperIteration::scaled && scaling_ != ScalingKind::none;
    if (!scale) {
        const i64 bad = extract_diag(n_, rp, ci, v, d_.p, st);
        if (bad >= 0 && (upper_ == UpperIteration::jacobi || direct_plans))
            fail_numeric("ilu factors: zero diagonal entry in U at row " + std::to_string(bad));
    } else {
        DBuf<double> dr, dc;
        if (scaling_ == ScalingKind::row_col) dr.alloc(n_), dc.alloc(n_);
        const i64 bad = scale_upper(n_, rp, ci, v, scaling_ == ScalingKind::row ? 1 : 2, rs_.p, cs_.p, dr.p, dc.p, st);
        if (bad >= 0)
            fail_numeric(std::string(scaling_ == ScalingKind::row ? "row_scale" : "row_col_scale") +
                         ": zero diagonal entry in U at row " + std::to_string(bad));
    }
    sell_refill(Us_, rp, ci, v, Part::strict_upper, st);
    if (direct_plans) {
        lower_plan_.refill(df.Lrp.p, df.Lci.p, df.Lv.p, st);
        upper_plan_.refill(rp, ci, v, st);
    }
    if (cs_lower_ || cs_upper_) fail_invalid("ilu refactor: the cuSPARSE comparison path is not refilled");
    ILUG_CUDA(cudaStreamSynchronize(st));
}

bool DeviceIlu::use_wave(bool upper, i64 m) const {
    return m >= 3 && m <= kWaveMaxSweeps + 1 && (upper ? wave_U_ : wave_L_).ready();
}

void DeviceIlu::sweep_lower(const double* b, double* y, i64 m, double* ws, cudaStream_t st) const {
    if (m < 1) fail_invalid("richardson_lower: iteration count must be >= 1");
    if (m == 1) return vec_copy(y, b, n_, st);
    if (use_wave(false, m) && y != b) {
        return wave_sweeps(Ls_, wave_L_, static_cast<int>(m - 1), b, b, nullptr, ws, WaveLast::plain,
                           nullptr, y, nullptr, st);
    }
    const double* cur = b;
    for (i64 k = 2; k <= m; ++k) {
        double* out = k == m && y != b ? y : ws + (k % 2) * n_;
        residual(Ls_, cur, b, out, st); // y_k = b - L_s y_{k-1}
        cur = out;
    }
    if (cur != y) vec_copy(y, cur, n_, st);
}

void DeviceIlu::sweep_upper(const double* b, double* x, i64 m, double* ws, cudaStream_t st) const {
    if (m < 1) fail_invalid("richardson_upper_scaled: iteration count must be >= 1");
    double* bs = ws;
    if (upper_ == UpperIteration::jacobi) {
        // x1 = D^-1 b; x_{k+1} = D^-1 (b - N x_k)
        vec_div(bs, b, d_.p, n_, st);
        if (use_wave(true, m)) {
            return wave_sweeps(Us_, wave_U_, static_cast<int>(m - 1), bs, b, d_.p, ws + n_, WaveLast::div,
                               d_.p, x, nullptr, st);
        }
        const double* cur = bs;
        for (i64 k = 2; k <= m; ++k) {
            double* out = k == m ? x : ws + (1 + k % 2) * n_;
            sweep_div(Us_, cur, b, d_.p, out, st);
            cur = out;
        }
        if (cur != x) vec_copy(x, cur, n_, st);
        return;
    }
    if (!has_rs()) fail_invalid("richardson_upper_scaled: factors carry no row scaling");
    vec_div(bs, b, rs_.p, n_, st); // b_s = b / row_scale (division, src/trisolve.cpp:113)
    if (use_wave(true, m)) {
        return wave_sweeps(Us_, wave_U_, static_cast<int>(m - 1), bs, bs, nullptr, ws + n_,
                           has_cs() ? WaveLast::div : WaveLast::plain, has_cs() ? cs_.p : nullptr, x, nullptr, st);
    }
    const double* cur = bs;
    for (i64 k = 2; k <= m; ++k) {
        double* out = k == m ? x : ws + (1 + k % 2) * n_;
        residual(Us_, cur, bs, out, st); // x_k = b_s - U_s x_{k-1}
        cur = out;
    }
    if (has_cs())
        vec_div(x, cur, cs_.p, n_, st);
    else if (cur != x)
        vec_copy(x, cur, n_, st);
}

void DeviceIlu::lower_direct(const double* b, double* y, cudaStream_t st) const {
    if (cs_lower_) return cs_lower_->solve(b, y, st);
    lower_plan_.solve(b, y, nullptr, st);
}

void DeviceIlu::upper_direct(const double* b, double* x, cudaStream_t st) const {
    if (cs_upper_) return cs_upper_->solve(b, x, st);
    upper_plan_.solve(b, x, nullptr, st);
}

void DeviceIlu::solve_lower(const double* b, double* y, cudaStream_t st) const {
    if (!has_plans()) fail_invalid("ilu factors: level plans were not built (direct mode off)");
    lower_direct(b, y, st);
}

void DeviceIlu::solve_upper(const double* b, double* x, double* ws, cudaStream_t st) const {
    if (!has_plans()) fail_invalid("ilu factors: level plans were not built (direct mode off)");
    if (has_rs()) {
        vec_div(ws, b, rs_.p, n_, st);
        upper_direct(ws, x, st);
        if (has_cs()) vec_div(x, x, cs_.p, n_, st);
    } else {
        upper_direct(b, x, st);
    }
}

Vec DeviceIlu::download(const DBuf<double>& b) const {
    Vec h(static_cast<size_t>(b.n));
    b.download(h.data());
    ILUG_CUDA(cudaDeviceSynchronize());
    return h;
}

Csr DeviceIlu::scaled_upper_host() const {
    const Csr S = sell_to_host(Us_);
    Csr U;
    U.nrows = U.ncols = n_;
    U.rp.assign(static_cast<size_t>(n_) + 1, 0);
    U.ci.reserve(static_cast<size_t>(S.nnz() + n_));
    U.v.reserve(static_cast<size_t>(S.nnz() + n_));
    Vec d;
    if (!has_rs()) d = download(d_);
    for (i64 i = 0; i < n_; ++i) {
        U.ci.push_back(static_cast<i32>(i));
        U.v.push_back(has_rs() ? 1.0 : d[i]);
        for (i64 k = S.rp[i]; k < S.rp[i + 1]; ++k) U.ci.push_back(S.ci[k]), U.v.push_back(S.v[k]);
        U.rp[i + 1] = static_cast<i64>(U.ci.size());
    }
    return U;
}

// ============================================================ DeviceSmoother
namespace {

// 1/a_ii per row from a device CSR: the first entry with column i, 0.0 when
// absent (csr_diag); the lowest zero row fails like inverted_diag below.
__global__ void k_inv_diag(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                           const double* __restrict__ v, double* __restrict__ invd,
                           unsigned long long* __restrict__ first_zero) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x) {
        double d = 0.0;
        for (i64 k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) {
                d = v[k];
                break;
            }
        if (d == 0.0) atomicMin(first_zero, static_cast<unsigned long long>(i));
        invd[i] = 1.0 / d;
    }
}

void inverted_diag_device(const DevCsr& M, DBuf<double>& invd, const char* what, cudaStream_t st) {
    const i64 n = M.nrows;
    invd.alloc(std::max<i64>(n, 1));
    DBuf<unsigned long long> fz(1);
    const unsigned long long none = ~0ull;
    ILUG_CUDA(cudaMemcpyAsync(fz.p, &none, sizeof none, cudaMemcpyHostToDevice, st));
    if (n > 0) {
        k_inv_diag<<<static_cast<unsigned>(std::min<i64>((n + 255) / 256, 148 * 32)), 256, 0, st>>>(
            n, M.rp.p, M.ci.p, M.v.p, invd.p, fz.p);
        ILUG_LAUNCH_CHECK();
    }
    unsigned long long z = 0;
    ILUG_CUDA(cudaStreamSynchronize(st)); // not inside the pageable copy (kernels/ilut.cu)
    ILUG_CUDA(cudaMemcpyAsync(&z, fz.p, sizeof z, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    if (z != ~0ull) fail_numeric(std::string(what) + ": zero diagonal at row " + std::to_string(z));
}

Vec inverted_diag(const Csr& A, const char* what) {
    Vec d = csr_diag(A);
    for (i64 i = 0; i < A.nrows; ++i) {
        if (d[i] == 0.0) fail_numeric(std::string(what) + ": zero diagonal at row " + std::to_string(i));
        d[i] = 1.0 / d[i];
    }
    return d;
}

} // namespace

void DeviceSmoother::build(const Csr& A, const DeviceMatrix& dA, const SmootherConfig& cfg,
                           cudaStream_t st, DevFactors* pre, const HaloPlan* dist, const DevCsr* dcsr) {
    if (cfg.sweeps < 0) fail_invalid("build_smoother_state: sweeps must be >= 0");
    if (cfg.poly_degree < 0) fail_invalid("build_smoother_state: poly_degree must be >= 0");
    cfg_ = cfg;
    n_ = A.nrows;
    A_ = &dA;
    if (dA.halo && !dist) fail_invalid("distributed smoothing: the rank's halo plan is required");
    switch (cfg.kind) {
    case SmootherKind::jacobi: {
        const Vec d = inverted_diag(A, "jacobi");
        invd_.upload(d.data(), n_, st);
        break;
    }
    case SmootherKind::l1_jacobi: {
        Vec d(static_cast<size_t>(n_), 0.0);
        const Csr& rows = dist ? dist->A_ext : A; // the whole row, in its global entry order
        for (i64 i = 0; i < n_; ++i)
            for (i64 k = rows.rp[i]; k < rows.rp[i + 1]; ++k) d[i] += std::abs(rows.v[k]);
        for (i64 i = 0; i < n_; ++i) {
            if (d[i] == 0.0)
                fail_numeric("l1_jacobi: row " + std::to_string(i) + " is entirely zero");
            d[i] = 1.0 / d[i];
        }
        invd_.upload(d.data(), n_, st);
        break;
    }
    case SmootherKind::gauss_seidel: {
        const Vec d = csr_diag(A);
        for (i64 i = 0; i < n_; ++i)
            if (d[i] == 0.0)
                fail_numeric("gauss_seidel_sweep: zero diagonal at row " + std::to_string(i));
        gs_ = std::make_unique<LevelPlan>();
        gs_->build(A, LevelPlan::Kind::gauss_seidel, st);
        if (dist) sell_from_host_split(Aoff_, dist->A_off, dist->nloc, st); // hybrid GS: off-block part
        break;
    }
    case SmootherKind::poly_gs: {
        if (dcsr && !dist && dcsr->nrows == n_) { // from the device copy: no second upload of A
            inverted_diag_device(*dcsr, invd_, "poly_gs", st);
            sell_from_device(Lstrict_, dcsr->nrows, dcsr->ncols, dcsr->ci.n, dcsr->rp.p, dcsr->ci.p, dcsr->v.p, st,
                             Part::strict_lower);
            break;
        }
        const Vec d = inverted_diag(A, "poly_gs");
        invd_.upload(d.data(), n_, st);
        sell_from_host(Lstrict_, A, Part::strict_lower, st);
        break;
    }
    case SmootherKind::ilu: {
        const bool rich = cfg.trisolve.mode == TriSolveMode::richardson;
        if (rich && cfg.scaling == ScalingKind::none && cfg.trisolve.upper == UpperIteration::scaled)
            fail_invalid("ilu smoother: the iterative U solve requires row or row/col scaling");
        ilu_ = std::make_unique<DeviceIlu>();
        ilu_->build(pre ? std::move(*pre) : factorize_resident(A, cfg.ilu_params, st), cfg.scaling,
                    rich ? cfg.trisolve.upper : UpperIteration::scaled, !rich, st);
        break;
    }
    case SmootherKind::schur_ilut:
        schur_ = std::make_unique<DeviceSchur>();
        if (dist)
            schur_->build_dist(*dist, *dA.halo->tr, cfg, st); // block b = rank b
        else
            schur_->build(A, cfg, st);
        break;
    }
    // r, y ping-pong, bs, x ping-pong, spare; then the wavefront intermediates
    // (only when a fused plan exists)
    const i64 mmax = std::max(cfg.trisolve.m_lower, cfg.trisolve.m_upper);
    const bool wave = ilu_ && (ilu_->wave_L().ready() || ilu_->wave_U().ready());
    ws_.alloc((7 + (wave ? std::max<i64>(mmax - 2, 0) : 0)) * std::max<i64>(n_, 1));
    ILUG_CUDA(cudaStreamSynchronize(st));
}

void DeviceSmoother::ilu_sweep(const double* b, double* x, bool x_zero, cudaStream_t st) const {
    const DeviceIlu& f = *ilu_;
    const i64 n = n_;
    double* r = ws_.p;
    double* ya = ws_.p + n;
    double* yb = ws_.p + 2 * n;
    double* bs = ws_.p + 3 * n;
    double* xa = ws_.p + 4 * n;
    double* xb = ws_.p + 5 * n;
    const double* rr = b; // r = b - A*0 = b exactly when x == 0
    if (!x_zero) {
        A_->residual(x, b, r, st); // halo-exchanged when A_ is a distributed block
        rr = r;
    }
    const TriSolveConfig& ts = cfg_.trisolve;
    if (ts.mode == TriSolveMode::direct) {
        f.solve_lower(rr, ya, st);
        if (f.has_rs()) {
            vec_div(bs, ya, f.rs(), n, st);
            f.upper_direct(bs, xa, st);
        } else {
            f.upper_direct(ya, xa, st);
        }
        if (f.has_cs())
            vec_acc_div(x, xa, f.cs(), n, st);
        else
            vec_acc(x, xa, n, st);
        return;
    }
    const i64 mL = ts.m_lower, mU = ts.m_upper;
    if (mL < 1) fail_invalid("richardson_lower: iteration count must be >= 1");
    if (mU < 1) fail_invalid("richardson_upper_scaled: iteration count must be >= 1");
    const bool jac = f.upper_iteration() == UpperIteration::jacobi;
    const double* dv = jac ? f.diag() : f.rs();
    // ---- L sweeps; the last one also produces x_1 of the U iteration (bs)
    const double* y = rr;
    double* tmp = ws_.p + 7 * n; // wavefront intermediates (max(mL, mU) - 2 vectors)
    if (mL == 1) {
        vec_div(bs, rr, dv, n, st);
    } else if (f.use_wave(false, mL)) {
        // mL-1 fused sweeps; the last writes y (Jacobi form only) and x_1 = y / d
        if (jac)
            wave_sweeps(f.Ls(), f.wave_L(), static_cast<int>(mL - 1), rr, rr, nullptr, tmp, WaveLast::both, dv, ya,
                        bs, st);
        else
            wave_sweeps(f.Ls(), f.wave_L(), static_cast<int>(mL - 1), rr, rr, nullptr, tmp, WaveLast::div, dv, bs,
                        nullptr, st);
        y = ya;
    } else {
        const double* cur = rr;
        for (i64 k = 2; k <= mL; ++k) {
            double* out = (k % 2) ? ya : yb;
            if (k == mL) {
                if (jac)
                    sweep_both(f.Ls(), cur, rr, dv, out, bs, st); // y and x1 = y / d
                else
                    sweep_div(f.Ls(), cur, rr, dv, bs, st); // b_s = y / row_scale
            } else {
                residual(f.Ls(), cur, rr, out, st);
            }
            cur = out;
        }
        y = cur;
    }
    // ---- U sweeps; the last one accumulates into x (with the column unscale)
    const double* rhs = jac ? y : bs;
    const double* post = jac ? f.diag() : (f.has_cs() ? f.cs() : nullptr);
    if (mU == 1) {
        if (post)
            vec_acc_div(x, jac ? y : bs, post, n, st);
        else
            vec_acc(x, bs, n, st);
        return;
    }
    if (f.use_wave(true, mU)) {
        wave_sweeps(f.Us(), f.wave_U(), static_cast<int>(mU - 1), bs, rhs, jac ? f.diag() : nullptr, tmp,
                    post ? WaveLast::acc_div : WaveLast::acc, post, x, nullptr, st);
        return;
    }
    const double* cur = bs;
    for (i64 k = 2; k <= mU; ++k) {
        if (k == mU) {
            sweep_acc(f.Us(), cur, rhs, post, x, st);
        } else {
            double* out = (k % 2) ? xa : xb;
            if (jac)
                sweep_div(f.Us(), cur, rhs, f.diag(), out, st);
            else
                residual(f.Us(), cur, rhs, out, st);
            cur = out;
        }
    }
}

void DeviceSmoother::smooth(const double* b, double* x, bool x_zero, cudaStream_t st) const {
    const i64 n = n_;
    for (i64 s = 0; s < cfg_.sweeps; ++s) {
        const bool zero = x_zero && s == 0;
        switch (cfg_.kind) {
        case SmootherKind::jacobi:
        case SmootherKind::l1_jacobi:
            if (const HaloExchange* h = A_->halo) {
                h->begin(x, st);
                const HaloWait w = h->waiter();
                residual_scale_step_split(A_->A, x, h->halo.p, h->nloc, b, invd_.p, ws_.p, st, &w);
            } else {
                residual_scale_step(A_->A, x, b, invd_.p, ws_.p, st);
            }
            vec_copy(x, ws_.p, n, st);
            break;
        case SmootherKind::gauss_seidel:
            if (const HaloExchange* h = A_->halo) {
                // hybrid GS: b' = b - A_off x (current halo), then GS on the diagonal block
                h->begin(x, st);
                const HaloWait w = h->waiter();
                residual_split(Aoff_, x, h->halo.p, h->nloc, b, ws_.p + n, st, &w);
                gs_->solve(ws_.p + n, ws_.p, x, st);
            } else {
                gs_->solve(b, ws_.p, x, st);
            }
            vec_copy(x, ws_.p, n, st);
            break;
        case SmootherKind::poly_gs: {
            double* t0 = ws_.p;
            double* t1 = ws_.p + n;
            double* acc = ws_.p + 2 * n;
            if (const HaloExchange* h = A_->halo) {
                h->begin(x, st);
                const HaloWait w = h->waiter();
                residual_scale_init_split(A_->A, x, h->halo.p, h->nloc, b, invd_.p, t0, acc, st, &w);
            } else {
                residual_scale_init(A_->A, x, b, invd_.p, t0, acc, st);
            }
            for (i64 j = 1; j <= cfg_.poly_degree; ++j) {
                neg_scale_acc(Lstrict_, t0, invd_.p, t1, acc, st);
                std::swap(t0, t1);
            }
            vec_acc(x, acc, n, st);
            break;
        }
        case SmootherKind::ilu:
            ilu_sweep(b, x, zero, st);
            break;
        case SmootherKind::schur_ilut:
            schur_->apply(*A_, b, x, st);
            break;
        }
    }
}

// ============================================================ DeviceHierarchy
DeviceHierarchy::~DeviceHierarchy() {
    if (exec_) cudaGraphExecDestroy(exec_);
}

void DeviceHierarchy::build(const HostHierarchy& h, cudaStream_t st, DevFactors* level0) {
    const int L = static_cast<int>(h.levels.size());
    begin();
    for (int k = 0; k < L; ++k)
        build_level(k, h.levels[k], h.params.plan.for_level(k), k + 1 == L, k == 0 ? level0 : nullptr, st);
    finish(h, st);
}

void DeviceHierarchy::begin() {
    levels_.clear();
    if (exec_) cudaGraphExecDestroy(exec_);
    exec_ = nullptr;
}

void DeviceHierarchy::build_level(int k, const HostLevel& hl, const SmootherConfig& sc, bool last,
                                  DevFactors* level0, cudaStream_t st) {
    if (k != num_levels()) fail_invalid("device hierarchy: levels must be built in order");
    SetupTimer tm("device");
    Lev& lv = levels_.emplace_back();
    lv.n = hl.A.nrows;
    if (k == 0 && level0 && level0->Av.n == hl.A.nnz() && hl.A.nnz() > 0) {
        lv.A.build(hl.A, level0->Arp.p, level0->Aci.p, level0->Av.p, st); // the factorisation's upload
        ILUG_CUDA(cudaStreamSynchronize(st));
        level0->Arp.release(), level0->Aci.release(), level0->Av.release();
    } else if (hl.dA && hl.A.nnz() > 0) { // the device AMG setup's copy
        lv.A.build(hl.A, hl.dA->rp.p, hl.dA->ci.p, hl.dA->v.p, st);
    } else {
        lv.A.build(hl.A, st);
    }
    if (!last) {
        if (hl.dP) sell_from_device(lv.P, hl.dP->nrows, hl.dP->ncols, hl.dP->ci.n, hl.dP->rp.p, hl.dP->ci.p, hl.dP->v.p, st);
        else sell_from_host(lv.P, hl.P, Part::all, st);
        if (hl.dR) sell_from_device(lv.R, hl.dR->nrows, hl.dR->ncols, hl.dR->ci.n, hl.dR->rp.p, hl.dR->ci.p, hl.dR->v.p, st);
        else sell_from_host(lv.R, hl.R, Part::all, st);
        tm.mark("A,P,R", k);
        lv.smoother.build(hl.A, lv.A, sc, st, level0, nullptr, hl.dA.get());
        tm.mark("smoother", k);
    }
    lv.b.alloc(std::max<i64>(lv.n, 1));
    lv.x.alloc(std::max<i64>(lv.n, 1));
    lv.r.alloc(std::max<i64>(lv.n, 1));
    ILUG_CUDA(cudaStreamSynchronize(st));
    hl.dA.reset(), hl.dP.reset(), hl.dR.reset(); // the SELL copies exist now
}

void DeviceHierarchy::build_level0_ops(const HostLevel& hl, const i64* rp, const i32* ci, const double* v,
                                       cudaStream_t st) {
    if (num_levels() != 0) fail_invalid("device hierarchy: levels must be built in order");
    SetupTimer tm("device");
    Lev& lv = levels_.emplace_back();
    lv.n = hl.A.nrows;
    lv.A.build(hl.A, rp, ci, v, st);
    if (hl.dP) sell_from_device(lv.P, hl.dP->nrows, hl.dP->ncols, hl.dP->ci.n, hl.dP->rp.p, hl.dP->ci.p, hl.dP->v.p, st);
    else sell_from_host(lv.P, hl.P, Part::all, st);
    if (hl.dR) sell_from_device(lv.R, hl.dR->nrows, hl.dR->ncols, hl.dR->ci.n, hl.dR->rp.p, hl.dR->ci.p, hl.dR->v.p, st);
    else sell_from_host(lv.R, hl.R, Part::all, st);
    lv.b.alloc(std::max<i64>(lv.n, 1));
    lv.x.alloc(std::max<i64>(lv.n, 1));
    lv.r.alloc(std::max<i64>(lv.n, 1));
    ILUG_CUDA(cudaStreamSynchronize(st));
    hl.dA.reset(), hl.dP.reset(), hl.dR.reset();
    tm.mark("A,P,R", 0);
}

void DeviceHierarchy::build_smoother0(const HostLevel& hl, const SmootherConfig& sc, DevFactors* level0,
                                      cudaStream_t st) {
    SetupTimer tm("device");
    Lev& lv = levels_.at(0);
    lv.smoother.build(hl.A, lv.A, sc, st, level0);
    ILUG_CUDA(cudaStreamSynchronize(st));
    tm.mark("smoother", 0);
}

void DeviceHierarchy::finish(const HostHierarchy& h, cudaStream_t st) {
    lu_.upload(h.coarse.lu.data(), static_cast<i64>(h.coarse.lu.size()), st);
    piv_.upload(h.coarse.piv.data(), static_cast<i64>(h.coarse.piv.size()), st);
    nu_ = h.params.cycles_nu;
    trace_ = std::getenv("ILUG_TRACE") != nullptr && !use_graph_;
    if (exec_) cudaGraphExecDestroy(exec_);
    exec_ = nullptr;
    ILUG_CUDA(cudaStreamSynchronize(st));
}

void DeviceHierarchy::cycle(int k, bool x_zero, cudaStream_t st) {
    Lev& lv = levels_[k];
    if (k + 1 == num_levels()) {
        dense_lu_solve_dev(lv.n, lu_.p, piv_.p, lv.b.p, lv.x.p, st);
        return;
    }
    Lev& nx = levels_[k + 1];
    // ILUG_TRACE=1 (eager mode only): per-level phase times on stderr.
    auto mark = [&](const char* what) {
        if (!trace_) return;
        static cudaEvent_t last = nullptr;
        cudaEvent_t e;
        ILUG_CUDA(cudaEventCreate(&e));
        ILUG_CUDA(cudaEventRecord(e, st));
        ILUG_CUDA(cudaEventSynchronize(e));
        if (last) {
            float ms = 0.f;
            ILUG_CUDA(cudaEventElapsedTime(&ms, last, e));
            std::fprintf(stderr, "[trace] level %d n=%lld %-10s %.3f ms\n", k, static_cast<long long>(lv.n),
                         what, ms);
            cudaEventDestroy(last);
        }
        last = e;
    };
    mark("enter");
    lv.smoother.smooth(lv.b.p, lv.x.p, x_zero, st);
    mark("presmooth");
    residual(lv.A.A, lv.x.p, lv.b.p, lv.r.p, st);
    spmv(lv.R, lv.r.p, nx.b.p, st);
    vec_zero(nx.x.p, nx.n, st);
    mark("restrict");
    for (i64 i = 0; i < nu_; ++i) cycle(k + 1, i == 0, st);
    mark("coarse");
    spmv_add(lv.P, nx.x.p, lv.x.p, st);
    mark("prolong");
    lv.smoother.smooth(lv.b.p, lv.x.p, false, st);
    mark("postsmooth");
}

void DeviceHierarchy::vcycle_eager(const double* r, double* z, cudaStream_t st) {
    Lev& l0 = levels_[0];
    vec_copy(l0.b.p, r, l0.n, st);
    vec_zero(l0.x.p, l0.n, st);
    cycle(0, true, st);
    vec_copy(z, l0.x.p, l0.n, st);
}

void DeviceHierarchy::prepare_graph() {
    if (!use_graph_ || exec_ || levels_.empty()) return;
    Lev& l0 = levels_[0];
    // Capture the whole cycle once (fixed internal in/out buffers).
    cudaStream_t cap;
    ILUG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    ILUG_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    try {
        vec_zero(l0.x.p, l0.n, cap);
        cycle(0, true, cap);
    } catch (...) {
        cudaStreamEndCapture(cap, &g);
        if (g) cudaGraphDestroy(g);
        cudaStreamDestroy(cap);
        throw;
    }
    ILUG_CUDA(cudaStreamEndCapture(cap, &g));
    size_t nodes = 0;
    ILUG_CUDA(cudaGraphGetNodes(g, nullptr, &nodes));
    kernels_per_cycle_ = static_cast<i64>(nodes);
    ILUG_CUDA(cudaGraphInstantiate(&exec_, g, 0));
    cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
}

void DeviceHierarchy::vcycle(const double* r, double* z, cudaStream_t st) {
    if (!use_graph_) return vcycle_eager(r, z, st);
    Lev& l0 = levels_[0];
    prepare_graph();
    vec_copy(l0.b.p, r, l0.n, st);
    ILUG_CUDA(cudaGraphLaunch(exec_, st));
    vec_copy(z, l0.x.p, l0.n, st);
}

} // namespace ilug
