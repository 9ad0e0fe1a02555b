// The C ABI: iluamg_* (drop-in for the reference's include/iluamg.h, mirroring
// src/capi.cpp's handle/status/last-error conventions) and ilug_* (device
// handles for the individual hot-path subsystems). No exception crosses it.
#include "capi_handles.hpp"
#include "../kernels/amg_setup.hpp"
#include "../kernels/spgemm.hpp"
#include "../host/problems.hpp"

#include <cmath>
#include <exception>
#include <functional>
#include <string>

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& fn) {
    try {
        g_err.clear();
        return fn();
    } catch (const ilug::Error& e) {
        g_err = e.what();
        return e.kind() == ilug::ErrorKind::numeric ? ILUAMG_ERR_NUMERIC : ILUAMG_ERR_INVALID;
    } catch (const std::bad_alloc&) {
        g_err = "out of host memory";
        return ILUAMG_ERR_NUMERIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ILUAMG_ERR_INVALID;
    }
}

void need(bool ok) {
    if (!ok) ilug::fail_invalid("null argument");
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

iluamg_report* wrap(ilug::Report rep) {
    auto* r = new iluamg_report_s{std::move(rep), {}, {}, {}};
    r->json = r->rep.json();
    r->text = r->rep.text();
    for (const auto& t : r->rep.tables) r->csv.push_back(t.csv());
    return r;
}

using RunFn = ilug::Report (*)(const ilug::Csr&, const ilug::Config&, const std::string&);

int run(const iluamg_matrix* A, const iluamg_config* cfg, iluamg_report** out, RunFn fn) {
    return guarded([&] {
        need(cfg && out);
        *out = nullptr;
        ilug::Report rep;
        if (A) {
            rep = fn(A->A, cfg->cfg, A->label);
        } else {
            const ilug::Csr M = ilug::load_matrix_from(cfg->cfg);
            rep = fn(M, cfg->cfg, cfg->cfg.get("matrix"));
        }
        const int status = rep.status == 0 ? ILUAMG_OK : ILUAMG_NOT_CONVERGED;
        if (status == ILUAMG_NOT_CONVERGED) g_err = "run completed without meeting its convergence criterion";
        *out = wrap(std::move(rep));
        return status;
    });
}

ilug::Csr csr_from_ll(long long nrows, long long ncols, const long long* rp, const long long* ci,
                      const double* v) {
    need(rp != nullptr);
    static_assert(sizeof(long long) == sizeof(ilug::i64));
    return ilug::csr_from_arrays(nrows, ncols, reinterpret_cast<const ilug::i64*>(rp),
                                 reinterpret_cast<const ilug::i64*>(ci), v);
}

ilug::ScalingKind scaling_of(int s) {
    if (s < 0 || s > 2) ilug::fail_invalid("scaling must be 0 (none), 1 (row) or 2 (row_col)");
    return static_cast<ilug::ScalingKind>(s);
}

ilug::UpperIteration upper_of(int u) {
    if (u < 0 || u > 1) ilug::fail_invalid("upper_iteration must be 0 (scaled) or 1 (jacobi)");
    return static_cast<ilug::UpperIteration>(u);
}

} // namespace

namespace ilug {
// Shared by the other C-ABI translation units (capi_dist.cpp).
int capi_guarded(const std::function<int()>& fn) { return guarded(fn); }
} // namespace ilug

extern "C" {

// ============================================================ iluamg_* (drop-in)
const char* iluamg_version(void) { return "0.1.0-b200"; }
const char* iluamg_last_error(void) { return g_err.c_str(); }

int iluamg_matrix_read(const char* path, iluamg_matrix** out) {
    return guarded([&] {
        need(path && out);
        *out = new iluamg_matrix_s{ilug::mm_read(path), path};
        return ILUAMG_OK;
    });
}
int iluamg_matrix_generate(const char* spec, iluamg_matrix** out) {
    return guarded([&] {
        need(spec && out);
        *out = new iluamg_matrix_s{ilug::generate_problem(spec), spec};
        return ILUAMG_OK;
    });
}
int iluamg_matrix_write(const iluamg_matrix* A, const char* path) {
    return guarded([&] {
        need(A && path);
        ilug::mm_write(A->A, path);
        return ILUAMG_OK;
    });
}
long long iluamg_matrix_rows(const iluamg_matrix* A) { return A ? A->A.nrows : -1; }
long long iluamg_matrix_cols(const iluamg_matrix* A) { return A ? A->A.ncols : -1; }
long long iluamg_matrix_nnz(const iluamg_matrix* A) { return A ? A->A.nnz() : -1; }
void iluamg_matrix_free(iluamg_matrix* A) { delete A; }

int iluamg_config_create(iluamg_config** out) {
    return guarded([&] {
        need(out);
        *out = new iluamg_config_s{};
        return ILUAMG_OK;
    });
}
int iluamg_config_load(iluamg_config* cfg, const char* path) {
    return guarded([&] {
        need(cfg && path);
        cfg->cfg.load_file(path);
        return ILUAMG_OK;
    });
}
int iluamg_config_set(iluamg_config* cfg, const char* key, const char* value) {
    return guarded([&] {
        need(cfg && key && value);
        cfg->cfg.set(key, value);
        return ILUAMG_OK;
    });
}
const char* iluamg_config_get(const iluamg_config* cfg, const char* key) {
    if (!cfg || !key || !cfg->cfg.has(key)) return nullptr;
    return cfg->cfg.get(key).c_str();
}
const char* iluamg_config_reference(void) {
    static const std::string ref = ilug::Config::reference();
    return ref.c_str();
}
void iluamg_config_free(iluamg_config* cfg) { delete cfg; }

int iluamg_run_analyze(const iluamg_matrix* A, const iluamg_config* cfg, iluamg_report** out) {
    return run(A, cfg, out, &ilug::run_analyze);
}
int iluamg_run_solve(const iluamg_matrix* A, const iluamg_config* cfg, iluamg_report** out) {
    return run(A, cfg, out, &ilug::run_solve);
}
int iluamg_run_bench_trisolve(const iluamg_matrix* A, const iluamg_config* cfg, iluamg_report** out) {
    return run(A, cfg, out, &ilug::run_bench_trisolve);
}
int iluamg_run_schur_solve(const iluamg_matrix* A, const iluamg_config* cfg, iluamg_report** out) {
    return run(A, cfg, out, &ilug::run_schur_solve);
}

int iluamg_report_status(const iluamg_report* r) { return r ? r->rep.status : ILUAMG_ERR_INVALID; }
int iluamg_report_scalar_count(const iluamg_report* r) {
    return r ? static_cast<int>(r->rep.scalars.size()) : 0;
}
const char* iluamg_report_scalar_key(const iluamg_report* r, int i) {
    if (!r || i < 0 || i >= static_cast<int>(r->rep.scalars.size())) return nullptr;
    return r->rep.scalars[i].first.c_str();
}
const char* iluamg_report_scalar_value(const iluamg_report* r, int i) {
    if (!r || i < 0 || i >= static_cast<int>(r->rep.scalars.size())) return nullptr;
    return r->rep.scalars[i].second.c_str();
}
const char* iluamg_report_get(const iluamg_report* r, const char* key) {
    if (!r || !key) return nullptr;
    const std::string* v = r->rep.find(key);
    return v ? v->c_str() : nullptr;
}
int iluamg_report_table_count(const iluamg_report* r) {
    return r ? static_cast<int>(r->rep.tables.size()) : 0;
}
const char* iluamg_report_table_name(const iluamg_report* r, int i) {
    if (!r || i < 0 || i >= static_cast<int>(r->rep.tables.size())) return nullptr;
    return r->rep.tables[i].name.c_str();
}
const char* iluamg_report_table_csv(const iluamg_report* r, const char* name) {
    if (!r || !name) return nullptr;
    for (size_t i = 0; i < r->rep.tables.size(); ++i)
        if (r->rep.tables[i].name == name) return r->csv[i].c_str();
    return nullptr;
}
const char* iluamg_report_json(const iluamg_report* r) { return r ? r->json.c_str() : nullptr; }
const char* iluamg_report_text(const iluamg_report* r) { return r ? r->text.c_str() : nullptr; }
void iluamg_report_free(iluamg_report* r) { delete r; }

// ============================================================ ilug_* (device handles)
const char* ilug_last_error(void) { return g_err.c_str(); }

int ilug_device_count(int* count) {
    return guarded([&] {
        need(count);
        *count = 0;
        const cudaError_t e = cudaGetDeviceCount(count);
        if (e != cudaSuccess) *count = 0;
        return ILUAMG_OK;
    });
}
int ilug_set_device(int device) {
    return guarded([&] {
        ILUG_CUDA(cudaSetDevice(device));
        return ILUAMG_OK;
    });
}
int ilug_synchronize(void* stream) {
    return guarded([&] {
        ILUG_CUDA(cudaStreamSynchronize(S(stream)));
        return ILUAMG_OK;
    });
}

int ilug_matrix_from_csr(long long nrows, long long ncols, const long long* rp, const long long* ci,
                         const double* v, iluamg_matrix** out) {
    return guarded([&] {
        need(out);
        *out = new iluamg_matrix_s{csr_from_ll(nrows, ncols, rp, ci, v), "csr"};
        return ILUAMG_OK;
    });
}
int ilug_matrix_copy_csr(const iluamg_matrix* A, long long* rp, long long* ci, double* v) {
    return guarded([&] {
        need(A && rp);
        for (size_t i = 0; i < A->A.rp.size(); ++i) rp[i] = A->A.rp[i];
        for (ilug::i64 k = 0; k < A->A.nnz(); ++k) {
            if (ci) ci[k] = A->A.ci[k];
            if (v) v[k] = A->A.v[k];
        }
        return ILUAMG_OK;
    });
}

namespace {
int make_factors(ilug::HostFactors hf, int scaling, int upper, int direct, ilug_factors** out) {
    const ilug::ScalingKind sk = scaling_of(scaling);
    const ilug::UpperIteration ui = upper_of(upper);
    auto* f = new ilug_factors_s();
    try {
        f->nnz_L = hf.L.nnz();
        f->nnz_U = hf.U.nnz();
        f->f.build(hf, sk, ui, direct != 0, nullptr);
    } catch (...) {
        delete f;
        throw;
    }
    *out = f;
    return ILUAMG_OK;
}
} // namespace

int ilug_factors_create(const iluamg_matrix* A, const iluamg_config* cfg, int scaling, int upper,
                        int direct, ilug_factors** out) {
    return guarded([&] {
        need(A && cfg && out);
        const ilug::IluParams ip = ilug::ilu_params_from(cfg->cfg);
        const int st = make_factors(ilug::factorize(A->A, ip, nullptr), scaling, upper, direct, out);
        if (ip.variant == ilug::IluVariant::ilu0) {
            (*out)->ilu0 = true;
            (*out)->patch = ip.pivot_patch;
            (*out)->a_rp = A->A.rp;
            (*out)->a_hash = ilug::csr_pattern_hash(A->A);
        }
        return st;
    });
}
int ilug_factors_refactor(ilug_factors* f, const iluamg_matrix* A) {
    return guarded([&] {
        need(f && A);
        if (!f->ilu0) ilug::fail_invalid("refactor: only ILU(0) factors (fixed pattern) can be refactorised");
        if (!f->sym) { // later calls are checked against the symbolic data (the same pattern)
            if (A->A.rp != f->a_rp || ilug::csr_pattern_hash(A->A) != f->a_hash)
                ilug::fail_invalid("refactor: the matrix pattern differs from the factorised one");
            f->sym = ilug::Ilu0Symbolic::analyse(A->A, nullptr);
        }
        f->f.refactor(f->sym->factor(A->A, f->patch, nullptr), nullptr);
        return ILUAMG_OK;
    });
}
int ilug_factors_from_csr(long long n, const long long* Lr, const long long* Lc, const double* Lv,
                          const long long* Ur, const long long* Uc, const double* Uv, int scaling,
                          int upper, int direct, ilug_factors** out) {
    return guarded([&] {
        need(out);
        ilug::HostFactors hf;
        hf.L = csr_from_ll(n, n, Lr, Lc, Lv);
        hf.U = csr_from_ll(n, n, Ur, Uc, Uv);
        for (ilug::i64 i = 0; i < n; ++i) {
            for (ilug::i64 k = hf.L.rp[i]; k < hf.L.rp[i + 1]; ++k)
                if (hf.L.ci[k] >= i) ilug::fail_invalid("factors: L must be strictly lower triangular");
            for (ilug::i64 k = hf.U.rp[i]; k < hf.U.rp[i + 1]; ++k)
                if (hf.U.ci[k] < i) ilug::fail_invalid("factors: U must be upper triangular");
        }
        return make_factors(std::move(hf), scaling, upper, direct, out);
    });
}
long long ilug_factors_rows(const ilug_factors* f) { return f ? f->f.n() : -1; }
int ilug_factors_nnz(const ilug_factors* f, long long* nl, long long* nu) {
    return guarded([&] {
        need(f);
        if (nl) *nl = f->nnz_L;
        if (nu) *nu = f->nnz_U;
        return ILUAMG_OK;
    });
}
int ilug_factors_download_upper(const ilug_factors* f, long long* rows, long long* cols, double* vals,
                                double* rs, double* cs, int* flags) {
    return guarded([&] {
        need(f);
        const ilug::Csr U = f->f.scaled_upper_host();
        if (rows)
            for (size_t i = 0; i < U.rp.size(); ++i) rows[i] = U.rp[i];
        for (ilug::i64 k = 0; k < U.nnz(); ++k) {
            if (cols) cols[k] = U.ci[k];
            if (vals) vals[k] = U.v[k];
        }
        int fl = 0;
        if (f->f.has_rs()) {
            fl |= 1;
            if (rs) f->f.rs_buf().download(rs);
        }
        if (f->f.has_cs()) {
            fl |= 2;
            if (cs) f->f.cs_buf().download(cs);
        }
        ILUG_CUDA(cudaDeviceSynchronize());
        if (flags) *flags = fl;
        return ILUAMG_OK;
    });
}

namespace {
// Per-call workspace (3n) for the sweeps; allocated with stream-ordered malloc.
struct Ws {
    double* p = nullptr;
    cudaStream_t s;
    Ws(ilug::i64 n, cudaStream_t st) : s(st) {
        ILUG_CUDA(cudaMallocAsync(&p, static_cast<size_t>(std::max<ilug::i64>(n, 1)) * sizeof(double), st));
    }
    ~Ws() {
        if (p) cudaFreeAsync(p, s);
    }
};
} // namespace

int ilug_sweep_lower(const ilug_factors* f, const double* b, double* y, long long m, void* stream) {
    return guarded([&] {
        need(f && b && y);
        Ws ws(f->f.sweep_ws(m), S(stream));
        f->f.sweep_lower(b, y, m, ws.p, S(stream));
        return ILUAMG_OK;
    });
}
int ilug_sweep_upper(const ilug_factors* f, const double* b, double* x, long long m, void* stream) {
    return guarded([&] {
        need(f && b && x);
        Ws ws(f->f.sweep_ws(m) + f->f.n(), S(stream));
        f->f.sweep_upper(b, x, m, ws.p, S(stream));
        return ILUAMG_OK;
    });
}
int ilug_sweep_upper_host(const ilug_factors* f, const double* bh, double* xh, long long m) {
    return guarded([&] {
        need(f && bh && xh);
        const ilug::i64 n = f->f.n();
        ilug::DBuf<double> b, x(n), ws(std::max<ilug::i64>(f->f.sweep_ws(m) + n, 3));
        b.upload(bh, n);
        f->f.sweep_upper(b.p, x.p, m, ws.p, nullptr);
        x.download(xh);
        ILUG_CUDA(cudaStreamSynchronize(nullptr));
        return ILUAMG_OK;
    });
}
int ilug_solve_lower(const ilug_factors* f, const double* b, double* y, void* stream) {
    return guarded([&] {
        need(f && b && y);
        f->ser.run(S(stream), [&] { f->f.solve_lower(b, y, S(stream)); });
        ilug::levelset_check_error(S(stream));
        return ILUAMG_OK;
    });
}
int ilug_solve_upper(const ilug_factors* f, const double* b, double* x, void* stream) {
    return guarded([&] {
        need(f && b && x);
        Ws ws(f->f.n(), S(stream));
        f->ser.run(S(stream), [&] { f->f.solve_upper(b, x, ws.p, S(stream)); });
        ilug::levelset_check_error(S(stream));
        return ILUAMG_OK;
    });
}
int ilug_factors_stats(const ilug_factors* f, long long* n, long long* nl, long long* nu,
                       long long* padded, int* lev_l, int* lev_u) {
    return guarded([&] {
        need(f);
        if (n) *n = f->f.n();
        if (nl) *nl = f->f.Ls().nnz;
        if (nu) *nu = f->f.Us().nnz;
        if (padded) *padded = f->f.Us().padded;
        if (lev_l) *lev_l = f->f.lower_plan().levels();
        if (lev_u) *lev_u = f->f.upper_plan().levels();
        return ILUAMG_OK;
    });
}
namespace {
void wave_report(const ilug::DeviceIlu* f, long long* tl, long long* tu, int* stalled, long long* waits) {
    long long wl = 0, wu = 0;
    const bool bad_l = f && ilug::wave_stalled(f->wave_L(), &wl);
    const bool bad_u = f && ilug::wave_stalled(f->wave_U(), &wu);
    if (tl) *tl = f ? f->wave_L().ntiles : 0;
    if (tu) *tu = f ? f->wave_U().ntiles : 0;
    if (stalled) *stalled = bad_l || bad_u ? 1 : 0;
    if (waits) *waits = wl + wu;
}
} // namespace
int ilug_factors_wave(const ilug_factors* f, long long* tl, long long* tu, int* stalled, long long* waits) {
    return guarded([&] {
        need(f);
        wave_report(&f->f, tl, tu, stalled, waits);
        return ILUAMG_OK;
    });
}
void ilug_factors_free(ilug_factors* f) { delete f; }

int ilug_dmatrix_create(const iluamg_matrix* A, ilug_dmatrix** out) {
    return guarded([&] {
        need(A && out);
        auto* d = new ilug_dmatrix_s();
        try {
            d->M.build(A->A, nullptr);
            ILUG_CUDA(cudaStreamSynchronize(nullptr));
        } catch (...) {
            delete d;
            throw;
        }
        *out = d;
        return ILUAMG_OK;
    });
}
int ilug_spmv(const ilug_dmatrix* A, const double* x, double* y, void* stream) {
    return guarded([&] {
        need(A && x && y);
        ilug::spmv(A->M.A, x, y, S(stream));
        return ILUAMG_OK;
    });
}
int ilug_residual(const ilug_dmatrix* A, const double* x, const double* b, double* r, void* stream) {
    return guarded([&] {
        need(A && x && b && r);
        ilug::residual(A->M.A, x, b, r, S(stream));
        return ILUAMG_OK;
    });
}
void ilug_dmatrix_free(ilug_dmatrix* A) { delete A; }

int ilug_smoother_create(const iluamg_matrix* A, const iluamg_config* cfg, int which, ilug_smoother** out) {
    return guarded([&] {
        need(A && cfg && out);
        const ilug::SmootherConfig sc =
            which == 0 ? ilug::smoother_from(cfg->cfg) : ilug::fallback_smoother_from(cfg->cfg);
        auto* s = new ilug_smoother_s();
        try {
            s->A = A->A;
            s->dA.build(s->A, nullptr);
            s->s.build(s->A, s->dA, sc, nullptr);
            s->r.alloc(std::max<ilug::i64>(s->A.nrows, 1));
            s->scratch.alloc(1 + ilug::reduce_ws_doubles(s->A.nrows));
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
        return ILUAMG_OK;
    });
}
int ilug_smooth(const ilug_smoother* s, const double* b, double* x, double* resnorm, void* stream) {
    return guarded([&] {
        need(s && b && x);
        double h = 0.0;
        s->ser.run(S(stream), [&] {
            s->s.smooth(b, x, false, S(stream));
            if (resnorm) {
                ilug::residual(s->dA.A, x, b, s->r.p, S(stream));
                ilug::nrm2sq_dev(s->r.p, s->A.nrows, s->scratch.p, s->scratch.p + 1, S(stream));
                ILUG_CUDA(cudaMemcpyAsync(&h, s->scratch.p, sizeof h, cudaMemcpyDeviceToHost, S(stream)));
            }
        });
        if (resnorm) {
            ILUG_CUDA(cudaStreamSynchronize(S(stream)));
            *resnorm = std::sqrt(h);
        }
        return ILUAMG_OK;
    });
}
int ilug_ilu_smooth_sweep(const ilug_smoother* s, const double* b, double* x, void* stream) {
    return guarded([&] {
        need(s && b && x);
        if (s->s.config().kind != ilug::SmootherKind::ilu)
            ilug::fail_invalid("ilu_smooth_sweep: smoother is not an ILU smoother");
        s->ser.run(S(stream), [&] { s->s.ilu_sweep(b, x, false, S(stream)); });
        return ILUAMG_OK;
    });
}
int ilug_smooth_host(const ilug_smoother* s, const double* bh, double* xh) {
    return guarded([&] {
        need(s && bh && xh);
        const ilug::i64 n = s->A.nrows;
        s->ser.run_sync([&] {
            if (s->hb.n != n) s->hb.alloc(n), s->hx.alloc(n); // persistent staging buffers
            s->hb.upload(bh, n);
            s->hx.upload(xh, n);
            s->s.smooth(s->hb.p, s->hx.p, false, nullptr);
            s->hx.download(xh);
            ILUG_CUDA(cudaStreamSynchronize(nullptr));
        });
        return ILUAMG_OK;
    });
}
int ilug_smooth_host_many(const ilug_smoother* s, long long count, const double* const* bh, double* const* xh) {
    return guarded([&] {
        need(s && count >= 0 && (count == 0 || (bh && xh)));
        s->ser.run_sync([&] {
            s->pipe.run(s->A.nrows, count, bh, xh,
                        [&](const double* b, double* x, cudaStream_t st) { s->s.smooth(b, x, false, st); });
        });
        return ILUAMG_OK;
    });
}
int ilug_smoother_stats(const ilug_smoother* s, long long* n, long long* nnz_A, long long* nl,
                        long long* nu, long long* padded) {
    return guarded([&] {
        need(s);
        const ilug::DeviceIlu* f = s->s.ilu();
        if (n) *n = s->A.nrows;
        if (nnz_A) *nnz_A = s->A.nnz();
        if (nl) *nl = f ? f->Ls().nnz : 0;
        if (nu) *nu = f ? f->Us().nnz : 0;
        if (padded) *padded = f ? f->Us().padded : 0;
        return ILUAMG_OK;
    });
}
int ilug_smoother_wave(const ilug_smoother* s, long long* tl, long long* tu, int* stalled, long long* waits) {
    return guarded([&] {
        need(s);
        wave_report(s->s.ilu(), tl, tu, stalled, waits);
        return ILUAMG_OK;
    });
}
int ilug_smoother_sweeps_fused(const ilug_smoother* s, int which, int nsweeps, const double* x_in,
                               const double* rhs, double* tmp, double* out, void* stream) {
    return guarded([&] {
        need(s && x_in && rhs && out && (tmp || nsweeps == 1));
        const ilug::DeviceIlu* f = s->s.ilu();
        if (which != 0 && which != 1) ilug::fail_invalid("sweeps_fused: which must be 0 (L) or 1 (U)");
        if (!f || !(which ? f->wave_U() : f->wave_L()).ready())
            ilug::fail_invalid("sweeps_fused: no wavefront plan (ILUG_WAVEFRONT)");
        ilug::wave_sweeps(which ? f->Us() : f->Ls(), which ? f->wave_U() : f->wave_L(), nsweeps, x_in, rhs,
                          nullptr, tmp, ilug::WaveLast::plain, nullptr, out, nullptr, S(stream));
        return ILUAMG_OK;
    });
}
int ilug_smoother_sweep_once(const ilug_smoother* s, int which, const double* x_in, const double* rhs,
                             double* out, void* stream) {
    return guarded([&] {
        need(s && x_in && rhs && out);
        const ilug::DeviceIlu* f = s->s.ilu();
        if (!f) ilug::fail_invalid("sweep_once: smoother is not an ILU smoother");
        ilug::residual(which == 0 ? f->Ls() : f->Us(), x_in, rhs, out, S(stream));
        return ILUAMG_OK;
    });
}
void ilug_smoother_free(ilug_smoother* s) { delete s; }

int ilug_hierarchy_create(const iluamg_matrix* A, const iluamg_config* cfg, ilug_hierarchy** out) {
    return guarded([&] {
        need(A && cfg && out);
        auto* h = new ilug_hierarchy_s();
        try {
            const ilug::AmgParams ap = ilug::amg_params_from(cfg->cfg);
            h->h = ap.device_setup != 0 && ilug::amg_device_supported(ap) ? ilug::amg_setup_device(A->A, ap, {}, nullptr)
                                                                         : ilug::amg_setup(A->A, ap);
            h->d.set_use_graph(cfg->cfg.get_bool("device.graph"));
            h->d.build(h->h, nullptr);
            h->on_device = true;
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
        return ILUAMG_OK;
    });
}
int ilug_hierarchy_create_host(const iluamg_matrix* A, const iluamg_config* cfg, ilug_hierarchy** out) {
    return guarded([&] {
        need(A && cfg && out);
        auto* h = new ilug_hierarchy_s();
        try {
            // host-only handles keep the host setup unless device.amg_setup=device asks for the GPU
            const ilug::AmgParams ap = ilug::amg_params_from(cfg->cfg);
            if (ap.device_setup == 2 && !ilug::amg_device_supported(ap))
                ilug::fail_invalid("device.amg_setup=device needs amg.coarsening=pmis");
            h->h = ap.device_setup == 2 ? ilug::amg_setup_device(A->A, ap, {}, nullptr) : ilug::amg_setup(A->A, ap);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
        return ILUAMG_OK;
    });
}
int ilug_ilu_factorize(const iluamg_matrix* A, const iluamg_config* cfg, iluamg_matrix** L,
                       iluamg_matrix** U) {
    return guarded([&] {
        need(A && cfg && L && U);
        ilug::HostFactors f = ilug::ilu_factorize(A->A, ilug::ilu_params_from(cfg->cfg));
        *L = new iluamg_matrix_s{std::move(f.L), "L"};
        *U = new iluamg_matrix_s{std::move(f.U), "U"};
        return ILUAMG_OK;
    });
}
int ilug_ilu_factorize_device(const iluamg_matrix* A, const iluamg_config* cfg, iluamg_matrix** L,
                              iluamg_matrix** U) {
    return guarded([&] {
        need(A && cfg && L && U);
        ilug::HostFactors f = ilug::factorize(A->A, ilug::ilu_params_from(cfg->cfg), nullptr);
        *L = new iluamg_matrix_s{std::move(f.L), "L"};
        *U = new iluamg_matrix_s{std::move(f.U), "U"};
        return ILUAMG_OK;
    });
}
int ilug_matmul_device(const iluamg_matrix* A, const iluamg_matrix* B, iluamg_matrix** C) {
    return guarded([&] {
        need(A && B && C);
        *C = new iluamg_matrix_s{ilug::spgemm_device_host(A->A, B->A, nullptr), "C"};
        return ILUAMG_OK;
    });
}
int ilug_galerkin_device(const iluamg_matrix* A, const iluamg_matrix* P, const iluamg_matrix* R,
                         iluamg_matrix** C) {
    return guarded([&] {
        need(A && P && R && C);
        *C = new iluamg_matrix_s{ilug::galerkin_device(A->A, P->A, R->A, nullptr), "RAP"};
        return ILUAMG_OK;
    });
}
int ilug_hierarchy_levels(const ilug_hierarchy* h) { return h ? static_cast<int>(h->h.num_levels()) : -1; }
int ilug_hierarchy_level_matrix(const ilug_hierarchy* h, int level, int which, iluamg_matrix** out) {
    return guarded([&] {
        need(h && out);
        if (level < 0 || level >= h->h.num_levels() || which < 0 || which > 2)
            ilug::fail_invalid("hierarchy: level/which out of range");
        const ilug::HostLevel& L = h->h.levels[level];
        const ilug::Csr& M = which == 0 ? L.A : (which == 1 ? L.P : L.R);
        *out = new iluamg_matrix_s{M, "level"};
        return ILUAMG_OK;
    });
}
double ilug_hierarchy_operator_complexity(const ilug_hierarchy* h) {
    return h ? h->h.operator_complexity() : -1.0;
}
int ilug_vcycle(ilug_hierarchy* h, const double* r, double* z, void* stream) {
    return guarded([&] {
        need(h && r && z);
        if (!h->on_device) ilug::fail_invalid("vcycle: hierarchy was created host-only");
        h->ser.run(S(stream), [&] { h->d.vcycle(r, z, S(stream)); });
        return ILUAMG_OK;
    });
}
long long ilug_vcycle_graph_nodes(const ilug_hierarchy* h) { return h ? h->d.kernels_per_cycle() : -1; }
void ilug_hierarchy_free(ilug_hierarchy* h) { delete h; }

int ilug_gmres(ilug_hierarchy* h, const iluamg_config* cfg, const double* b, double* x,
               long long* iterations, double* final_relres, void* stream) {
    return guarded([&] {
        need(h && cfg && b && x);
        if (!h->on_device) ilug::fail_invalid("gmres: hierarchy was created host-only");
        ilug::KrylovParams p;
        const auto& c = cfg->cfg;
        p.flexible = c.get("krylov.method") == "fgmres";
        if (!p.flexible && c.get("krylov.method") != "gmres")
            ilug::fail_invalid("config: krylov.method must be gmres or fgmres");
        p.restart = c.get_index("krylov.restart");
        p.max_iters = c.get_index("krylov.max_iters");
        p.tol = c.get_double("krylov.tol");
        p.nrbe_criterion = c.get("krylov.criterion") == "nrbe";
        p.record_history = c.get_bool("krylov.record_history");
        p.anorm_seed = static_cast<std::uint64_t>(c.get_index("krylov.anorm_seed"));
        p.form_iterates = c.get_bool("krylov.form_iterates");
        p.estimate_anorm = p.form_iterates || p.nrbe_criterion;
        ilug::KrylovReport r;
        h->ser.run(S(stream), [&] {
            r = ilug::device_gmres(h->d.A0(), &h->h.levels[0].A, ilug::vcycle_of(h->d), b, x, p, S(stream));
        });
        ILUG_CUDA(cudaStreamSynchronize(S(stream)));
        if (iterations) *iterations = r.iterations;
        if (final_relres) *final_relres = r.final_relres;
        if (!r.converged) {
            g_err = "run completed without meeting its convergence criterion";
            return ILUAMG_NOT_CONVERGED;
        }
        return ILUAMG_OK;
    });
}

} // extern "C"

// ============================================================ ilug_dist_* (multi-GPU)
extern "C" {

int ilug_dist_partition(long long n, int nranks, long long* starts) {
    return guarded([&] {
        need(starts != nullptr);
        const ilug::RowPartition p = ilug::row_partition(n, nranks);
        for (int r = 0; r <= nranks; ++r) starts[r] = p.starts[r];
        return ILUAMG_OK;
    });
}
int ilug_dist_generate_rows(const char* spec, long long row0, long long row1, iluamg_matrix** out) {
    return guarded([&] {
        need(spec && out);
        *out = new iluamg_matrix_s{ilug::generate_rows(spec, row0, row1), spec};
        return ILUAMG_OK;
    });
}
int ilug_dist_plan_create(const iluamg_matrix* rows, long long n_global, int nranks, int rank,
                          ilug_dist_plan** out) {
    return guarded([&] {
        need(rows && out);
        const ilug::RowPartition part = ilug::row_partition(n_global, nranks);
        *out = new ilug_dist_plan_s{ilug::halo_plan(rows->A, part, rank)};
        return ILUAMG_OK;
    });
}
int ilug_dist_plan_info(const ilug_dist_plan* p, long long* row0, long long* row1, long long* nhalo) {
    return guarded([&] {
        need(p);
        if (row0) *row0 = p->plan.row0;
        if (row1) *row1 = p->plan.row1;
        if (nhalo) *nhalo = p->plan.nhalo;
        return ILUAMG_OK;
    });
}
long long ilug_dist_plan_requests(const ilug_dist_plan* p, int q, long long* ids) {
    if (!p) return -1;
    const std::vector<ilug::i64> r = ilug::halo_requests(p->plan, q);
    if (ids) std::copy(r.begin(), r.end(), ids);
    return static_cast<long long>(r.size());
}
int ilug_dist_plan_set_sends(ilug_dist_plan* p, int q, const long long* ids, long long count) {
    return guarded([&] {
        need(p && (ids || count == 0));
        ilug::halo_set_sends(p->plan, q, std::vector<ilug::i64>(ids, ids + count));
        return ILUAMG_OK;
    });
}
long long ilug_dist_plan_sends(const ilug_dist_plan* p, int q, long long* rows) {
    if (!p) return -1;
    const auto& h = p->plan;
    for (size_t k = 0; k < h.send_ranks.size(); ++k)
        if (h.send_ranks[k] == q) {
            const long long cnt = h.send_offsets[k + 1] - h.send_offsets[k];
            if (rows)
                for (long long i = 0; i < cnt; ++i) rows[i] = h.send_local[h.send_offsets[k] + i];
            return cnt;
        }
    return 0;
}
int ilug_dist_plan_matrix(const ilug_dist_plan* p, int which, iluamg_matrix** out) {
    return guarded([&] {
        need(p && out);
        if (which < 0 || which > 2) ilug::fail_invalid("plan matrix: which must be 0 (ext), 1 (diag) or 2 (off)");
        *out = new iluamg_matrix_s{which == 0 ? p->plan.A_ext : which == 1 ? p->plan.diag() : p->plan.A_off, "dist"};
        return ILUAMG_OK;
    });
}
void ilug_dist_plan_free(ilug_dist_plan* p) { delete p; }
int ilug_dist_unique_id(char* out128) {
    return guarded([&] {
        need(out128);
        ilug::dist_unique_id(out128);
        return ILUAMG_OK;
    });
}
int ilug_dist_comm_create(int nranks, int rank, const char* id128, ilug_dist_comm** out) {
    return guarded([&] {
        need(id128 && out);
        *out = new ilug_dist_comm_s{std::make_unique<ilug::DistComm>(ilug::make_nccl_transport(nranks, rank, id128))};
        return ILUAMG_OK;
    });
}
int ilug_dist_group_create(int nranks, ilug_dist_group** out) {
    return guarded([&] {
        need(out);
        *out = new ilug_dist_group_s{std::make_shared<ilug::LocalGroup>(nranks)};
        return ILUAMG_OK;
    });
}
void ilug_dist_group_free(ilug_dist_group* g) { delete g; }
void ilug_dist_group_abort(ilug_dist_group* g) {
    if (g) g->g->abort();
}
int ilug_dist_comm_create_local(ilug_dist_group* g, int rank, ilug_dist_comm** out) {
    return guarded([&] {
        need(g && out);
        *out = new ilug_dist_comm_s{std::make_unique<ilug::DistComm>(ilug::make_local_transport(g->g, rank))};
        return ILUAMG_OK;
    });
}
int ilug_dist_plan_exchange(ilug_dist_plan* p, const ilug_dist_comm* c) {
    return guarded([&] {
        need(p && c);
        ilug::plan_exchange(p->plan, *c->c->t);
        return ILUAMG_OK;
    });
}
int ilug_dist_allreduce_sum(const ilug_dist_comm* c, double* buf, long long count, void* stream) {
    return guarded([&] {
        need(c && buf);
        c->c->allreduce_sum(buf, count, S(stream));
        return ILUAMG_OK;
    });
}
void ilug_dist_comm_free(ilug_dist_comm* c) { delete c; }
int ilug_dist_smoother_create(const ilug_dist_plan* p, const ilug_dist_comm* c, const iluamg_config* cfg,
                              ilug_dist_smoother** out) {
    return guarded([&] {
        need(p && c && cfg && out);
        auto* s = new ilug_dist_smoother_s();
        try {
            s->s.build(p->plan, *c->c, ilug::smoother_from(cfg->cfg), nullptr);
            s->nnz_A = p->plan.A_ext.nnz();
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
        return ILUAMG_OK;
    });
}
int ilug_dist_smooth(const ilug_dist_smoother* s, const double* b, double* x, void* stream) {
    return guarded([&] {
        need(s && b && x);
        s->s.smooth(b, x, S(stream));
        return ILUAMG_OK;
    });
}
int ilug_dist_residual(const ilug_dist_smoother* s, const double* x, const double* b, double* r, void* stream) {
    return guarded([&] {
        need(s && x && b && r);
        s->s.residual(x, b, r, S(stream));
        return ILUAMG_OK;
    });
}
int ilug_dist_smoother_stats(const ilug_dist_smoother* s, long long* nloc, long long* nnz_A, long long* nl,
                             long long* nu) {
    return guarded([&] {
        need(s);
        const ilug::DeviceIlu* f = s->s.smoother().ilu();
        if (nloc) *nloc = s->s.nloc();
        if (nnz_A) *nnz_A = s->nnz_A;
        if (nl) *nl = f ? f->Ls().nnz : 0;
        if (nu) *nu = f ? f->Us().nnz : 0;
        return ILUAMG_OK;
    });
}
void ilug_dist_smoother_free(ilug_dist_smoother* s) { delete s; }

} // extern "C"
