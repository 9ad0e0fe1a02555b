// C ABI of the distributed GMRES+AMG solver (ilug_dist_solver_*) and the
// pipelined host-buffer entry of the distributed smoother. Handle layouts:
// capi_handles.hpp (shared with capi.cpp).
#include "capi_handles.hpp"

namespace ilug {
int capi_guarded(const std::function<int()>& fn); // capi.cpp: exception -> status + last error
}

extern "C" {

int ilug_dist_solver_create(const ilug_hierarchy* h, const ilug_dist_comm* c, ilug_dist_solver** out) {
    return ilug::capi_guarded([&] {
        if (!h || !c || !out) ilug::fail_invalid("null argument");
        auto* s = new ilug_dist_solver_s();
        try {
            s->s.build(h->h, *c->c, nullptr);
        } catch (...) {
            delete s;
            throw;
        }
        *out = s;
        return ILUAMG_OK;
    });
}

int ilug_dist_gmres(ilug_dist_solver* s, const iluamg_config* cfg, const double* b, double* x,
                    long long* iterations, double* final_relres, void* stream) {
    return ilug::capi_guarded([&] {
        if (!s || !cfg || !b || !x) ilug::fail_invalid("null argument");
        const auto& c = cfg->cfg;
        ilug::KrylovParams p;
        p.flexible = c.get("krylov.method") == "fgmres";
        if (!p.flexible && c.get("krylov.method") != "gmres")
            ilug::fail_invalid("config: krylov.method must be gmres or fgmres");
        p.restart = c.get_index("krylov.restart");
        p.max_iters = c.get_index("krylov.max_iters");
        p.tol = c.get_double("krylov.tol");
        p.nrbe_criterion = c.get("krylov.criterion") == "nrbe";
        if (p.nrbe_criterion) ilug::fail_invalid("distributed gmres: the nrbe criterion needs |A|_2 (not distributed)");
        p.record_history = c.get_bool("krylov.record_history");
        p.form_iterates = c.get_bool("krylov.form_iterates");
        const ilug::KrylovReport r = s->s.solve(b, x, p, static_cast<cudaStream_t>(stream));
        ILUG_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        if (iterations) *iterations = r.iterations;
        if (final_relres) *final_relres = r.final_relres;
        return r.converged ? ILUAMG_OK : ILUAMG_NOT_CONVERGED;
    });
}

int ilug_dist_vcycle(ilug_dist_solver* s, const double* r, double* z, void* stream) {
    return ilug::capi_guarded([&] {
        if (!s || !r || !z) ilug::fail_invalid("null argument");
        s->s.vcycle(r, z, static_cast<cudaStream_t>(stream));
        return ILUAMG_OK;
    });
}

int ilug_dist_solver_info(const ilug_dist_solver* s, long long* row0, long long* nloc, int* levels) {
    return ilug::capi_guarded([&] {
        if (!s) ilug::fail_invalid("null argument");
        if (row0) *row0 = s->s.row0();
        if (nloc) *nloc = s->s.nloc();
        if (levels) *levels = s->s.levels();
        return ILUAMG_OK;
    });
}

int ilug_dist_solver_levels(const ilug_dist_solver* s) { return s ? s->s.levels() : -1; }

int ilug_dist_level_plans(const ilug_hierarchy* h, int nranks, int rank, ilug_dist_levels** out) {
    return ilug::capi_guarded([&] {
        if (!h || !out) ilug::fail_invalid("null argument");
        *out = new ilug_dist_levels_s{ilug::dist_level_plans(h->h, nranks, rank)};
        return ILUAMG_OK;
    });
}

int ilug_dist_levels_count(const ilug_dist_levels* l) { return l ? static_cast<int>(l->levels.size()) : -1; }

int ilug_dist_levels_plan(const ilug_dist_levels* l, int k, int which, ilug_dist_plan** out) {
    return ilug::capi_guarded([&] {
        if (!l || !out) ilug::fail_invalid("null argument");
        if (k < 0 || k >= static_cast<int>(l->levels.size())) ilug::fail_invalid("level out of range");
        const ilug::DistLevelPlan& d = l->levels[k];
        if (which < 0 || which > 2 || (d.last && which > 0))
            ilug::fail_invalid("which: 0 = A, 1 = R, 2 = P (R/P of the last smoothed level are not halo plans)");
        *out = new ilug_dist_plan_s{which == 0 ? d.A : which == 1 ? d.R : d.P};
        return ILUAMG_OK;
    });
}

int ilug_dist_levels_last(const ilug_dist_levels* l, int which, iluamg_matrix** out) {
    return ilug::capi_guarded([&] {
        if (!l || !out || l->levels.empty()) ilug::fail_invalid("null argument or no smoothed level");
        const ilug::DistLevelPlan& d = l->levels.back();
        *out = new iluamg_matrix_s{which == 0 ? ilug::csr_copy(d.R_full) : ilug::csr_copy(d.P_rows), "dist"};
        return ILUAMG_OK;
    });
}

void ilug_dist_levels_free(ilug_dist_levels* l) { delete l; }

int ilug_dist_smooth_host(const ilug_dist_smoother* s, const double* bh, double* xh) {
    return ilug::capi_guarded([&] {
        if (!s || !bh || !xh) ilug::fail_invalid("null argument");
        const ilug::i64 n = s->s.nloc();
        if (s->hb.n != n) s->hb.alloc(n), s->hx.alloc(n);
        s->hb.upload(bh, n);
        s->hx.upload(xh, n);
        s->s.smooth(s->hb.p, s->hx.p, nullptr);
        s->hx.download(xh);
        ILUG_CUDA(cudaStreamSynchronize(nullptr));
        return ILUAMG_OK;
    });
}

int ilug_dist_smooth_host_many(const ilug_dist_smoother* s, long long count, const double* const* bh,
                               double* const* xh) {
    return ilug::capi_guarded([&] {
        if (!s || count < 0 || (count > 0 && (!bh || !xh))) ilug::fail_invalid("null argument");
        s->pipe.run(s->s.nloc(), count, bh, xh,
                    [&](const double* b, double* x, cudaStream_t st) { s->s.smooth(b, x, st); });
        return ILUAMG_OK;
    });
}

int ilug_dist_smoother_sweep_once(const ilug_dist_smoother* s, int which, const double* x_in, const double* rhs,
                                  double* out, void* stream) {
    return ilug::capi_guarded([&] {
        if (!s || !x_in || !rhs || !out) ilug::fail_invalid("null argument");
        const ilug::DeviceIlu* f = s->s.smoother().ilu();
        ilug::residual(which == 0 ? f->Ls() : f->Us(), x_in, rhs, out, static_cast<cudaStream_t>(stream));
        return ILUAMG_OK;
    });
}

void ilug_dist_solver_free(ilug_dist_solver* s) { delete s; }

} // extern "C"
