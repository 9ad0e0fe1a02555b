// K8: right-preconditioned (F)GMRES on the device with CGS2 orthogonalisation.
//
// Control flow mirrors gmres_impl (src/krylov.cpp:75-238) step for step —
// restart cycles, Givens rotations, the solve_y back substitution, the explicit
// x_k (non-flexible: x_cycle + M(V y), a second preconditioner application;
// flexible: x_cycle + Z y), history/NRBE records, false-convergence flag. The
// deliberate deviation is the orthogonalisation: modified Gram-Schmidt's j+1
// dependent dot/axpy passes become three fused CGS2 passes over the basis
// (SURVEY.md §8a a11b(iii)); iteration counts agree with the reference to ±1.
#include "dist.hpp"
#include "../host/problems.hpp"

#include <cmath>

namespace ilug {

namespace {

struct Scalars {
    DBuf<double> d;   // device scalars: h1[64] h2[64] nrm[1] misc[8]
    DBuf<double> ws;  // reduction workspace
    std::vector<double> h;
    const DistComm* comm = nullptr; // row-block distributed: sum partial reductions over ranks
    explicit Scalars(i64 n, const DistComm* c = nullptr)
        : d(64 * 2 + 16), ws(reduce_ws_doubles(n)), h(64 * 2 + 16), comm(c) {}
    void sum(double* p, i64 k, cudaStream_t st) const {
        if (comm) comm->allreduce_sum(p, k, st);
    }
    double* h1() { return d.p; }
    double* h2() { return d.p + 64; }
    double* nrm() { return d.p + 128; }
    double* misc() { return d.p + 129; }
};

double dev_norm(const double* v, i64 n, Scalars& s, cudaStream_t st) {
    nrm2sq_dev(v, n, s.misc(), s.ws.p, st);
    s.sum(s.misc(), 1, st);
    double h = 0.0;
    ILUG_CUDA(cudaMemcpyAsync(&h, s.misc(), sizeof h, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(h);
}

} // namespace

double device_estimate_two_norm(const DeviceMatrix& A, const Csr& A_host, i64 steps,
                                std::uint64_t seed, cudaStream_t st) {
    if (A.n == 0 || A_host.nnz() == 0) return 0.0;
    Sell At;
    sell_from_host(At, csr_transpose(A_host), Part::all, st);
    // random_unit(n, seed): mt19937_64 uniform(-1,1), normalised (src/rng.cpp:5-11)
    Vec v0 = random_uniform(A.n, seed);
    double nr = 0.0;
    for (double x : v0) nr += x * x;
    nr = std::sqrt(nr);
    if (nr > 0.0)
        for (double& x : v0) x /= nr;
    DBuf<double> v, w, u;
    v.upload(v0.data(), A.n, st);
    w.alloc(A.n);
    u.alloc(A.n);
    Scalars sc(A.n);
    for (i64 s = 0; s < steps; ++s) {
        spmv(A.A, v.p, w.p, st);
        spmv(At, w.p, u.p, st);
        const double nrm = dev_norm(u.p, A.n, sc, st);
        if (nrm == 0.0) return 0.0;
        vec_scale_div(v.p, u.p, nrm, A.n, st);
    }
    spmv(A.A, v.p, w.p, st);
    return dev_norm(w.p, A.n, sc, st);
}

void GmresWork::ensure(i64 n, i64 restart, bool flexible) {
    auto need = [](DBuf<double>& d, i64 count) {
        if (d.n != count) d.alloc(count);
    };
    need(V, (restart + 1) * n);
    need(Z, flexible ? restart * n : 0);
    for (DBuf<double>* d : {&w, &r, &xk, &xc, &vy, &mz}) need(*d, n);
    need(ydev, 64);
}

KrylovReport device_gmres(const DeviceMatrix& A, const Csr& A_host, DeviceHierarchy& M,
                          const double* b, double* x, const KrylovParams& p, cudaStream_t st,
                          const DistComm* comm, GmresWork* work) {
    const i64 n = A.n;
    if (p.restart < 1) fail_invalid("gmres: restart must be >= 1");
    if (p.restart > 63) fail_invalid("gmres: restart must be <= 63 on the device (basis width)");
    if (!(p.tol > 0.0)) fail_invalid("gmres: tol must be > 0");
    const i64 R = p.restart;
    KrylovReport rep;
    Scalars sc(n, comm);
    const bool distributed = comm && comm->nranks > 1; // |A|_2 needs a global transpose: skipped
    rep.anorm_estimate = p.estimate_anorm && !distributed
                             ? device_estimate_two_norm(A, A_host, 50, p.anorm_seed, st)
                             : std::nan("");
    rep.bnorm = dev_norm(b, n, sc, st);
    const double bden = rep.bnorm > 0.0 ? rep.bnorm : 1.0;

    GmresWork local;
    GmresWork& W = work ? *work : local;
    W.ensure(n, R, p.flexible);
    DBuf<double>&V = W.V, &Z = W.Z, &w = W.w, &r = W.r, &xk = W.xk, &xc = W.xc, &vy = W.vy, &mz = W.mz,
    &ydev = W.ydev;
    double* zbuf = mz.p;

    auto true_norms = [&](const double* xv, double& res, double& xn) {
        A.residual(xv, b, r.p, st);
        res = dev_norm(r.p, n, sc, st);
        xn = dev_norm(xv, n, sc, st);
    };
    auto record = [&](i64 iter, double arnoldi, const double* xv) {
        HistoryEntry e;
        e.iter = iter;
        e.arnoldi = arnoldi;
        double xn = 0.0;
        true_norms(xv, e.true_res, xn);
        const double den = rep.bnorm + rep.anorm_estimate * xn;
        e.nrbe = den == 0.0 ? 0.0 : e.true_res / den;
        if (p.record_history) rep.history.push_back(e);
        return e;
    };
    auto met = [&](double arnoldi, const HistoryEntry& e) {
        return p.nrbe_criterion ? e.nrbe < p.tol : arnoldi / bden < p.tol;
    };

    i64 total = 0;
    double last_arnoldi = 0.0;
    {
        A.residual(x, b, r.p, st);
        const double r0 = dev_norm(r.p, n, sc, st);
        const HistoryEntry e0 = record(0, r0, x);
        last_arnoldi = e0.arnoldi;
        if (met(e0.arnoldi, e0)) {
            rep.converged = true;
            rep.final_relres = e0.true_res / bden;
            rep.final_nrbe = e0.nrbe;
            return rep;
        }
    }

    std::vector<double> H(static_cast<size_t>((R + 1) * R), 0.0), cs(R), sn(R), g(R + 1);
    auto h = [&](i64 i, i64 j) -> double& { return H[static_cast<size_t>(j * (R + 1) + i)]; };
    bool done = false;
    while (!done && total < p.max_iters) {
        A.residual(x, b, r.p, st);
        const double beta = dev_norm(r.p, n, sc, st);
        if (!std::isfinite(beta)) fail_numeric("gmres: residual is not finite");
        if (beta == 0.0) {
            rep.converged = true;
            break;
        }
        vec_scale_div(V.p, r.p, beta, n, st);
        std::fill(g.begin(), g.end(), 0.0);
        std::fill(H.begin(), H.end(), 0.0);
        g[0] = beta;
        vec_copy(xc.p, x, n, st);
        for (i64 j = 0; j < R && total < p.max_iters; ++j) {
            double* zj = p.flexible ? Z.p + j * n : zbuf;
            M.vcycle(V.p + j * n, zj, st);
            ++rep.vcycles;
            A.spmv(zj, w.p, st);
            const int k = static_cast<int>(j + 1);
            multi_dot(V.p, n, k, w.p, n, sc.h1(), sc.ws.p, st);
            sc.sum(sc.h1(), k, st);
            multi_axpy_dot(V.p, n, k, sc.h1(), w.p, n, sc.h2(), sc.ws.p, st);
            sc.sum(sc.h2(), k, st);
            multi_axpy_nrm(V.p, n, k, sc.h2(), w.p, n, sc.nrm(), sc.ws.p, st);
            sc.sum(sc.nrm(), 1, st);
            ILUG_CUDA(cudaMemcpyAsync(sc.h.data(), sc.d.p, sizeof(double) * 129, cudaMemcpyDeviceToHost, st));
            ILUG_CUDA(cudaStreamSynchronize(st));
            for (i64 i = 0; i <= j; ++i) h(i, j) = sc.h[i] + sc.h[64 + i];
            const double hnext = std::sqrt(sc.h[128]);
            h(j + 1, j) = hnext;
            bool finite = std::isfinite(hnext);
            for (i64 i = 0; finite && i <= j; ++i) finite = std::isfinite(h(i, j));
            if (!finite)
                fail_numeric("gmres: Arnoldi coefficients are not finite at iteration " +
                             std::to_string(total + 1));
            const bool happy = hnext == 0.0;
            if (!happy) vec_scale_div(V.p + (j + 1) * n, w.p, hnext, n, st);

            for (i64 i = 0; i < j; ++i) {
                const double t = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
                h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
                h(i, j) = t;
            }
            {
                const double a = h(j, j), c = h(j + 1, j);
                const double rho = std::hypot(a, c);
                cs[j] = rho == 0.0 ? 1.0 : a / rho;
                sn[j] = rho == 0.0 ? 0.0 : c / rho;
                h(j, j) = rho;
                h(j + 1, j) = 0.0;
            }
            g[j + 1] = -sn[j] * g[j];
            g[j] = cs[j] * g[j];
            const double arnoldi = std::abs(g[j + 1]);
            ++total;
            last_arnoldi = arnoldi;

            const bool conv_relres = !p.nrbe_criterion && arnoldi / bden < p.tol;
            const bool need_x = p.form_iterates || p.nrbe_criterion || conv_relres || happy ||
                                j + 1 == R || total >= p.max_iters;
            if (!need_x) {
                if (p.record_history)
                    rep.history.push_back({total, arnoldi, std::nan(""), std::nan("")});
                continue;
            }
            // y = H(0:j,0:j)^-1 g  (solve_y, src/krylov.cpp:63-72)
            std::vector<double> y(static_cast<size_t>(j + 1));
            for (i64 i = j + 1; i-- > 0;) {
                double s = g[i];
                for (i64 kk = i + 1; kk <= j; ++kk) s -= h(i, kk) * y[kk];
                y[i] = s / h(i, i);
            }
            ILUG_CUDA(cudaMemcpyAsync(ydev.p, y.data(), sizeof(double) * y.size(), cudaMemcpyHostToDevice, st));
            if (p.flexible) {
                multi_combine(Z.p, n, k, ydev.p, xc.p, xk.p, n, st);
            } else {
                multi_combine(V.p, n, k, ydev.p, nullptr, vy.p, n, st);
                M.vcycle(vy.p, mz.p, st);
                ++rep.vcycles;
                vec_add_into(xk.p, xc.p, mz.p, n, st);
            }
            if (!std::isfinite(dev_norm(xk.p, n, sc, st)))
                fail_numeric("gmres: iterate is not finite at iteration " + std::to_string(total));
            HistoryEntry e;
            if (p.form_iterates || p.nrbe_criterion)
                e = record(total, arnoldi, xk.p);
            else if (p.record_history)
                rep.history.push_back({total, arnoldi, std::nan(""), std::nan("")});
            vec_copy(x, xk.p, n, st);
            if ((p.form_iterates || p.nrbe_criterion ? met(arnoldi, e) : conv_relres) || happy) {
                rep.converged = true;
                done = true;
                break;
            }
        }
    }
    rep.iterations = total;
    double tr = 0.0, xn = 0.0;
    true_norms(x, tr, xn);
    rep.final_relres = tr / bden;
    const double den = rep.bnorm + rep.anorm_estimate * xn;
    rep.final_nrbe = den == 0.0 ? 0.0 : tr / den;
    rep.false_convergence = std::abs(tr - last_arnoldi) / bden > 10.0 * p.tol;
    return rep;
}

} // namespace ilug
