// K8: right-preconditioned (F)GMRES on the device with CGS2 orthogonalisation.
//
// Control flow mirrors gmres_impl (src/krylov.cpp:75-238) step for step —
// restart cycles, Givens rotations, the solve_y back substitution, the explicit
// x_k (non-flexible: x_cycle + M(V y), a second preconditioner application;
// flexible: x_cycle + Z y), history/NRBE records, false-convergence flag. The
// deliberate deviation is the orthogonalisation: modified Gram-Schmidt's j+1
// dependent dot/axpy passes become three fused CGS2 passes over the basis
// (SURVEY.md §8a a11b(iii)); iteration counts agree with the reference to ±1.
//
// Device-resident scalar path: the Hessenberg matrix, the Givens rotations,
// the right-hand side g and y = H^-1 g live in device memory and are updated
// by single-thread kernels (k_arnoldi, k_solve_y); the basis width is any
// restart >= 1 (the CGS2 kernels chunk their outputs). Per iteration the host
// reads back one pinned 4-double status — |g_{j+1}|, h_{j+1,j}, a finiteness
// flag and the previous iterate's ||x||^2 — with the one stream sync the
// convergence test needs; true residual norms of the recorded history are
// written to a device array and read once at the end (NRBE criterion: one more
// sync per iteration, it needs the true residual to decide).
#include "dist.hpp"
#include "../host/problems.hpp"

#include <cmath>

namespace ilug {

namespace {

// Column-major (R+1) x R Hessenberg H, rotations cs/sn, rhs g (src/krylov.cpp:160-190):
// store column j from the two CGS2 passes, apply the previous rotations, form
// rotation j, update g. stat: [0] |g_{j+1}|, [1] h_{j+1,j}, [2] 1.0 if finite.
__global__ void k_arnoldi(int j, int R, const double* __restrict__ h1, const double* __restrict__ h2,
                          const double* __restrict__ nrm, double* H, double* cs, double* sn, double* g,
                          double* hnext_out, double* stat) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int ld = R + 1;
    double* col = H + static_cast<i64>(j) * ld;
    bool finite = true;
    for (int i = 0; i <= j; ++i) {
        col[i] = h1[i] + h2[i];
        finite = finite && isfinite(col[i]);
    }
    const double hnext = sqrt(nrm[0]);
    finite = finite && isfinite(hnext);
    col[j + 1] = hnext;
    *hnext_out = finite ? hnext : 0.0; // a non-finite column is reported, v_{j+1} left unset
    for (int i = 0; i < j; ++i) {
        const double t = cs[i] * col[i] + sn[i] * col[i + 1];
        col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1];
        col[i] = t;
    }
    const double a = col[j], c = col[j + 1];
    const double rho = hypot(a, c);
    cs[j] = rho == 0.0 ? 1.0 : a / rho;
    sn[j] = rho == 0.0 ? 0.0 : c / rho;
    col[j] = rho;
    col[j + 1] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    stat[0] = fabs(g[j + 1]);
    stat[1] = hnext;
    stat[2] = finite ? 1.0 : 0.0;
}

// y = H(0:j,0:j)^-1 g (solve_y, src/krylov.cpp:63-72): the serial back
// substitution, same operation order as the reference.
__global__ void k_solve_y(int j, int R, const double* __restrict__ H, const double* __restrict__ g,
                          double* y) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const i64 ld = R + 1;
    for (int i = j + 1; i-- > 0;) {
        double s = g[i];
        for (int kk = i + 1; kk <= j; ++kk) s -= H[kk * ld + i] * y[kk];
        y[i] = s / H[i * ld + i];
    }
}

// start of a restart cycle: H = 0, g = (beta, 0, ..., 0)
__global__ void k_cycle_init(double* H, i64 nH, double* g, int R, double beta) {
    for (i64 i = threadIdx.x; i < nH; i += blockDim.x) H[i] = 0.0;
    for (int i = threadIdx.x; i <= R; i += blockDim.x) g[i] = i == 0 ? beta : 0.0;
}

struct Reducer {
    DBuf<double> misc; // one device scalar
    double* ws;
    const DistComm* comm;
    void sum(double* p, i64 k, cudaStream_t st) const {
        if (comm) comm->allreduce_sum(p, k, st);
    }
    /// ||v||^2 into out (device), summed over ranks
    void nrm2sq(const double* v, i64 n, double* out, cudaStream_t st) const {
        nrm2sq_dev(v, n, out, ws, st);
        sum(out, 1, st);
    }
    double norm(const double* v, i64 n, cudaStream_t st) const {
        nrm2sq(v, n, misc.p, st);
        double h = 0.0;
        ILUG_CUDA(cudaMemcpyAsync(&h, misc.p, sizeof h, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        return std::sqrt(h);
    }
};

double dev_norm(const double* v, i64 n, const double* /*unused*/, cudaStream_t st, double* ws,
                const DistComm* comm = nullptr) {
    Reducer r{DBuf<double>(1), ws, comm};
    return r.norm(v, n, st);
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
    DBuf<double> ws(reduce_ws_doubles(A.n));
    for (i64 s = 0; s < steps; ++s) {
        spmv(A.A, v.p, w.p, st);
        spmv(At, w.p, u.p, st);
        const double nrm = dev_norm(u.p, A.n, nullptr, st, ws.p);
        if (nrm == 0.0) return 0.0;
        vec_scale_div(v.p, u.p, nrm, A.n, st);
    }
    spmv(A.A, v.p, w.p, st);
    return dev_norm(w.p, A.n, nullptr, st, ws.p);
}

GmresWork::~GmresWork() {
    if (stat) cudaFreeHost(stat);
}

void GmresWork::ensure(i64 n, i64 restart, bool flexible, i64 max_iters) {
    auto need = [](DBuf<double>& d, i64 count) {
        if (d.n != count) d.alloc(count);
    };
    const i64 R = std::max<i64>(restart, 1);
    need(V, (R + 1) * n);
    need(Z, flexible ? R * n : 0);
    for (DBuf<double>* d : {&w, &r, &xk, &xc, &vy, &mz}) need(*d, n);
    // h1[R+1] h2[R+1] nrm hnext misc[6] | H[(R+1)R] | cs[R] sn[R] g[R+1] y[R]
    need(S, 2 * (R + 1) + 8 + (R + 1) * R + 4 * R + 1);
    need(hist, 2 * (std::max<i64>(max_iters, 0) + 2));
    need(ws, reduce_ws_doubles(n, R + 1));
    if (!stat) ILUG_CUDA(cudaMallocHost(&stat, 8 * sizeof(double)));
    R_ = R;
}

KrylovReport device_gmres(const DeviceMatrix& A, const Csr* A_host, const Preconditioner& M,
                          const double* b, double* x, const KrylovParams& p, cudaStream_t st,
                          const DistComm* comm, GmresWork* work) {
    const i64 n = A.n;
    if (p.restart < 1) fail_invalid("gmres: restart must be >= 1");
    if (!(p.tol > 0.0)) fail_invalid("gmres: tol must be > 0");
    const i64 R = p.restart;
    KrylovReport rep;
    GmresWork local;
    GmresWork& W = work ? *work : local;
    W.ensure(n, R, p.flexible, p.max_iters);
    const Reducer red{DBuf<double>(1), W.ws.p, comm};
    double* h1 = W.S.p;
    double* h2 = h1 + (R + 1);
    double* nrm = h2 + (R + 1);
    double* hnext = nrm + 1;
    double* dstat = hnext + 1; // 4 status doubles
    double* H = h1 + 2 * (R + 1) + 8;
    double* csd = H + (R + 1) * R;
    double* snd = csd + R;
    double* g = snd + R;
    double* yd = g + R + 1;
    double* hist = W.hist.p;
    double* stat = W.stat;

    const bool distributed = comm && comm->nranks > 1; // |A|_2 needs a global transpose: skipped
    rep.anorm_estimate = p.estimate_anorm && !distributed && A_host
                             ? device_estimate_two_norm(A, *A_host, 50, p.anorm_seed, st)
                             : std::nan("");
    rep.bnorm = red.norm(b, n, st);
    const double bden = rep.bnorm > 0.0 ? rep.bnorm : 1.0;
    DBuf<double>&V = W.V, &Z = W.Z, &w = W.w, &r = W.r, &xk = W.xk, &xc = W.xc, &vy = W.vy, &mz = W.mz;
    double* zbuf = mz.p;
    const bool records = p.form_iterates || p.nrbe_criterion;

    auto nrbe_of = [&](double res, double xn) {
        const double den = rep.bnorm + rep.anorm_estimate * xn;
        return den == 0.0 ? 0.0 : res / den;
    };
    // true residual and ||x|| of the iterate xv into hist[2t], hist[2t+1] (device, no sync)
    auto record_dev = [&](i64 t, const double* xv) {
        A.residual(xv, b, r.p, st);
        red.nrm2sq(r.p, n, hist + 2 * t, st);
        red.nrm2sq(xv, n, hist + 2 * t + 1, st);
    };
    auto read_record = [&](i64 t, double& res, double& xn) {
        ILUG_CUDA(cudaMemcpyAsync(stat + 4, hist + 2 * t, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        res = std::sqrt(stat[4]);
        xn = std::sqrt(stat[5]);
    };

    i64 total = 0;
    double last_arnoldi = 0.0;
    // history entries whose true norms are still on the device (filled at the end)
    std::vector<std::pair<size_t, i64>> pending;
    {
        A.residual(x, b, r.p, st);
        const double r0 = red.norm(r.p, n, st);
        HistoryEntry e0;
        e0.iter = 0;
        e0.arnoldi = r0;
        record_dev(0, x);
        double xn = 0.0;
        read_record(0, e0.true_res, xn);
        e0.nrbe = nrbe_of(e0.true_res, xn);
        if (p.record_history) rep.history.push_back(e0);
        last_arnoldi = r0;
        if (p.nrbe_criterion ? e0.nrbe < p.tol : r0 / bden < p.tol) {
            rep.converged = true;
            rep.final_relres = e0.true_res / bden;
            rep.final_nrbe = e0.nrbe;
            rep.iterations = 0;
            return rep;
        }
    }

    bool done = false;
    i64 xk_slot = -1; // hist slot whose ||x||^2 is the last formed iterate's (finiteness check)
    while (!done && total < p.max_iters) {
        A.residual(x, b, r.p, st);
        const double beta = red.norm(r.p, n, st);
        if (!std::isfinite(beta)) fail_numeric("gmres: residual is not finite");
        if (beta == 0.0) {
            rep.converged = true;
            break;
        }
        vec_scale_div(V.p, r.p, beta, n, st);
        k_cycle_init<<<1, 256, 0, st>>>(H, (R + 1) * R, g, static_cast<int>(R), beta);
        ILUG_LAUNCH_CHECK();
        vec_copy(xc.p, x, n, st);
        for (i64 j = 0; j < R && total < p.max_iters; ++j) {
            double* zj = p.flexible ? Z.p + j * n : zbuf;
            M(V.p + j * n, zj, st);
            ++rep.vcycles;
            A.spmv(zj, w.p, st);
            const int k = static_cast<int>(j + 1);
            multi_dot(V.p, n, k, w.p, n, h1, W.ws.p, st);
            red.sum(h1, k, st);
            multi_axpy_dot(V.p, n, k, h1, w.p, n, h2, W.ws.p, st);
            red.sum(h2, k, st);
            multi_axpy_nrm(V.p, n, k, h2, w.p, n, nrm, W.ws.p, st);
            red.sum(nrm, 1, st);
            k_arnoldi<<<1, 32, 0, st>>>(static_cast<int>(j), static_cast<int>(R), h1, h2, nrm, H, csd, snd, g,
                                        hnext, dstat);
            ILUG_LAUNCH_CHECK();
            vec_scale_div_dev(V.p + (j + 1) * n, w.p, hnext, n, st); // skipped on happy breakdown
            // the one sync of the iteration: the convergence test's scalars
            ILUG_CUDA(cudaMemcpyAsync(stat, dstat, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
            if (xk_slot >= 0)
                ILUG_CUDA(cudaMemcpyAsync(stat + 3, hist + 2 * xk_slot + 1, sizeof(double),
                                          cudaMemcpyDeviceToHost, st));
            ILUG_CUDA(cudaStreamSynchronize(st));
            if (xk_slot >= 0 && !std::isfinite(stat[3]))
                fail_numeric("gmres: iterate is not finite at iteration " + std::to_string(xk_slot));
            xk_slot = -1;
            if (stat[2] != 1.0)
                fail_numeric("gmres: Arnoldi coefficients are not finite at iteration " +
                             std::to_string(total + 1));
            const double arnoldi = stat[0];
            const bool happy = stat[1] == 0.0;
            ++total;
            last_arnoldi = arnoldi;

            const bool conv_relres = !p.nrbe_criterion && arnoldi / bden < p.tol;
            const bool need_x = records || conv_relres || happy || j + 1 == R || total >= p.max_iters;
            if (!need_x) {
                if (p.record_history) rep.history.push_back({total, arnoldi, std::nan(""), std::nan("")});
                continue;
            }
            k_solve_y<<<1, 32, 0, st>>>(static_cast<int>(j), static_cast<int>(R), H, g, yd);
            ILUG_LAUNCH_CHECK();
            if (p.flexible) {
                multi_combine(Z.p, n, k, yd, xc.p, xk.p, n, st);
            } else {
                multi_combine(V.p, n, k, yd, nullptr, vy.p, n, st);
                M(vy.p, mz.p, st);
                ++rep.vcycles;
                vec_add_into(xk.p, xc.p, mz.p, n, st);
            }
            bool met = conv_relres;
            if (records) {
                record_dev(total, xk.p); // true residual + ||x_k||^2 (also the finiteness check)
                HistoryEntry e{total, arnoldi, std::nan(""), std::nan("")};
                if (p.nrbe_criterion) { // the criterion needs the true residual now
                    double xn = 0.0;
                    read_record(total, e.true_res, xn);
                    if (!std::isfinite(stat[5]))
                        fail_numeric("gmres: iterate is not finite at iteration " + std::to_string(total));
                    e.nrbe = nrbe_of(e.true_res, xn);
                    met = e.nrbe < p.tol;
                } else {
                    pending.emplace_back(rep.history.size(), total);
                }
                if (p.record_history) rep.history.push_back(e);
            } else {
                red.nrm2sq(xk.p, n, hist + 2 * total + 1, st);
                if (p.record_history) rep.history.push_back({total, arnoldi, std::nan(""), std::nan("")});
            }
            xk_slot = total;
            vec_copy(x, xk.p, n, st);
            if (met || happy) {
                rep.converged = true;
                done = true;
                break;
            }
        }
    }
    if (xk_slot >= 0) { // the last formed iterate's finiteness
        ILUG_CUDA(cudaMemcpyAsync(stat + 3, hist + 2 * xk_slot + 1, sizeof(double), cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        if (!std::isfinite(stat[3]))
            fail_numeric("gmres: iterate is not finite at iteration " + std::to_string(xk_slot));
    }
    if (!pending.empty()) { // history true norms: one download at the end
        std::vector<double> hh(static_cast<size_t>(2 * (total + 1)));
        ILUG_CUDA(cudaMemcpyAsync(hh.data(), hist, hh.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        for (auto [idx, t] : pending) {
            if (!p.record_history) break;
            HistoryEntry& e = rep.history[idx];
            e.true_res = std::sqrt(hh[2 * t]);
            e.nrbe = nrbe_of(e.true_res, std::sqrt(hh[2 * t + 1]));
        }
    }
    rep.iterations = total;
    A.residual(x, b, r.p, st);
    red.nrm2sq(r.p, n, hist, st);
    red.nrm2sq(x, n, hist + 1, st);
    double tr = 0.0, xn = 0.0;
    read_record(0, tr, xn);
    rep.final_relres = tr / bden;
    rep.final_nrbe = nrbe_of(tr, xn);
    rep.false_convergence = std::abs(tr - last_arnoldi) / bden > 10.0 * p.tol;
    levelset_check_error(st);
    return rep;
}

} // namespace ilug
