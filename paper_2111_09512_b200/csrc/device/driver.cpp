#include "driver.hpp"
#include "../kernels/amg_setup.hpp"
#include "../host/problems.hpp"
#include "../kernels/spgemm.hpp"

#include <chrono>
#include <future>
#include <thread>
#include <mutex>
#include <optional>
#include <deque>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <sstream>

namespace ilug {

namespace {

double since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

KrylovParams krylov_from(const Config& c) {
    KrylovParams p;
    const std::string& m = c.get("krylov.method");
    if (m == "gmres")
        p.flexible = false;
    else if (m == "fgmres")
        p.flexible = true;
    else
        fail_invalid("config: krylov.method must be gmres or fgmres");
    p.restart = c.get_index("krylov.restart");
    p.max_iters = c.get_index("krylov.max_iters");
    p.tol = c.get_double("krylov.tol");
    const std::string& cr = c.get("krylov.criterion");
    if (cr == "relres")
        p.nrbe_criterion = false;
    else if (cr == "nrbe")
        p.nrbe_criterion = true;
    else
        fail_invalid("config: krylov.criterion must be relres or nrbe");
    p.record_history = c.get_bool("krylov.record_history");
    p.anorm_seed = static_cast<std::uint64_t>(c.get_index("krylov.anorm_seed"));
    p.form_iterates = c.get_bool("krylov.form_iterates");
    p.estimate_anorm = true;
    return p;
}

struct SolveOutcome {
    Vec x;
    KrylovReport kr;
    HostHierarchy hier;
    double setup_seconds = 0.0, solve_seconds = 0.0;
    i64 graph_nodes = 0;
    i64 schur_interface = 0;
};

SolveOutcome solve_with(const Csr& A, const AmgParams& ap, const KrylovParams& kp, const Vec& b,
                        bool use_graph, cudaStream_t st) {
    SolveOutcome oc;
    const auto t0 = std::chrono::steady_clock::now();
    std::optional<DeferFrees> defer(std::in_place); // setup threads must not serialise on cudaFree
    SetupTimer tm("solve_with");
    // The finest level's factorisation (ILU(0)/ILUT on the device) runs
    // concurrently with the host AMG setup, which does not need it and does
    // not touch the GPU. Identical factors either way (same function, same input).
    const SmootherConfig& s0 = ap.plan.for_level(0);
    // the hierarchy itself on the GPU when supported (kernels/amg_setup.cu), else the host
    const bool dev_setup = ap.device_setup != 0 && amg_device_supported(ap);
    if (ap.device_setup == 2 && !dev_setup) fail_invalid("device.amg_setup=device needs amg.coarsening=pmis");
    const bool fact0 = s0.kind == SmootherKind::ilu && A.nrows > ap.coarse_size;
    // With both on the GPU, A crosses PCIe once: the factorisation and the AMG
    // setup read the same device copy, which then becomes the level-0 operator.
    DevCsr Ad;
    const char* sa = std::getenv("ILUG_SHARE_A"); // =0: separate uploads (A/B)
    const bool share_A = dev_setup && fact0 && !(sa && sa[0] == '0');
    // the device hierarchy's operators built from the device AMG setup's own
    // copies of A_k, P_k, R_k (ILUG_KEEP_DEVICE_LEVELS=0: re-uploaded from the host, A/B)
    const char* kd = std::getenv("ILUG_KEEP_DEVICE_LEVELS");
    const bool keep_dev = dev_setup && !(kd && kd[0] == '0');
    if (share_A) {
        Ad.upload(A, st);
        ILUG_CUDA(cudaStreamSynchronize(st));
        tm.mark("upload A (shared)");
    }
    std::future<DevFactors> f0;
    if (fact0)
        f0 = std::async(std::launch::async,
                        [&] { return factorize_resident(A, s0.ilu_params, st, true, share_A ? &Ad : nullptr); });
    // The device objects of level k are built (own stream, own thread) as soon
    // as the host setup has finished level k, overlapping the host setup of
    // the coarser levels. Level 0's smoother takes the factors computed above.
    DeviceHierarchy dh;
    dh.set_use_graph(use_graph);
    dh.begin();
    // The setup's other GPU work (AMG kernels, SELL layouts) runs at the
    // highest stream priority: its CTAs take the slots the factorisation's
    // retiring CTAs free (kernels/ilut.cu launch_ilut) instead of queueing behind it.
    int prio_lo = 0, prio_hi = 0;
    ILUG_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    cudaStream_t bst = nullptr;
    ILUG_CUDA(cudaStreamCreateWithPriority(&bst, cudaStreamNonBlocking, prio_hi));
    struct Item {
        i64 k;
        const HostLevel* lev;
        bool last;
    };
    std::mutex qm;
    std::condition_variable qcv;
    std::deque<Item> queue;
    bool closed = false;
    std::exception_ptr build_err;
    DevFactors pre;
    bool have_pre = false;
    // With A shared on the device, level 0's operators are built from it as
    // soon as the AMG's level 0 is final, and its smoother once the factors
    // are (the builder does not wait for the factorisation before level 1).
    bool pending0 = false;
    const HostLevel* lev0 = nullptr;
    auto finish0 = [&](bool block) {
        if (!pending0 || (!block && f0.wait_for(std::chrono::seconds(0)) != std::future_status::ready)) return;
        pending0 = false;
        pre = f0.get();
        have_pre = true;
        dh.build_smoother0(*lev0, ap.plan.for_level(0), &pre, bst);
    };
    std::thread builder([&] {
        for (;;) {
            Item it{};
            bool done = false;
            {
                std::unique_lock<std::mutex> g(qm);
                qcv.wait(g, [&] { return closed || !queue.empty(); });
                if (queue.empty()) {
                    done = true;
                } else {
                    it = queue.front();
                    queue.pop_front();
                }
            }
            if (build_err) {
                if (done) return;
                continue; // drain after a failure
            }
            try {
                if (done) {
                    finish0(true);
                    return;
                }
                if (it.k == 0 && !it.last && f0.valid() && share_A) {
                    dh.build_level0_ops(*it.lev, Ad.rp.p, Ad.ci.p, Ad.v.p, bst);
                    pending0 = true;
                    lev0 = it.lev;
                } else {
                    DevFactors* l0 = nullptr;
                    if (it.k == 0 && !it.last && f0.valid()) { // the level-0 smoother uses the early factors
                        pre = f0.get();
                        have_pre = true;
                        l0 = &pre;
                    }
                    dh.build_level(static_cast<int>(it.k), *it.lev, ap.plan.for_level(it.k), it.last, l0, bst);
                }
                finish0(false);
            } catch (...) {
                build_err = std::current_exception();
                if (done) return;
            }
        }
    });
    auto close_queue = [&] {
        {
            std::lock_guard<std::mutex> g(qm);
            closed = true;
        }
        qcv.notify_all();
        builder.join();
        cudaStreamDestroy(bst);
    };
    // Galerkin products on the GPU (own stream), bitwise the host SpGEMM
    AmgParams apd = ap;
    cudaStream_t gst = nullptr;
    if (galerkin_on_device()) {
        ILUG_CUDA(cudaStreamCreateWithPriority(&gst, cudaStreamNonBlocking, prio_hi));
        apd.galerkin = [gst](const Csr& Ak, const Csr& P, const Csr& R) { return galerkin_device(Ak, P, R, gst); };
    }
    struct StreamGuard {
        cudaStream_t s;
        ~StreamGuard() {
            if (s) cudaStreamDestroy(s);
        }
    } gguard{gst};
    try {
        cudaStream_t sst = nullptr;
        if (dev_setup) ILUG_CUDA(cudaStreamCreateWithPriority(&sst, cudaStreamNonBlocking, prio_hi));
        StreamGuard sguard{sst};
        auto setup = [&](const LevelReady& cb) {
            return dev_setup ? amg_setup_device(A, apd, cb, sst, share_A ? &Ad : nullptr, keep_dev) : amg_setup(A, apd, cb);
        };
        oc.hier = setup([&](i64 k, const HostLevel& lev, bool last) {
            {
                std::lock_guard<std::mutex> g(qm);
                queue.push_back({k, &lev, last});
            }
            qcv.notify_one();
        });
    } catch (...) {
        close_queue();
        if (f0.valid()) f0.wait();
        throw;
    }
    tm.mark("hierarchy");
    close_queue();
    for (const HostLevel& l : oc.hier.levels) l.dA.reset(), l.dP.reset(), l.dR.reset(); // any the builder left
    tm.mark("device objects");
    if (f0.valid()) pre = f0.get(); // single-level hierarchies: still surface factorisation errors
    (void)have_pre;
    if (build_err) std::rethrow_exception(build_err);
    dh.finish(oc.hier, st);
    // device-side setup that the first iteration would otherwise pay inside the
    // timed solve: the V-cycle graph and the GMRES basis (multi-GB at C2)
    dh.prepare_graph();
    tm.mark("graph");
    GmresWork gw;
    if (kp.restart >= 1) gw.ensure(A.nrows, kp.restart, kp.flexible, kp.max_iters); // else gmres reports it
    defer.reset();
    tm.mark("gmres basis + frees");
    oc.setup_seconds = since(t0);

    const i64 n = A.nrows;
    DBuf<double> db, dx(n);
    db.upload(b.data(), n, st);
    vec_zero(dx.p, n, st);
    ILUG_CUDA(cudaStreamSynchronize(st));
    // Fast mode (x formed once per cycle, relres criterion): nothing in the
    // solve consumes |A|_2, so its estimate (only the reported NRBE uses it) is
    // taken after the timed region. Reference mode keeps it inside, like
    // gmres_impl (src/krylov.cpp:86).
    KrylovParams kpr = kp;
    const bool late_anorm = !kp.form_iterates && !kp.nrbe_criterion;
    if (late_anorm) kpr.estimate_anorm = false;
    const auto t1 = std::chrono::steady_clock::now();
    oc.kr = device_gmres(dh.A0(), &A, vcycle_of(dh), db.p, dx.p, kpr, st, nullptr, &gw);
    ILUG_CUDA(cudaStreamSynchronize(st));
    oc.solve_seconds = since(t1);
    oc.x.resize(static_cast<size_t>(n));
    dx.download(oc.x.data(), st);
    ILUG_CUDA(cudaStreamSynchronize(st));
    if (late_anorm) {
        oc.kr.anorm_estimate = device_estimate_two_norm(dh.A0(), A, 50, kp.anorm_seed, st);
        double xn = 0.0;
        for (double v : oc.x) xn += v * v;
        const double tr = oc.kr.final_relres * (oc.kr.bnorm > 0.0 ? oc.kr.bnorm : 1.0);
        const double den = oc.kr.bnorm + oc.kr.anorm_estimate * std::sqrt(xn);
        oc.kr.final_nrbe = den == 0.0 ? 0.0 : tr / den;
    }
    oc.graph_nodes = dh.kernels_per_cycle();
    if (dh.num_levels() > 1 && dh.smoother(0).schur())
        oc.schur_interface = dh.smoother(0).schur()->interface_size();
    return oc;
}

void solve_scalars(Report& r, const SolveOutcome& oc, const KrylovParams& kp) {
    r.add("method", kp.flexible ? "fgmres" : "gmres");
    r.add("criterion", kp.nrbe_criterion ? "nrbe" : "relres");
    r.add("tol", kp.tol);
    r.add("iterations", oc.kr.iterations);
    r.add("converged", oc.kr.converged);
    r.add("false_convergence", oc.kr.false_convergence);
    r.add("final_relres", oc.kr.final_relres);
    r.add("final_nrbe", oc.kr.final_nrbe);
    r.add("anorm_estimate", oc.kr.anorm_estimate);
    r.add("levels", oc.hier.num_levels());
    r.add("operator_complexity", oc.hier.operator_complexity());
    const FlopsModel fm = flops_model(oc.hier);
    r.add("flops_smoothing", static_cast<i64>(fm.smoothing));
    r.add("flops_coarse_solve", static_cast<i64>(fm.coarse_solve));
    r.add("flops_krylov_spmv", static_cast<i64>(fm.krylov_spmv));
    r.add("setup_seconds", oc.setup_seconds);
    r.add("solve_seconds", oc.solve_seconds);
}

void device_scalars(Report& r, const SolveOutcome& oc) {
    int dev = 0;
    cudaGetDevice(&dev);
    r.add("device", static_cast<i64>(dev));
    r.add("device_vcycles", oc.kr.vcycles);
    r.add("vcycle_graph_nodes", oc.graph_nodes);
}

void history_tables(Report& r, const SolveOutcome& oc) {
    const double bden = oc.kr.bnorm > 0.0 ? oc.kr.bnorm : 1.0;
    ReportTable h;
    h.name = "history";
    h.columns = {"iter", "arnoldi_rel", "true_rel", "nrbe"};
    for (const auto& e : oc.kr.history)
        h.rows.push_back({std::to_string(e.iter), format_num(e.arnoldi / bden), format_num(e.true_res / bden),
                          format_num(e.nrbe)});
    r.tables.push_back(std::move(h));
    ReportTable lv;
    lv.name = "hierarchy";
    lv.columns = {"level", "n", "nnz"};
    for (i64 k = 0; k < oc.hier.num_levels(); ++k)
        lv.rows.push_back({std::to_string(k), std::to_string(oc.hier.levels[k].A.nrows),
                           std::to_string(oc.hier.levels[k].A.nnz())});
    r.tables.push_back(std::move(lv));
}

} // namespace

std::string format_num(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.16e", v);
    return buf;
}

std::string ReportTable::csv() const {
    std::ostringstream o;
    for (size_t c = 0; c < columns.size(); ++c) o << columns[c] << (c + 1 < columns.size() ? "," : "");
    o << "\n";
    for (const auto& row : rows) {
        for (size_t c = 0; c < row.size(); ++c) o << row[c] << (c + 1 < row.size() ? "," : "");
        o << "\n";
    }
    return o.str();
}

void Report::add(const std::string& k, double v) { add(k, format_num(v)); }

const std::string* Report::find(const std::string& k) const {
    for (const auto& [key, v] : scalars)
        if (key == k) return &v;
    return nullptr;
}

std::string Report::text() const {
    std::ostringstream o;
    for (const auto& [k, v] : scalars) o << k << " = " << v << "\n";
    return o.str();
}

std::string Report::json() const {
    auto esc = [](const std::string& s) {
        std::string r;
        for (char c : s) {
            if (c == '"' || c == '\\') r += '\\';
            r += c;
        }
        return r;
    };
    std::ostringstream o;
    o << "{";
    bool first = true;
    for (const auto& [k, v] : scalars) {
        if (!first) o << ",";
        first = false;
        o << "\"" << esc(k) << "\":\"" << esc(v) << "\"";
    }
    o << "}";
    return o.str();
}

DeviceContext::DeviceContext(const Config& c) {
    const i64 dev = c.get_index("device.id");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        fail_invalid("no CUDA device is available (this build has no CPU path)");
    if (dev < 0 || dev >= count) fail_invalid("config: device.id out of range");
    ILUG_CUDA(cudaSetDevice(static_cast<int>(dev)));
    ILUG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
}

DeviceContext::~DeviceContext() {
    if (stream) cudaStreamDestroy(stream);
}

Report run_solve(const Csr& A, const Config& cfg, const std::string& label) {
    const AmgParams ap = amg_params_from(cfg);
    const KrylovParams kp = krylov_from(cfg);
    const Vec b = make_rhs(cfg, A);
    DeviceContext ctx(cfg);
    const SolveOutcome oc = solve_with(A, ap, kp, b, cfg.get_bool("device.graph"), ctx.stream);
    Report r;
    r.status = oc.kr.converged ? 0 : 1;
    r.add("matrix", label);
    r.add("n", A.nrows);
    r.add("nnz", A.nnz());
    solve_scalars(r, oc, kp);
    if (cfg.get("rhs") == "ones-times-A") {
        double err = 0.0;
        for (double v : oc.x) err = std::max(err, std::abs(v - 1.0));
        r.add("ones_solution_inf_err", err);
    }
    device_scalars(r, oc);
    history_tables(r, oc);
    return r;
}

namespace {

double dev_norm2(const double* v, i64 n, double* scratch, cudaStream_t st) {
    nrm2sq_dev(v, n, scratch, scratch + 1, st);
    double h = 0.0;
    ILUG_CUDA(cudaMemcpyAsync(&h, scratch, sizeof h, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(h);
}

// neumann_tail_norm (src/trisolve.cpp:158-180) with the products on the device.
double tail_norm(const Sell& T, i64 p, i64 probes, std::uint64_t seed, double* scratch, cudaStream_t st) {
    const i64 n = T.nrows;
    if (p >= n) return 0.0;
    DBuf<double> v(n), t(n);
    double best = 0.0;
    for (i64 s = 0; s < probes; ++s) {
        Vec h = random_uniform(n, seed + static_cast<std::uint64_t>(s));
        double nr = 0.0;
        for (double x : h) nr += x * x;
        nr = std::sqrt(nr);
        if (nr > 0.0)
            for (double& x : h) x /= nr;
        v.upload(h.data(), n, st);
        for (i64 k = 0; k < p; ++k) {
            spmv(T, v.p, t.p, st);
            std::swap(v.p, t.p);
        }
        best = std::max(best, dev_norm2(v.p, n, scratch, st));
    }
    return best;
}

} // namespace

Report run_bench_trisolve(const Csr& A, const Config& cfg, const std::string& label) {
    const IluParams ip = ilu_params_from(cfg);
    ScalingKind sc = scaling_from(cfg);
    if (sc == ScalingKind::none) sc = ScalingKind::row;
    const i64 m_max = cfg.get_index("bench.m_max");
    const auto seed = static_cast<std::uint64_t>(cfg.get_index("bench.seed"));
    const i64 probes = cfg.get_index("bench.probes");
    if (m_max < 1) fail_invalid("bench-trisolve: bench.m_max must be >= 1");
    DeviceContext ctx(cfg);
    cudaStream_t st = ctx.stream;
    const HostFactors f = factorize(A, ip, st);
    DeviceIlu dev;
    dev.build(f, sc, UpperIteration::scaled, true, st);
    const i64 n = A.nrows;
    const Vec bh = random_uniform(n, seed);
    DBuf<double> b, yl(n), yu(n), z(n), d(n), ws(std::max<i64>(dev.sweep_ws(m_max) + n, 3)), scr(1 + reduce_ws_doubles(n));
    b.upload(bh.data(), n, st);
    dev.solve_lower(b.p, yl.p, st);
    dev.solve_upper(b.p, yu.p, ws.p, st);
    const double nl = dev_norm2(yl.p, n, scr.p, st), nu = dev_norm2(yu.p, n, scr.p, st);
    auto rel = [&](const double* a, const double* ref, double refn) {
        vec_sub_into(d.p, a, ref, n, st);
        const double e = dev_norm2(d.p, n, scr.p, st);
        return refn > 0.0 ? e / refn : e;
    };
    ReportTable t;
    t.name = "bench";
    t.columns = {"factor", "m", "err_direct_rel", "tail_norm_estimate"};
    for (i64 m = 1; m <= m_max; ++m) {
        dev.sweep_lower(b.p, z.p, m, ws.p, st);
        t.rows.push_back({"L", std::to_string(m), format_num(rel(z.p, yl.p, nl)),
                          format_num(tail_norm(dev.Ls(), m, probes, seed, scr.p, st))});
    }
    for (i64 m = 1; m <= m_max; ++m) {
        dev.sweep_upper(b.p, z.p, m, ws.p, st);
        t.rows.push_back({"U", std::to_string(m), format_num(rel(z.p, yu.p, nu)),
                          format_num(tail_norm(dev.Us(), m, probes, seed, scr.p, st))});
    }
    Report r;
    r.add("matrix", label);
    r.add("n", n);
    r.add("variant", ip.variant == IluVariant::ilu0 ? "ilu0" : "ilut");
    r.add("scaling", sc == ScalingKind::row ? "row" : "row_col");
    r.add("m_max", m_max);
    r.tables.push_back(std::move(t));
    return r;
}

// run_schur_solve (src/driver.cpp:318-375): one solve per block count of
// schur.blocks_list with the Schur smoother on the finest level, FGMRES forced
// (the one-step interface GMRES makes the preconditioner nonstationary).
Report run_schur_solve(const Csr& A, const Config& cfg, const std::string& label) {
    std::vector<i64> blocks;
    {
        std::string list = cfg.get("schur.blocks_list");
        for (char& c : list)
            if (c == ',') c = ' ';
        std::istringstream in(list);
        i64 p = 0;
        while (in >> p) blocks.push_back(p);
        if (blocks.empty()) fail_invalid("schur-solve: schur.blocks_list is empty");
    }
    KrylovParams kp = krylov_from(cfg);
    kp.flexible = true;
    const Vec b = make_rhs(cfg, A);
    DeviceContext ctx(cfg);
    Report r;
    r.add("matrix", label);
    r.add("n", A.nrows);
    r.add("nnz", A.nnz());
    r.add("method", "fgmres");
    ReportTable t;
    t.name = "schur";
    t.columns = {"p", "interface_size", "iterations", "converged", "final_relres", "final_nrbe"};
    i64 it_min = -1, it_max = -1;
    for (i64 p : blocks) {
        AmgParams ap = amg_params_from(cfg);
        ap.plan.finest = schur_smoother_from(cfg);
        ap.plan.finest.schur_blocks = p;
        ap.plan.finest_levels = 1;
        const SolveOutcome oc = solve_with(A, ap, kp, b, cfg.get_bool("device.graph"), ctx.stream);
        t.rows.push_back({std::to_string(p), std::to_string(oc.schur_interface), std::to_string(oc.kr.iterations),
                          oc.kr.converged ? "true" : "false", format_num(oc.kr.final_relres),
                          format_num(oc.kr.final_nrbe)});
        if (!oc.kr.converged) r.status = 1;
        if (it_min < 0 || oc.kr.iterations < it_min) it_min = oc.kr.iterations;
        if (it_max < 0 || oc.kr.iterations > it_max) it_max = oc.kr.iterations;
    }
    r.add("iterations_min", it_min);
    r.add("iterations_max", it_max);
    r.add("iterations_spread", it_max - it_min);
    r.tables.push_back(std::move(t));
    return r;
}


} // namespace ilug
