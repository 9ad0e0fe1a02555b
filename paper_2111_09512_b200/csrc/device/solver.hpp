// Device-resident solve phase: ILU factors (K1-K5), smoothers (K4 + the
// fallback family), the AMG V-cycle (K6/K7) and (F)GMRES with CGS2 (K8).
//
// Reference anchors: SmootherState/build_smoother_state/smooth
// (include/iluamg/smoother.hpp:33-49, src/smoother.cpp:49-187), cycle_level
// (src/amg.cpp:394-418), gmres_impl (src/krylov.cpp:75-238). Setup-phase data
// (factors, hierarchy) comes from the host (csrc/host/), is uploaded once and is
// read-only afterwards, so handles can be shared by concurrent solves on
// different streams (the reference's threading contract, README.md:152-154).
#pragma once

#include "../host/amg.hpp"
#include "../host/dist.hpp"
#include "../host/schur.hpp"
#include "../kernels/ilu0.hpp"
#include "../kernels/levelset.hpp"
#include "../kernels/wavefront.hpp"
#include "spsv_cusparse.hpp"

#include <deque>
#include <functional>
#include <memory>

namespace ilug {

struct DevCsr; // kernels/spgemm.hpp

class Transport;

/// Device side of a HaloPlan (host/dist.hpp): packs the rows other ranks need
/// and hands the segments to the job's transport (device/dist.cu). The
/// transfer runs on the exchange's own stream: begin() packs on the caller's
/// stream and starts the transport behind an event, end() makes the caller's
/// stream wait for the halo — the split products launch their local-only rows
/// in between (HaloWait), so those rows overlap the exchange.
struct HaloExchange {
    const Transport* tr = nullptr;
    i64 nloc = 0, nhalo = 0; ///< owned columns (split point of the extended operator), halo entries
    std::vector<i64> recv_ranks, recv_offsets, send_ranks, send_offsets;
    DBuf<i32> send_idx;
    mutable DBuf<double> sendbuf, halo;
    HaloExchange() = default;
    HaloExchange(const HaloExchange&) = delete;
    HaloExchange& operator=(const HaloExchange&) = delete;
    ~HaloExchange();
    void setup(const HaloPlan& plan, const Transport& t, cudaStream_t st);
    void begin(const double* x_local, cudaStream_t st) const;
    void end(cudaStream_t st) const;
    /// end() as the split products' mid-launch callback
    HaloWait waiter() const { return {&HaloExchange::end_cb, this}; }
    void exchange(const double* x_local, cudaStream_t st) const {
        begin(x_local, st);
        end(st);
    }

private:
    static void end_cb(const void* self, cudaStream_t st) { static_cast<const HaloExchange*>(self)->end(st); }
    cudaStream_t cst_ = nullptr;
    cudaEvent_t packed_ = nullptr, done_ = nullptr;
    mutable bool pending_ = false;
};
/// Sum over the transport's ranks (no-op for null / one rank).
void transport_allreduce(const Transport* t, double* buf, i64 count, cudaStream_t st);

/// Device copy of an operator. With a halo, the rows are a rank's rows of a
/// distributed matrix whose columns >= n index the halo buffer.
struct DeviceMatrix {
    Sell A;
    i64 n = 0;
    const HaloExchange* halo = nullptr;
    void build(const Csr& host, cudaStream_t st);
    /// From a device CSR copy of `host` (same rows/columns/values).
    void build(const Csr& host, const i64* rp, const i32* ci, const double* v, cudaStream_t st);
    void residual(const double* x, const double* b, double* r, cudaStream_t st) const;
    void spmv(const double* x, double* y, cudaStream_t st) const;
};

/// K1-K5: scaled ILU factors on the device plus the sweep/solve entry points.
class DeviceIlu {
public:
    /// Uploads L (strict) and U (with diagonal), applies `scaling` with the K1
    /// kernel, packs strict parts into SELL. Level plans are built when
    /// `direct_plans` is set (trisolve.mode=direct or explicit sptrsv use).
    void build(const HostFactors& f, ScalingKind scaling, UpperIteration upper, bool direct_plans,
               cudaStream_t st);
    /// Same from device-resident factors (consumed: U is scaled in place and
    /// packed, then the CSR copies are freed). No host round trip of the
    /// factors unless a wavefront or level-set plan needs the patterns.
    void build(DevFactors&& f, ScalingKind scaling, UpperIteration upper, bool direct_plans, cudaStream_t st);
    /// Numeric refactorisation: new factors with the pattern these were built
    /// from (Ilu0Symbolic::factor) — K1 scaling and every SELL copy (sweeps,
    /// level plans) refilled in place, no layout work, no host round trip.
    void refactor(DevFactors&& f, cudaStream_t st);

    i64 n() const { return n_; }
    ScalingKind scaling() const { return scaling_; }
    bool has_rs() const { return rs_.n > 0; }
    bool has_cs() const { return cs_.n > 0; }
    const double* rs() const { return rs_.p; }
    const double* cs() const { return cs_.p; }
    const double* diag() const { return d_.p; }
    const Sell& Ls() const { return Ls_; }
    const Sell& Us() const { return Us_; }
    UpperIteration upper_iteration() const { return upper_; }

    /// richardson_lower (src/trisolve.cpp:94-104): y = m sweeps from 0.
    /// ws: sweep_ws(m) doubles.
    void sweep_lower(const double* b, double* y, i64 m, double* ws, cudaStream_t st) const;
    /// richardson_upper_scaled (src/trisolve.cpp:132-147) or its Jacobi form on the
    /// unscaled factor: x = m sweeps from 0 (pre/post scaling included).
    /// ws: sweep_ws(m) + n doubles.
    void sweep_upper(const double* b, double* x, i64 m, double* ws, cudaStream_t st) const;
    /// Workspace (doubles) of sweep_lower with m sweeps; sweep_upper needs n more.
    i64 sweep_ws(i64 m) const {
        return ((wave_L_.ready() || wave_U_.ready()) ? std::max<i64>(2, m) : 2) * n_;
    }
    /// m sweeps of the U (upper) or L factor run as one wavefront launch
    /// (m-1 fused sweeps after the first).
    bool use_wave(bool upper, i64 m) const;
    const WavePlan& wave_L() const { return wave_L_; }
    const WavePlan& wave_U() const { return wave_U_; }
    /// Level-scheduled direct solves: solve_lower_direct and
    /// solve_upper_scaled_direct / solve_upper_direct (src/trisolve.cpp:20-55,149-156). ws: n.
    void solve_lower(const double* b, double* y, cudaStream_t st) const;
    void solve_upper(const double* b, double* x, double* ws, cudaStream_t st) const;
    bool has_plans() const { return lower_plan_.levels() > 0 || n_ == 0; }
    const LevelPlan& lower_plan() const { return lower_plan_; }
    const LevelPlan& upper_plan() const { return upper_plan_; }
    /// The triangular solves behind solve_lower/solve_upper without the scaling
    /// steps: K5 level schedules, or cuSPARSE SpSV under ILUG_DIRECT=cusparse.
    void lower_direct(const double* b, double* y, cudaStream_t st) const;
    void upper_direct(const double* b, double* x, cudaStream_t st) const;

    /// Download the scaled factor U (unit diagonal re-inserted) for parity tests.
    Csr scaled_upper_host() const;
    Vec download(const DBuf<double>& b) const;
    const DBuf<double>& rs_buf() const { return rs_; }
    const DBuf<double>& cs_buf() const { return cs_; }

private:
    void finish(DevFactors& df, const HostFactors* host, ScalingKind scaling, UpperIteration upper,
                bool direct_plans, cudaStream_t st);

    i64 n_ = 0;
    ScalingKind scaling_ = ScalingKind::row;
    UpperIteration upper_ = UpperIteration::scaled;
    Sell Ls_, Us_;          // strict parts (Us_ scaled unless upper_ == jacobi)
    DBuf<double> rs_, cs_, d_;
    LevelPlan lower_plan_, upper_plan_;
    std::unique_ptr<CusparseTri> cs_lower_, cs_upper_; // ILUG_DIRECT=cusparse
    WavePlan wave_L_, wave_U_; // fused multi-sweep plans (large n only, see wave_enabled)
};

/// K9: the ILUT Schur-complement smoother (src/schur.cpp:137-219) on the device.
/// Block solves run on the block-diagonal factor of the interior unknowns (all
/// blocks at once; rows never couple across blocks, so this is exactly the
/// reference's per-block loop); the one-step interface GMRES keeps its scalars
/// (beta, h11, h21^2, alpha) in device memory, so an application never syncs
/// the host and can live inside the V-cycle graph.
class DeviceSchur {
public:
    void build(const Csr& A, const SmootherConfig& cfg, cudaStream_t st);
    /// Distributed form (schur.blocks = ranks, block b = rank b's rows): B, E,
    /// F are block-local; C couples the ranks' interface unknowns (halo
    /// exchange); beta^2, h11, h21^2 are summed over the ranks (collective).
    void build_dist(const HaloPlan& A, const Transport& t, const SmootherConfig& cfg, cudaStream_t st);
    /// x <- schur_smooth(A, b, x)
    void apply(const DeviceMatrix& A, const double* b, double* x, cudaStream_t st) const;
    i64 interface_size() const { return nf_; }
    i64 interior_size() const { return ni_; }

private:
    void block_solve(const double* f, double* out, cudaStream_t st) const;
    void finish_build(const Csr& B, const Csr& E, const Csr& F, const std::vector<i32>& perm, const SmootherConfig& cfg,
                      cudaStream_t st, SchurSetup* host);
    i64 n_ = 0, ni_ = 0, nf_ = 0, nf_global_ = 0;
    TriSolveConfig ts_;
    DeviceIlu blocks_;
    Sell E_, F_, C_;
    const Transport* tr_ = nullptr; // distributed: C's halo exchange and the scalar sums
    HaloExchange Chx_;
    DBuf<i32> perm_;
    mutable DBuf<double> ws_, red_, scal_;
};

/// One level's smoother (src/smoother.cpp:161-187 `smooth`).
class DeviceSmoother {
public:
    /// `pre`: factors of A computed ahead (moved from; ILU kinds only).
    /// `dist`: dA holds a rank's rows of a distributed operator (dA.halo set) —
    /// A is then the plan's diagonal block and the smoother is its rank-local
    /// form (block-Jacobi ILU / poly-GS, hybrid GS, global Jacobi / l1).
    /// `dcsr`: a device copy of A (the device AMG setup's), used where a
    /// smoother would otherwise re-upload A (poly-GS: diagonal and strict lower part).
    void build(const Csr& A, const DeviceMatrix& dA, const SmootherConfig& cfg, cudaStream_t st,
               DevFactors* pre = nullptr, const HaloPlan* dist = nullptr, const DevCsr* dcsr = nullptr);
    /// x <- smooth(A, b, x). `x_zero`: caller guarantees x == 0 on entry, so the
    /// first residual is b itself (bitwise what the SpMV would give).
    void smooth(const double* b, double* x, bool x_zero, cudaStream_t st) const;
    /// One ilu_smooth_sweep (src/smoother.cpp:143-159).
    void ilu_sweep(const double* b, double* x, bool x_zero, cudaStream_t st) const;
    const SmootherConfig& config() const { return cfg_; }
    const DeviceIlu* ilu() const { return ilu_.get(); }
    const DeviceSchur* schur() const { return schur_.get(); }
    i64 n() const { return n_; }

private:
    SmootherConfig cfg_;
    i64 n_ = 0;
    const DeviceMatrix* A_ = nullptr;
    std::unique_ptr<DeviceIlu> ilu_;
    std::unique_ptr<DeviceSchur> schur_;
    std::unique_ptr<LevelPlan> gs_;
    Sell Lstrict_;               // poly_gs
    Sell Aoff_;                  // hybrid GS: the rows' off-block entries (halo columns)
    DBuf<double> invd_;          // jacobi / l1 / poly_gs
    mutable DBuf<double> ws_;    // workspace (r, y ping-pong, bs, x ping-pong)
};

/// The AMG V-cycle on the device, optionally replayed as one CUDA graph.
class DeviceHierarchy {
public:
    /// `level0`: the finest level's ILU factors computed ahead (see solve_with).
    void build(const HostHierarchy& h, cudaStream_t st, DevFactors* level0 = nullptr);
    /// Incremental form of build(): begin(), then build_level() for k = 0, 1, ...
    /// in order (each as soon as the host level is final), then finish(h).
    void begin();
    void build_level(int k, const HostLevel& hl, const SmootherConfig& sc, bool last, DevFactors* level0,
                     cudaStream_t st);
    /// Level 0's operators from a device copy of A (rp, ci, v) with its
    /// smoother left for build_smoother0() (the factors are still computing).
    void build_level0_ops(const HostLevel& hl, const i64* rp, const i32* ci, const double* v, cudaStream_t st);
    void build_smoother0(const HostLevel& hl, const SmootherConfig& sc, DevFactors* level0, cudaStream_t st);
    void finish(const HostHierarchy& h, cudaStream_t st);
    /// z = M(r) with z zeroed first (the driver's precond lambda, src/driver.cpp:182-185).
    void vcycle(const double* r, double* z, cudaStream_t st);
    /// Capture and instantiate the V-cycle graph now (setup) instead of on the
    /// first vcycle() call.
    void prepare_graph();
    /// Same, without graph replay (direct kernel launches).
    void vcycle_eager(const double* r, double* z, cudaStream_t st);
    i64 n() const { return levels_.empty() ? 0 : levels_[0].n; }
    int num_levels() const { return static_cast<int>(levels_.size()); }
    const DeviceMatrix& A0() const { return levels_[0].A; }
    const DeviceSmoother& smoother(int k) const { return levels_[k].smoother; }
    void set_use_graph(bool g) { use_graph_ = g; }
    i64 kernels_per_cycle() const { return kernels_per_cycle_; }

private:
    struct Lev {
        i64 n = 0;
        DeviceMatrix A;
        Sell P, R;
        DeviceSmoother smoother;
        DBuf<double> b, x, r;
    };
    void cycle(int k, bool x_zero, cudaStream_t st);
    std::deque<Lev> levels_; // stable addresses: smoothers point at their level's operator
    DBuf<double> lu_;
    DBuf<i64> piv_;
    i64 nu_ = 1;
    bool use_graph_ = true;
    bool trace_ = false; // ILUG_TRACE (eager only): per-level phase times on stderr
    cudaGraphExec_t exec_ = nullptr;
    cudaStream_t graph_stream_ = nullptr;
    i64 kernels_per_cycle_ = 0;

public:
    DeviceHierarchy() = default;
    DeviceHierarchy(const DeviceHierarchy&) = delete;
    DeviceHierarchy& operator=(const DeviceHierarchy&) = delete;
    ~DeviceHierarchy();
};

struct KrylovParams {
    bool flexible = false;
    i64 restart = 50;
    i64 max_iters = 200;
    double tol = 1e-5;
    bool nrbe_criterion = false;
    bool record_history = true;
    std::uint64_t anorm_seed = 7;
    /// Reference behaviour: form x_k every iteration (non-flexible GMRES applies
    /// the preconditioner a second time, src/krylov.cpp:204-214) and record the
    /// true residual / NRBE. false = form x only at the end of each restart
    /// cycle (iteration counts unchanged under the relres criterion).
    bool form_iterates = true;
    bool estimate_anorm = true;
};

struct HistoryEntry {
    i64 iter = 0;
    double arnoldi = 0.0, true_res = 0.0, nrbe = 0.0;
};

struct KrylovReport {
    i64 iterations = 0;
    std::vector<HistoryEntry> history;
    bool converged = false, false_convergence = false;
    double anorm_estimate = 0.0, bnorm = 0.0, final_relres = 0.0, final_nrbe = 0.0;
    i64 vcycles = 0;
};

/// Right-preconditioned (F)GMRES on the device, CGS2 orthogonalisation; the
/// Hessenberg/Givens/solve_y scalars stay on the device (one status read per
/// iteration for the convergence test), any restart >= 1.
struct DistComm;
/// comm != nullptr: A holds this rank's rows (halo-exchanged SpMV), vectors are
/// rank-local, every reduction is summed over ranks (NCCL allreduce), and M is
/// this rank's block-Jacobi AMG hierarchy.
/// GMRES work vectors (basis V, flexible Z, temporaries): allocated at setup
/// by solve_with so the multi-GB basis allocation is not inside the timed solve.
struct GmresWork {
    DBuf<double> V, Z, w, r, xk, xc, vy, mz;
    DBuf<double> S, hist, ws; ///< device scalars (H, rotations, g, y), history norms, reductions
    double* stat = nullptr;   ///< pinned host status (8 doubles)
    i64 R_ = 0;
    GmresWork() = default;
    GmresWork(const GmresWork&) = delete;
    GmresWork& operator=(const GmresWork&) = delete;
    ~GmresWork();
    void ensure(i64 n, i64 restart, bool flexible, i64 max_iters = 200);
};
/// The preconditioner z = M(r) (the reference's LinearOperator,
/// include/iluamg/krylov.hpp:20): a V-cycle on this stream.
using Preconditioner = std::function<void(const double* r, double* z, cudaStream_t st)>;
/// A_host: the operator on the host for the |A|_2 power iteration (null: not estimated).
KrylovReport device_gmres(const DeviceMatrix& A, const Csr* A_host, const Preconditioner& M,
                          const double* b_dev, double* x_dev, const KrylovParams& p, cudaStream_t st,
                          const DistComm* comm = nullptr, GmresWork* work = nullptr);
inline Preconditioner vcycle_of(DeviceHierarchy& H) {
    return [&H](const double* r, double* z, cudaStream_t st) { H.vcycle(r, z, st); };
}

/// 50-step power iteration on A^T A (src/krylov.cpp:14-28) on the device.
double device_estimate_two_norm(const DeviceMatrix& A, const Csr& A_host, i64 steps,
                                std::uint64_t seed, cudaStream_t st);

} // namespace ilug
