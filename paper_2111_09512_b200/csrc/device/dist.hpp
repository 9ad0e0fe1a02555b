// Multi-GPU solve phase (device/dist.cu): the transports that move data
// between ranks, and the row-block distributed smoother, V-cycle and GMRES.
//
// Layout: every operator of the hierarchy is row-block
// partitioned (src/schur.cpp:28-33 rule, per level). Before each global
// product — the residual with A_k, the restriction R_k r, the prolongation
// P_k e — the entries of the input vector other ranks own are exchanged
// (HaloExchange, global entry order kept, so every product is bitwise the
// single-process one). Smoothers are rank-local: block-Jacobi ILU on the
// diagonal block (north star), hybrid Gauss-Seidel (GS on the diagonal block
// after the off-block part of the row is subtracted with the current halo),
// block poly-GS, and global Jacobi / l1-Jacobi. The coarsest right-hand side is
// all-gathered and solved redundantly on every rank. GMRES reductions are
// summed over ranks.
#pragma once

#include "../host/dist.hpp"
#include "solver.hpp"

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>

namespace ilug {

/// ncclUniqueId bytes for ncclCommInitRank (rank 0 creates, the caller broadcasts).
void dist_unique_id(char out[128]);

/// Data movement between the ranks of one job.
///  * NCCL: one process per GPU, grouped ncclSend/ncclRecv for halos and
///    ncclAllReduce for sums, stream-ordered (the product path).
///  * Local: the ranks are host threads of one process (any devices). Each
///    call synchronises the caller's stream, meets the other ranks at a host
///    barrier and copies peer buffers directly. No kernel ever waits on
///    another rank's kernel, so several ranks can share one GPU: the
///    single-GPU test stand-in for the multi-GPU path.
class Transport {
public:
    virtual ~Transport() = default;
    int nranks = 1, rank = 0;
    virtual void allreduce_sum(double* buf, i64 count, cudaStream_t st) const = 0;
    /// hx.sendbuf segments to hx.send_ranks; hx.halo segments from hx.recv_ranks
    virtual void exchange(const HaloExchange& hx, cudaStream_t st) const = 0;
    /// every rank's byte string, in rank order (host, blocking, collective)
    virtual std::vector<std::vector<char>> allgather(const std::vector<char>& mine) const = 0;
};

std::unique_ptr<Transport> make_nccl_transport(int nranks, int rank, const char id[128]);

/// Shared state of an in-process rank group.
class LocalGroup {
public:
    explicit LocalGroup(int nranks);
    int size() const { return p_; }
    /// Throws once abort() was called: a rank that failed releases the others.
    void barrier();
    void abort();
    std::vector<const void*> slot;    ///< per-rank published pointer of the current collective
    std::vector<std::vector<double>> stage; ///< per-rank host staging (allreduce)

private:
    int p_;
    std::mutex m_;
    std::condition_variable cv_;
    int arrived_ = 0;
    unsigned long long gen_ = 0;
    bool aborted_ = false;
};
std::unique_ptr<Transport> make_local_transport(std::shared_ptr<LocalGroup> g, int rank);

/// One rank's handle on a transport (what the GMRES reductions use).
struct DistComm {
    std::unique_ptr<Transport> t;
    int nranks = 1, rank = 0;
    explicit DistComm(std::unique_ptr<Transport> tr) : t(std::move(tr)), nranks(t->nranks), rank(t->rank) {}
    DistComm(const DistComm&) = delete;
    DistComm& operator=(const DistComm&) = delete;
    void allreduce_sum(double* buf, i64 count, cudaStream_t st) const {
        if (nranks > 1) t->allreduce_sum(buf, count, st);
    }
};

/// Complete a plan's send lists over the transport (collective): every rank
/// learns which of its rows the others read.
void plan_exchange(HaloPlan& plan, const Transport& t);

/// Device side of a plan: pack buffers, halo buffer, the extended operator.
struct DistOperator {
    HaloExchange hx;
    DeviceMatrix M;
    void build(const HaloPlan& plan, const Transport& t, cudaStream_t st);
};

/// Block-Jacobi ILU (or any distributed smoother kind) of a row-block
/// distributed matrix: global residual, rank-local factors.
class DistSmoother {
public:
    void build(const HaloPlan& plan, const DistComm& comm, const SmootherConfig& cfg, cudaStream_t st);
    void smooth(const double* b, double* x, cudaStream_t st) const { s_.smooth(b, x, false, st); }
    void residual(const double* x, const double* b, double* r, cudaStream_t st) const { op_.M.residual(x, b, r, st); }
    const DeviceSmoother& smoother() const { return s_; }
    i64 nloc() const { return op_.M.n; }

private:
    DistOperator op_;
    DeviceSmoother s_;
};

/// The AMG V-cycle of a row-block distributed hierarchy (cycle_level,
/// src/amg.cpp:394-418, per rank).
class DistHierarchy {
public:
    /// h: the global host hierarchy (every rank holds the same one).
    void build(const HostHierarchy& h, const DistComm& comm, cudaStream_t st);
    /// z = M(r) on this rank's rows (z zeroed first, src/driver.cpp:182-185). Collective.
    void vcycle(const double* r, double* z, cudaStream_t st);
    int num_levels() const { return nlev_; }
    i64 nloc() const { return levels_.empty() ? coarse_A_.M.n : levels_[0].A.M.n; }
    i64 row0() const { return row0_; }
    /// level-0 operator (this rank's rows, halo-exchanged products)
    const DeviceMatrix& A0() const { return levels_.empty() ? coarse_A_.M : levels_[0].A.M; }

private:
    struct Lev {
        i64 n = 0, row0 = 0;
        bool last = false;
        DistOperator A, R, P;
        Sell R_full, P_rows; // last smoothed level
        DeviceSmoother smoother;
        DBuf<double> b, x, r;
    };
    void cycle(int k, bool x_zero, cudaStream_t st);
    const DistComm* comm_ = nullptr;
    std::deque<Lev> levels_;
    int nlev_ = 0;
    i64 nu_ = 1, row0_ = 0;
    // coarsest level, replicated: dense LU, full rhs/solution, gathered residual of the level above
    i64 coarse_n_ = 0;
    DBuf<double> lu_, cb_, cx_, gather_;
    DBuf<i64> piv_;
    DistOperator coarse_A_; // single-level hierarchies: this rank's rows of the only level
};

/// Row-block distributed GMRES+AMG: global (F)GMRES over the ranks' rows
/// (halo-exchanged SpMV, summed CGS2 reductions) preconditioned by the
/// distributed V-cycle.
class DistSolver {
public:
    void build(const HostHierarchy& h, const DistComm& comm, cudaStream_t st);
    KrylovReport solve(const double* b, double* x, const KrylovParams& p, cudaStream_t st);
    void vcycle(const double* r, double* z, cudaStream_t st) { H_.vcycle(r, z, st); }
    i64 nloc() const { return H_.nloc(); }
    i64 row0() const { return H_.row0(); }
    int levels() const { return H_.num_levels(); }

private:
    const DistComm* comm_ = nullptr;
    DistHierarchy H_;
    GmresWork work_;
};

} // namespace ilug
