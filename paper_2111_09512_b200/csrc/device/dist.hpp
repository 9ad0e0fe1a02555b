// Multi-GPU solve-phase objects (device/dist.cu).
#pragma once

#include "../host/dist.hpp"
#include "solver.hpp"

#include <cstring>

namespace ilug {

/// ncclUniqueId bytes for ncclCommInitRank (rank 0 creates, the caller broadcasts).
void dist_unique_id(char out[128]);

/// One rank's NCCL communicator.
struct DistComm {
    void* comm = nullptr; ///< ncclComm_t
    int nranks = 1, rank = 0;
    DistComm(int nranks, int rank, const char id[128]);
    ~DistComm();
    DistComm(const DistComm&) = delete;
    DistComm& operator=(const DistComm&) = delete;
    void allreduce_sum(double* buf, i64 count, cudaStream_t st) const;
};

/// Block-Jacobi ILU smoother of a row-block distributed matrix: the residual
/// is global (halo exchange + split-gather SpMV), the L/U sweeps use this
/// rank's diagonal-block factors only (sweeps are rank-local).
class DistSmoother {
public:
    void build(const HaloPlan& plan, const DistComm& comm, const SmootherConfig& cfg, cudaStream_t st);
    void smooth(const double* b, double* x, cudaStream_t st) const { s_.smooth(b, x, false, st); }
    void residual(const double* x, const double* b, double* r, cudaStream_t st) const { A_.residual(x, b, r, st); }
    const DeviceSmoother& smoother() const { return s_; }
    i64 nloc() const { return A_.n; }

private:
    HaloExchange hx_;
    DeviceMatrix A_;
    DeviceSmoother s_;
};

/// Row-block distributed GMRES+AMG: global Krylov iteration (halo-exchanged
/// SpMV, NCCL-summed CGS2 reductions) preconditioned by this rank's AMG
/// V-cycle on its diagonal block (block-Jacobi AMG; ILU smoothing inside).
class DistSolver {
public:
    void build(const HaloPlan& plan, const DistComm& comm, const AmgParams& ap, bool use_graph, cudaStream_t st);
    KrylovReport solve(const double* b, double* x, const KrylovParams& p, cudaStream_t st);
    i64 nloc() const { return A_.n; }
    int levels() const { return H_.num_levels(); }

private:
    const DistComm* comm_ = nullptr;
    HaloExchange hx_;
    DeviceMatrix A_;
    Csr A_diag_;
    HostHierarchy hh_;
    DeviceHierarchy H_;
};

} // namespace ilug
