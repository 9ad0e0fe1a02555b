// Definitions of the opaque C-ABI handles (include/iluamg_b200.h, include/ilug.h).
// Every translation unit that touches a handle's fields includes THIS header,
// so each handle has exactly one definition (no per-TU copies that could drift).
#pragma once

#include "../../../include/ilug.h"
#include "../host/config.hpp"
#include "dist.hpp"
#include "driver.hpp"
#include "host_pipeline.hpp"

#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace ilug {
/// Calls on one handle from several host threads / streams share the handle's
/// device workspaces (level vectors, smoother scratch, level-set tickets). The
/// reference's contract is that concurrent V-cycles / smoothing on distinct
/// right-hand sides are safe and equal to serial calls bit for bit
/// (README.md:152-154, tests/test_amg.cpp:337-354), so each call's device work
/// is ordered after the previous call's (an event on that call's stream; the
/// host-side enqueue under a mutex). Same-stream callers pay one event record.
struct HandleSerial {
    std::mutex m;
    cudaEvent_t done = nullptr;
    bool armed = false;
    HandleSerial() = default;
    HandleSerial(const HandleSerial&) = delete;
    HandleSerial& operator=(const HandleSerial&) = delete;
    ~HandleSerial() {
        if (done) cudaEventDestroy(done);
    }
    /// f enqueues device work on st
    template <class F>
    void run(cudaStream_t st, F&& f) {
        std::lock_guard<std::mutex> g(m);
        if (!done) ILUG_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
        if (armed) ILUG_CUDA(cudaStreamWaitEvent(st, done, 0));
        f();
        ILUG_CUDA(cudaEventRecord(done, st));
        armed = true;
    }
    /// f is host-synchronous (its own streams, synchronised before it returns)
    template <class F>
    void run_sync(F&& f) {
        std::lock_guard<std::mutex> g(m);
        if (armed) ILUG_CUDA(cudaEventSynchronize(done));
        armed = false;
        f();
    }
};
} // namespace ilug

struct iluamg_matrix_s {
    ilug::Csr A;
    std::string label;
};
struct iluamg_config_s {
    ilug::Config cfg;
};
struct iluamg_report_s {
    ilug::Report rep;
    std::string json, text;
    std::vector<std::string> csv;
};
struct ilug_factors_s {
    ilug::DeviceIlu f;
    long long nnz_L = 0, nnz_U = 0;
    // ILU(0) handles: the factorised pattern (row starts + column hash) and the
    // device symbolic data, built on the first refactorisation
    bool ilu0 = false;
    ilug::PivotPatch patch = ilug::PivotPatch::error;
    ilug::RawVec<ilug::i64> a_rp;
    std::uint64_t a_hash = 0;
    std::unique_ptr<ilug::Ilu0Symbolic> sym;
    mutable ilug::HandleSerial ser; // direct solves share the level-set tickets
};
struct ilug_dmatrix_s {
    ilug::DeviceMatrix M;
};
struct ilug_smoother_s {
    ilug::Csr A;
    ilug::DeviceMatrix dA;
    ilug::DeviceSmoother s;
    ilug::DBuf<double> r, scratch;
    mutable ilug::DBuf<double> hb, hx; // staging for the host-buffer entry point
    mutable ilug::HostPipeline pipe;   // ilug_smooth_host_many
    mutable ilug::HandleSerial ser;
};
struct ilug_hierarchy_s {
    ilug::HostHierarchy h;
    ilug::DeviceHierarchy d;
    bool on_device = false;
    ilug::HandleSerial ser;
};
struct ilug_dist_plan_s {
    ilug::HaloPlan plan;
};
struct ilug_dist_comm_s {
    std::unique_ptr<ilug::DistComm> c;
};
struct ilug_dist_group_s {
    std::shared_ptr<ilug::LocalGroup> g;
};
struct ilug_dist_smoother_s {
    ilug::DistSmoother s;
    long long nnz_A = 0;
    mutable ilug::DBuf<double> hb, hx; // staging for ilug_dist_smooth_host
    mutable ilug::HostPipeline pipe;   // ilug_dist_smooth_host_many
};
struct ilug_dist_solver_s {
    ilug::DistSolver s;
};
struct ilug_dist_levels_s {
    std::vector<ilug::DistLevelPlan> levels;
};
