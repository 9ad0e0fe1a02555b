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
#include <string>
#include <vector>

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
};
struct ilug_hierarchy_s {
    ilug::HostHierarchy h;
    ilug::DeviceHierarchy d;
    bool on_device = false;
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
