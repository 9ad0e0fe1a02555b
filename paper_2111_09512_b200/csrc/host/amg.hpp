// Host AMG setup (the north star allows setup on the host): strength of
// connection, C/F splitting, interpolation, Galerkin products, the coarse
// dense LU. Algorithms follow the reference (src/amg.cpp:18-390,
// src/dense.cpp:8-38) with identical floating-point operation order, so the
// hierarchy is bitwise the reference's; the loops are row-parallel wherever a
// row's result does not depend on other rows of the same pass.
#pragma once

#include "csr.hpp"
#include "ilu.hpp"

#include <cstdint>
#include <memory>

namespace ilug {

enum class Coarsening { rs_greedy, pmis };
enum class Interpolation { direct, mm_ext };
enum class SmootherKind { jacobi, l1_jacobi, gauss_seidel, poly_gs, ilu, schur_ilut };
enum class TriSolveMode { direct, richardson };
/// How the U solve iterates in Richardson mode: on the row-scaled unit-diagonal
/// factor (the reference, src/trisolve.cpp:132-147) or as Jacobi on the unscaled
/// factor, x <- D^-1 (b - N x) (north-star deviation).
enum class UpperIteration { scaled, jacobi };

struct TriSolveConfig {
    TriSolveMode mode = TriSolveMode::richardson;
    i64 m_lower = 10;
    i64 m_upper = 10;
    UpperIteration upper = UpperIteration::scaled;
};

struct SmootherConfig {
    SmootherKind kind = SmootherKind::gauss_seidel;
    i64 sweeps = 2;
    i64 poly_degree = 2;
    IluParams ilu_params;
    TriSolveConfig trisolve;
    ScalingKind scaling = ScalingKind::row;
    i64 schur_blocks = 4;
};

struct SmootherPlan {
    SmootherConfig finest;
    i64 finest_levels = 1;
    SmootherConfig fallback;
    const SmootherConfig& for_level(i64 k) const { return k < finest_levels ? finest : fallback; }
};

struct AmgParams {
    double theta = 0.25;
    i64 max_levels = 25;
    i64 coarse_size = 16;
    Coarsening coarsening = Coarsening::rs_greedy;
    Interpolation interpolation = Interpolation::direct;
    i64 cycles_nu = 1;
    std::uint64_t pmis_seed = 1;
    SmootherPlan plan;
    /// Galerkin product R (A P) override (the device SpGEMM when the setup runs
    /// next to a GPU, kernels/spgemm.cu); empty: host csr_matmul. Same bits.
    std::function<Csr(const Csr& A, const Csr& P, const Csr& R)> galerkin;
    /// device.amg_setup: 0 host, 1 device when supported (auto), 2 device (required)
    int device_setup = 1;
};

struct CfSplit {
    std::vector<char> is_coarse;
    std::vector<i64> coarse_index;
    i64 n_coarse = 0;
};

struct DevCsr; // kernels/spgemm.hpp

struct HostLevel {
    Csr A, P, R;
    CfSplit split;
    i64 mm_ext_fallback_rows = 0;
    /// Device copies the device AMG setup leaves for the device-hierarchy
    /// builder when asked (solve_with): it builds its SELL copies from them
    /// instead of re-uploading A, P, R, then releases them.
    mutable std::shared_ptr<DevCsr> dA, dP, dR;
};

/// Dense LU with partial pivoting (first strict maximum wins), row-major.
struct DenseLu {
    i64 n = 0;
    std::vector<double> lu;
    std::vector<i64> piv;
};
DenseLu dense_lu_factor(const Csr& A);
Vec dense_lu_solve(const DenseLu& f, const Vec& b);

struct HostHierarchy {
    std::vector<HostLevel> levels;
    DenseLu coarse;
    AmgParams params;
    i64 num_levels() const { return static_cast<i64>(levels.size()); }
    double operator_complexity() const;
};

Csr strength(const Csr& A, double theta);
CfSplit coarsen_rs_greedy(const Csr& S);
CfSplit coarsen_pmis(const Csr& S, std::uint64_t seed);
Csr interp_direct(const Csr& A, const CfSplit& split, const Csr& S);
Csr interp_mm_ext(const Csr& A, const CfSplit& split, const Csr& S, i64* fallback_rows);

/// on_level(k, level, last) runs on the calling thread as soon as level k is
/// final (A, and P/R unless last): consumers (the device builder) may read the
/// level concurrently with the setup of the next ones. Level addresses are
/// stable (the level vector is reserved up front and moved, never reallocated).
using LevelReady = std::function<void(i64, const HostLevel&, bool)>;
HostHierarchy amg_setup(const Csr& A, const AmgParams& params, const LevelReady& on_level = {});

struct FlopsModel {
    std::int64_t smoothing = 0, coarse_solve = 0, krylov_spmv = 0;
};
/// Cost model of src/amg.cpp:420-440 (80 flops/nnz on ILU-smoothed levels, else 8).
FlopsModel flops_model(const HostHierarchy& h);

} // namespace ilug
