// Device AMG setup (kernels/amg_setup.cu): strength, PMIS, direct and MM-ext
// interpolation, transposes and the Galerkin product on the GPU, bitwise the
// host setup (host/amg.cpp) and the reference (src/amg.cpp:18-390).
#pragma once

#include "../host/amg.hpp"
#include "spgemm.hpp"

namespace ilug {

/// C/F split on the device: is_coarse (0/1), coarse_index (-1 for F points).
struct DevSplit {
    i64 n = 0, n_coarse = 0;
    DBuf<char> is_coarse;
    DBuf<i64> coarse_index;
};

/// Strength pattern of A (values not stored): S_ij iff j != i and
/// |a_ij| >= theta max_{k != i} |a_ik| (src/amg.cpp:18-50).
DevCsr strength_device(const DevCsr& A, double theta, cudaStream_t st);
/// Transpose with every row's columns ascending (values optional).
DevCsr transpose_device(const DevCsr& M, bool values, cudaStream_t st);
/// PMIS split with the reference's hash jitter and repair pass (src/amg.cpp:56-158).
DevSplit pmis_device(const DevCsr& S, const DevCsr& St, std::uint64_t seed, cudaStream_t st);
/// Direct interpolation (src/amg.cpp:162-232).
DevCsr interp_direct_device(const DevCsr& A, const DevCsr& S, const DevSplit& sp, cudaStream_t st);

/// MM-ext interpolation (src/amg.cpp:235-346); rows with no strong C-neighbour
/// sum take direct weights, counted in *fallback_rows.
DevCsr interp_mm_ext_device(const DevCsr& A, const DevCsr& S, const DevSplit& sp, i64* fallback_rows,
                            cudaStream_t st);

/// PMIS coarsening with direct or MM-ext interpolation (the device path's
/// scope; the order-dependent RS greedy coarsening stays on the host).
bool amg_device_supported(const AmgParams& p);
/// amg_setup on the device: the hierarchy is built level by level on the GPU
/// and every level's A/P/R/split is handed to the host structures (and to
/// on_level) as soon as it is final; the result equals amg_setup bit for bit.
/// Ad: A already on the device (read only; the caller keeps it alive until
/// on_level(0) has been called), else A is uploaded.
/// keep_device: each level handed to on_level keeps its device A (k >= 1), P, R
/// in HostLevel::dA/dP/dR for the consumer to build from and release; the host
/// P and R then carry only their dimensions (no download).
HostHierarchy amg_setup_device(const Csr& A, const AmgParams& prm, const LevelReady& on_level, cudaStream_t st,
                               const DevCsr* Ad = nullptr, bool keep_device = false);

} // namespace ilug
