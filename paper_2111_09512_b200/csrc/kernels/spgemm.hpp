// Device sparse matrix product for the AMG Galerkin operator (kernels/spgemm.cu).
#pragma once

#include "dev.cuh"
#include "../host/csr.hpp"

namespace ilug {

/// CSR on the device: int64 row starts, int32 columns, fp64 values.
struct DevCsr {
    i64 nrows = 0, ncols = 0;
    DBuf<i64> rp;
    DBuf<i32> ci;
    DBuf<double> v;
    void upload(const Csr& h, cudaStream_t st);
    Csr download(cudaStream_t st) const;
};

/// C = A B on the device, bitwise equal to csr_matmul (src/sparse.cpp:176-231
/// accumulation order, exact zeros dropped). False if a row has more distinct
/// columns than the largest per-warp table holds (the caller falls back).
bool spgemm_device(i64 nrows, i64 ncols, const DevCsr& A, const DevCsr& B, DevCsr& C, cudaStream_t st);

/// Host in/out forms: A B, and the Galerkin product R (A P) with A P kept on
/// the device. Fall back to csr_matmul when spgemm_device declines.
Csr spgemm_device_host(const Csr& A, const Csr& B, cudaStream_t st);
Csr galerkin_device(const Csr& A, const Csr& P, const Csr& R, cudaStream_t st);

/// ILUG_GALERKIN_DEVICE=1 moves the Galerkin products of solve_with to the
/// device (off by default: transfer-bound next to the host AMG setup).
bool galerkin_on_device();

} // namespace ilug
