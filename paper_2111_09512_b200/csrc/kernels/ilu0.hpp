// ILU(0) factorisation on the device (kernels/ilu0.cu).
#pragma once

#include "../host/ilu.hpp"
#include "ops.hpp"

namespace ilug {

/// ILU(0) of A on the device, bitwise equal to host ilu0 (and the reference):
/// same zero-pivot policy and error messages. Returns host factors (the device
/// object builders take their patterns from the host copies).
HostFactors ilu0_device(const Csr& A, PivotPatch patch, cudaStream_t st);

/// ILUG_ILU0_DEVICE=0 keeps ILU(0) on the host (A/B, tests).
bool ilu0_on_device();

/// ILUT(droptol, lfill) of A on the device (kernels/ilut.cu), bitwise equal to
/// host ilut (and the reference, src/ilu.cpp:120-265): warp per row, rows
/// scheduled by dependency flags. Same errors as the host path.
HostFactors ilut_device(const Csr& A, const IluParams& p, cudaStream_t st);

/// ILUG_ILUT_DEVICE=0 keeps ILUT on the host (A/B, tests).
bool ilut_on_device();

/// The factorisation the device objects use: ILU(0) and ILUT on the device
/// (host versions behind ILUG_ILU0_DEVICE=0 / ILUG_ILUT_DEVICE=0).
HostFactors factorize(const Csr& A, const IluParams& p, cudaStream_t st);

} // namespace ilug
