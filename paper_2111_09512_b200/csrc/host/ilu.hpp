// Host incomplete factorisations (setup phase; the north star keeps them on
// the host). Scaling of the factors is a device kernel (K1, kernels/factor.cu);
// the host only produces the unscaled L (strict, unit diagonal implicit) and U
// (diagonal stored), the layout of the reference's IluFactors
// (include/iluamg/ilu.hpp:33-40).
#pragma once

#include "csr.hpp"

namespace ilug {

enum class IluVariant { ilu0, ilut };
enum class PivotPatch { error, replace };
enum class ScalingKind { none, row, row_col };

struct IluParams {
    IluVariant variant = IluVariant::ilu0;
    double droptol = 0.0;
    i64 lfill = 0;
    PivotPatch pivot_patch = PivotPatch::error;
};

struct HostFactors {
    Csr L; ///< strictly lower, unit diagonal implicit
    Csr U; ///< upper, diagonal stored
};

/// ILU(0) over A's pattern, IKJ order (reference algorithm: src/ilu.cpp:56-118).
/// Rows are processed level by level over the lower-pattern dependency DAG;
/// within a row the update sequence is the serial one, so the factors are
/// bitwise identical to a serial IKJ sweep for any thread count.
HostFactors ilu0(const Csr& A, PivotPatch patch);

/// Dual-threshold ILUT (reference algorithm: src/ilu.cpp:120-265): multipliers
/// dropped below droptol*|a_i|_2, pattern entries kept on the threshold alone,
/// fill capped at the lfill largest (ties to the lower column) per L and U part.
HostFactors ilut(const Csr& A, const IluParams& p);

HostFactors ilu_factorize(const Csr& A, const IluParams& p);

} // namespace ilug
