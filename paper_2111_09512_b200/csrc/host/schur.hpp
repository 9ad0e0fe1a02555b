// Host setup of the ILUT Schur-complement smoother (reference:
// include/iluamg/schur.hpp:22-62, src/schur.cpp:19-135): contiguous row-block
// partition, interior/interface split, [[B,E],[F,C]] assembly under the
// interior-first permutation, per-block ILUT factors (built in parallel; the
// blocks are independent). The device applies it (device/solver.cu, K9).
#pragma once

#include "amg.hpp"

namespace ilug {

struct SchurSetup {
    i64 p = 1;
    std::vector<std::pair<i64, i64>> block_ranges; ///< [begin,end) global rows
    std::vector<i64> interior_idx, interface_idx;  ///< ascending global ids
    std::vector<i64> perm;                          ///< global id -> position (interior ++ interface)
    Csr B, E, F, C;
    std::vector<std::pair<i64, i64>> blocks;        ///< interior positions [begin,end) per block
    /// Block-diagonal factors over the interior unknowns: blockdiag(L_b) and
    /// blockdiag(U_b) (each block's ILUT, unscaled; scaling happens on the device).
    HostFactors factors;
};

/// partition (src/schur.cpp:19-105).
SchurSetup schur_partition(const Csr& A, i64 p);

/// factorize_blocks (src/schur.cpp:124-135) into one block-diagonal factor pair.
void schur_factorize(SchurSetup& s, const IluParams& ilu, ScalingKind scaling, const TriSolveConfig& ts);

} // namespace ilug
