// Row-block distribution of the solve phase over ranks (one process per GPU):
// the partition rule of the reference's Schur splitter (src/schur.cpp:28-33:
// base = n/p, the last rank takes the remainder), the halo plan for the
// global SpMV/residual, and the local diagonal block used for block-Jacobi
// ILU smoothing and the rank-local AMG hierarchy.
//
// Bitwise contract: the extended local matrix keeps every row's entries in the
// original GLOBAL column order (halo columns are renumbered, not re-sorted),
// so a distributed residual adds the same products in the same order as the
// single-process one and matches it bitwise.
#pragma once

#include "csr.hpp"

#include <string>

namespace ilug {

struct RowPartition {
    i64 n = 0, p = 1;
    std::vector<i64> starts; ///< p+1 entries
    i64 owner(i64 row) const;
};
RowPartition row_partition(i64 n, i64 p);

struct HaloPlan {
    i64 rank = 0, nranks = 1, row0 = 0, row1 = 0, nloc = 0, nhalo = 0;
    /// Local rows; columns < nloc are local (global - row0), columns >= nloc
    /// index the halo buffer (nloc + k). Entry order = global column order.
    Csr A_ext;
    /// Local diagonal block A[row0:row1, row0:row1] (sorted, local numbering).
    Csr A_diag;
    std::vector<i64> halo_global;              ///< ascending global ids of the halo entries
    std::vector<i64> recv_ranks, recv_offsets; ///< per source rank: halo segment [off_k, off_k+1)
    std::vector<i64> send_ranks, send_offsets; ///< per destination rank: segment of send_local
    std::vector<i32> send_local;               ///< local rows packed for each destination
};

/// Build the plan from this rank's rows (global column ids). Receives are
/// fully determined locally; sends need the other ranks' requests.
HaloPlan halo_plan(const Csr& rows, const RowPartition& part, i64 rank);

/// Global ids this rank needs from rank q (empty if none).
std::vector<i64> halo_requests(const HaloPlan& plan, i64 q);

/// Record rank q's request list (global ids owned by this rank).
void halo_set_sends(HaloPlan& plan, i64 q, const std::vector<i64>& global_ids);

/// Rows [row0, row1) of a 3D generator spec (poisson3d / stencil27 /
/// pressure27 / cutcell), identical to those rows of generate_problem(spec).
Csr generate_rows(const std::string& spec, i64 row0, i64 row1);

} // namespace ilug
