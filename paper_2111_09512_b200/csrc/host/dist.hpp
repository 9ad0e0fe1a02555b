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

#include "amg.hpp"
#include "csr.hpp"

#include <string>

namespace ilug {

struct RowPartition {
    i64 n = 0, p = 1;
    std::vector<i64> starts; ///< p+1 entries
    i64 owner(i64 row) const;
};
/// allow_empty: p > n is accepted (leading ranks own no rows) — coarse AMG levels.
RowPartition row_partition(i64 n, i64 p, bool allow_empty = false);

struct HaloPlan {
    /// [row0, row1) = the columns this rank owns (its rows of the vector the
    /// operator reads; for a square operator also its rows), nloc = row1 - row0.
    i64 rank = 0, nranks = 1, row0 = 0, row1 = 0, nloc = 0, nhalo = 0;
    /// Local rows; columns < nloc are local (global - row0), columns >= nloc
    /// index the halo buffer (nloc + k). Entry order = global column order.
    Csr A_ext;
    /// Square operators: local diagonal block A[row0:row1, row0:row1] (sorted,
    /// local numbering) and the off-block rest (halo columns only, ext numbering).
    /// Without a halo the block is A_ext itself (A_diag stays empty: use diag()).
    Csr A_diag, A_off;
    const Csr& diag() const { return nhalo == 0 ? A_ext : A_diag; }
    std::vector<i64> halo_global;              ///< ascending global ids of the halo entries
    std::vector<i64> recv_ranks, recv_offsets; ///< per source rank: halo segment [off_k, off_k+1)
    std::vector<i64> send_ranks, send_offsets; ///< per destination rank: segment of send_local
    std::vector<i32> send_local;               ///< local rows packed for each destination
};

/// Build the plan from this rank's rows (global column ids). Receives are
/// fully determined locally; sends need the other ranks' requests.
HaloPlan halo_plan(const Csr& rows, const RowPartition& part, i64 rank);
/// Same, consuming the rows (no copy of the values).
HaloPlan halo_plan(Csr&& rows, const RowPartition& part, i64 rank);
/// Same for an operator whose rows are partitioned differently from the vector
/// it reads (AMG restriction / prolongation): `cols` partitions the columns.
HaloPlan halo_plan_rect(Csr&& rows, const RowPartition& cols, i64 rank);

/// Rows [r0, r1) of M, global column ids.
Csr csr_row_block(const Csr& M, i64 r0, i64 r1);

/// One rank's share of an AMG level of a row-block distributed hierarchy
/// (SURVEY.md §8e): A_k and P_k rows by the level's partition, R_k rows by the
/// next level's. The last smoothed level keeps R whole (every rank forms the
/// full coarsest right-hand side from the all-gathered residual) and P with
/// global coarse columns (the coarsest solution is replicated).
struct DistLevelPlan {
    i64 n = 0;
    RowPartition part;
    HaloPlan A, R, P;
    bool last = false;
    Csr R_full, P_rows;
};
std::vector<DistLevelPlan> dist_level_plans(const HostHierarchy& h, i64 nranks, i64 rank);

/// Global ids this rank needs from rank q (empty if none).
std::vector<i64> halo_requests(const HaloPlan& plan, i64 q);

/// Record rank q's request list (global ids owned by this rank).
void halo_set_sends(HaloPlan& plan, i64 q, const std::vector<i64>& global_ids);

/// Rows [row0, row1) of a 3D generator spec (poisson3d / stencil27 /
/// pressure27 / cutcell), identical to those rows of generate_problem(spec).
Csr generate_rows(const std::string& spec, i64 row0, i64 row1);

} // namespace ilug
