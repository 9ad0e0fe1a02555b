#include "dist.hpp"

#include <algorithm>

namespace ilug {

RowPartition row_partition(i64 n, i64 p, bool allow_empty) {
    if (p < 1 || (!allow_empty && p > std::max<i64>(n, 1))) fail_invalid("row_partition: rank count out of range");
    RowPartition part;
    part.n = n;
    part.p = p;
    const i64 base = n / p;
    for (i64 r = 0; r < p; ++r) part.starts.push_back(r * base);
    part.starts.push_back(n); // the last rank absorbs the remainder
    return part;
}

i64 RowPartition::owner(i64 row) const {
    const auto it = std::upper_bound(starts.begin(), starts.end() - 1, row);
    return static_cast<i64>(it - starts.begin()) - 1;
}

namespace {
HaloPlan make_plan(Csr&& rows_in, const RowPartition& part, i64 rank, bool square) {
    const Csr rows = [&] { // pattern view: row starts and columns stay, values move into A_ext
        Csr r;
        r.nrows = rows_in.nrows, r.ncols = rows_in.ncols;
        r.rp = rows_in.rp;
        r.ci = std::move(rows_in.ci);
        return r;
    }();
    if (rank < 0 || rank >= part.p) fail_invalid("halo_plan: rank out of range");
    HaloPlan h;
    h.rank = rank;
    h.nranks = part.p;
    h.row0 = part.starts[rank];
    h.row1 = part.starts[rank + 1];
    h.nloc = h.row1 - h.row0;
    if (square && rows.nrows != h.nloc) fail_invalid("halo_plan: local row count does not match the partition");
    const i64 nr = rows.nrows, r0 = h.row0, r1 = h.row1;
    auto local = [&](i64 j) { return j >= r0 && j < r1; };
    // halo = sorted unique off-range columns (contiguous ranges => grouped by owner);
    // per-row off-range counts give the split of every row for the two-pass fills
    std::vector<i64> off_cnt(static_cast<size_t>(nr) + 1, 0);
    const int T = host_threads();
    std::vector<std::vector<i64>> part_halo(static_cast<size_t>(T));
    parallel_ranges(nr, [&](i64 b, i64 e, int t) {
        auto& hv = part_halo[static_cast<size_t>(t)];
        for (i64 i = b; i < e; ++i) {
            i64 c = 0;
            for (i64 k = rows.rp[i]; k < rows.rp[i + 1]; ++k)
                if (!local(rows.ci[k])) ++c, hv.push_back(rows.ci[k]);
            off_cnt[i + 1] = c;
        }
    });
    for (auto& hv : part_halo) h.halo_global.insert(h.halo_global.end(), hv.begin(), hv.end());
    std::sort(h.halo_global.begin(), h.halo_global.end());
    h.halo_global.erase(std::unique(h.halo_global.begin(), h.halo_global.end()), h.halo_global.end());
    h.nhalo = static_cast<i64>(h.halo_global.size());
    for (i64 k = 0; k < h.nhalo; ++k) {
        const i64 q = part.owner(h.halo_global[k]);
        if (h.recv_ranks.empty() || h.recv_ranks.back() != q) {
            h.recv_ranks.push_back(q);
            h.recv_offsets.push_back(k);
        }
    }
    h.recv_offsets.push_back(h.nhalo);
    for (i64 i = 0; i < nr; ++i) off_cnt[i + 1] += off_cnt[i];

    // extended matrix: same entry order, renumbered columns
    h.A_ext.nrows = nr;
    h.A_ext.ncols = h.nloc + h.nhalo;
    h.A_ext.rp = std::move(rows_in.rp);
    h.A_ext.ci.resize(rows.ci.size());
    h.A_ext.v = std::move(rows_in.v);
    const RawVec<double>& vals = h.A_ext.v;
    const bool split = square && h.nhalo > 0; // without a halo the block is A_ext (diag())
    if (square) {
        h.A_off.nrows = nr;
        h.A_off.ncols = h.nloc + h.nhalo;
        h.A_off.rp.assign(static_cast<size_t>(nr) + 1, 0);
    }
    if (split) {
        h.A_diag.nrows = h.A_diag.ncols = h.nloc;
        h.A_diag.rp.resize(static_cast<size_t>(nr) + 1);
        for (i64 i = 0; i <= nr; ++i) {
            h.A_off.rp[i] = off_cnt[i];
            h.A_diag.rp[i] = rows.rp[i] - rows.rp[0] - off_cnt[i];
        }
        h.A_diag.ci.resize(static_cast<size_t>(h.A_diag.rp[nr]));
        h.A_diag.v.resize(static_cast<size_t>(h.A_diag.rp[nr]));
        h.A_off.ci.resize(static_cast<size_t>(off_cnt[nr]));
        h.A_off.v.resize(static_cast<size_t>(off_cnt[nr]));
    }
    parallel_ranges(nr, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            i64 dd = split ? h.A_diag.rp[i] : 0, oo = split ? h.A_off.rp[i] : 0;
            for (i64 k = rows.rp[i]; k < rows.rp[i + 1]; ++k) {
                const i64 j = rows.ci[k];
                if (local(j)) {
                    h.A_ext.ci[k] = static_cast<i32>(j - r0);
                    if (split) h.A_diag.ci[dd] = static_cast<i32>(j - r0), h.A_diag.v[dd++] = vals[k];
                } else {
                    const auto it = std::lower_bound(h.halo_global.begin(), h.halo_global.end(), j);
                    h.A_ext.ci[k] = static_cast<i32>(h.nloc + (it - h.halo_global.begin()));
                    if (split) h.A_off.ci[oo] = h.A_ext.ci[k], h.A_off.v[oo++] = vals[k];
                }
            }
        }
    });
    return h;
}
} // namespace

HaloPlan halo_plan(const Csr& rows, const RowPartition& part, i64 rank) { return make_plan(csr_copy(rows), part, rank, true); }
HaloPlan halo_plan(Csr&& rows, const RowPartition& part, i64 rank) { return make_plan(std::move(rows), part, rank, true); }

HaloPlan halo_plan_rect(Csr&& rows, const RowPartition& cols, i64 rank) {
    return make_plan(std::move(rows), cols, rank, false);
}

Csr csr_row_block(const Csr& M, i64 r0, i64 r1) {
    if (r0 < 0 || r1 < r0 || r1 > M.nrows) fail_invalid("csr_row_block: row range out of bounds");
    Csr B;
    B.nrows = r1 - r0;
    B.ncols = M.ncols;
    B.rp.resize(static_cast<size_t>(B.nrows) + 1);
    const i64 base = M.rp[r0];
    for (i64 i = 0; i <= B.nrows; ++i) B.rp[i] = M.rp[r0 + i] - base;
    const i64 nnz = M.rp[r1] - base;
    B.ci.resize(static_cast<size_t>(nnz));
    B.v.resize(static_cast<size_t>(nnz));
    parallel_ranges(nnz, [&](i64 b, i64 e, int) { // first touch spread over the pool
        std::copy(M.ci.begin() + base + b, M.ci.begin() + base + e, B.ci.begin() + b);
        std::copy(M.v.begin() + base + b, M.v.begin() + base + e, B.v.begin() + b);
    }, 1 << 16);
    return B;
}

std::vector<DistLevelPlan> dist_level_plans(const HostHierarchy& h, i64 nranks, i64 rank) {
    const i64 L = h.num_levels();
    std::vector<DistLevelPlan> out;
    if (L < 2) return out; // a single level is the replicated coarse solve
    out.resize(static_cast<size_t>(L - 1));
    std::vector<RowPartition> parts;
    for (i64 k = 0; k < L; ++k) parts.push_back(row_partition(h.levels[k].A.nrows, nranks, true));
    for (i64 k = 0; k + 1 < L; ++k) {
        const HostLevel& hl = h.levels[k];
        DistLevelPlan& d = out[k];
        d.n = hl.A.nrows;
        d.part = parts[k];
        if (d.n < nranks)
            fail_invalid("distributed AMG: level " + std::to_string(k) + " has " + std::to_string(d.n) +
                         " rows for " + std::to_string(nranks) + " ranks (raise amg.coarse_size)");
        const i64 f0 = d.part.starts[rank], f1 = d.part.starts[rank + 1];
        d.A = halo_plan(csr_row_block(hl.A, f0, f1), d.part, rank);
        d.last = k + 2 == L;
        if (d.last) {
            d.R_full = csr_copy(hl.R);
            d.P_rows = csr_row_block(hl.P, f0, f1);
        } else {
            const RowPartition& cp = parts[k + 1];
            d.R = halo_plan_rect(csr_row_block(hl.R, cp.starts[rank], cp.starts[rank + 1]), d.part, rank);
            d.P = halo_plan_rect(csr_row_block(hl.P, f0, f1), cp, rank);
        }
    }
    return out;
}

std::vector<i64> halo_requests(const HaloPlan& h, i64 q) {
    for (size_t s = 0; s < h.recv_ranks.size(); ++s)
        if (h.recv_ranks[s] == q)
            return {h.halo_global.begin() + h.recv_offsets[s], h.halo_global.begin() + h.recv_offsets[s + 1]};
    return {};
}

void halo_set_sends(HaloPlan& h, i64 q, const std::vector<i64>& ids) {
    if (ids.empty()) return;
    if (q == h.rank || q < 0 || q >= h.nranks) fail_invalid("halo_set_sends: bad destination rank");
    if (std::find(h.send_ranks.begin(), h.send_ranks.end(), q) != h.send_ranks.end())
        fail_invalid("halo_set_sends: destination already set");
    if (h.send_offsets.empty()) h.send_offsets.push_back(0);
    h.send_ranks.push_back(q);
    for (i64 g : ids) {
        if (g < h.row0 || g >= h.row1) fail_invalid("halo_set_sends: requested row not owned by this rank");
        h.send_local.push_back(static_cast<i32>(g - h.row0));
    }
    h.send_offsets.push_back(static_cast<i64>(h.send_local.size()));
}

} // namespace ilug
