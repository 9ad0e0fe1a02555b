#include "schur.hpp"

namespace ilug {

SchurSetup schur_partition(const Csr& A, i64 p) {
    if (A.nrows != A.ncols) fail_invalid("partition: matrix must be square");
    if (p < 1 || p > A.nrows)
        fail_invalid("partition: block count " + std::to_string(p) + " out of range [1," +
                     std::to_string(A.nrows) + "]");
    const i64 n = A.nrows;
    SchurSetup s;
    s.p = p;
    const i64 base = n / p;
    std::vector<i32> owner(static_cast<size_t>(n));
    for (i64 b = 0; b < p; ++b) {
        const i64 lo = b * base, hi = b == p - 1 ? n : lo + base; // last block takes the remainder
        s.block_ranges.emplace_back(lo, hi);
        for (i64 i = lo; i < hi; ++i) owner[i] = static_cast<i32>(b);
    }
    // A row is interface iff it couples across a cut, by row or by column.
    std::vector<char> iface(static_cast<size_t>(n), 0);
    for (i64 i = 0; i < n; ++i)
        for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k)
            if (owner[i] != owner[A.ci[k]]) iface[i] = iface[A.ci[k]] = 1;
    s.perm.assign(static_cast<size_t>(n), -1);
    for (i64 i = 0; i < n; ++i) (iface[i] ? s.interface_idx : s.interior_idx).push_back(i);
    const i64 ni = static_cast<i64>(s.interior_idx.size()), nf = static_cast<i64>(s.interface_idx.size());
    for (i64 k = 0; k < ni; ++k) s.perm[s.interior_idx[k]] = k;
    for (i64 k = 0; k < nf; ++k) s.perm[s.interface_idx[k]] = ni + k;

    std::vector<Triplet> tb, te, tf, tc;
    for (i64 i = 0; i < n; ++i) {
        const i64 pi = s.perm[i];
        for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const i64 pj = s.perm[A.ci[k]];
            const double v = A.v[k];
            if (pi < ni)
                (pj < ni ? tb : te).push_back({pi, pj < ni ? pj : pj - ni, v});
            else
                (pj < ni ? tf : tc).push_back({pi - ni, pj < ni ? pj : pj - ni, v});
        }
    }
    s.B = csr_from_triplets(ni, ni, std::move(tb), true);
    s.E = csr_from_triplets(ni, nf, std::move(te), true);
    s.F = csr_from_triplets(nf, ni, std::move(tf), true);
    s.C = csr_from_triplets(nf, nf, std::move(tc), true);

    // Interior positions of one block form a contiguous run of the interior order.
    i64 cur = 0;
    for (i64 b = 0; b < p; ++b) {
        const i64 lo = cur;
        while (cur < ni && owner[s.interior_idx[cur]] == b) ++cur;
        s.blocks.emplace_back(lo, cur);
    }
    return s;
}

void schur_factorize(SchurSetup& s, const IluParams& ilu, ScalingKind scaling, const TriSolveConfig& ts) {
    if (ts.mode == TriSolveMode::richardson && scaling == ScalingKind::none)
        fail_invalid("factorize_blocks: Richardson block solves require row or row/col scaling");
    const i64 ni = s.B.nrows;
    HostFactors& f = s.factors;
    for (Csr* M : {&f.L, &f.U}) {
        M->nrows = M->ncols = ni;
        M->rp.assign(1, 0);
        M->ci.clear();
        M->v.clear();
    }
    for (const auto& [lo, hi] : s.blocks) {
        if (hi == lo) continue;
        // extract_block (src/schur.cpp:109-122): B is block diagonal, so the
        // block's rows hold exactly its in-block entries.
        Csr Bb;
        Bb.nrows = Bb.ncols = hi - lo;
        Bb.rp.assign(static_cast<size_t>(hi - lo) + 1, 0);
        for (i64 i = lo; i < hi; ++i) {
            for (i64 k = s.B.rp[i]; k < s.B.rp[i + 1]; ++k) {
                const i64 j = s.B.ci[k];
                if (j < lo || j >= hi) continue;
                Bb.ci.push_back(static_cast<i32>(j - lo));
                Bb.v.push_back(s.B.v[k]);
            }
            Bb.rp[i - lo + 1] = static_cast<i64>(Bb.ci.size());
        }
        const HostFactors fb = ilu_factorize(Bb, ilu);
        for (const auto& [dst, src] : {std::pair<Csr*, const Csr*>{&f.L, &fb.L}, {&f.U, &fb.U}}) {
            for (i64 i = 0; i < src->nrows; ++i) {
                for (i64 k = src->rp[i]; k < src->rp[i + 1]; ++k) {
                    dst->ci.push_back(static_cast<i32>(src->ci[k] + lo));
                    dst->v.push_back(src->v[k]);
                }
                dst->rp.push_back(static_cast<i64>(dst->ci.size()));
            }
        }
    }
    // rows of empty blocks: none (blocks tile [0, ni) exactly)
    if (static_cast<i64>(f.L.rp.size()) != ni + 1 || static_cast<i64>(f.U.rp.size()) != ni + 1)
        fail_invalid("schur: block ranges do not tile the interior");
}

} // namespace ilug
