#include "amg.hpp"
#include "problems.hpp"

#include <atomic>
#include <cmath>

namespace ilug {

double HostHierarchy::operator_complexity() const {
    if (levels.empty() || levels.front().A.nnz() == 0) return 0.0;
    double total = 0.0;
    for (const auto& l : levels) total += static_cast<double>(l.A.nnz());
    return total / static_cast<double>(levels.front().A.nnz());
}

namespace {

// Two-pass row-parallel CSR assembly: count(i) then fill(i, cols, vals).
template <typename Count, typename Fill>
Csr assemble(i64 nrows, i64 ncols, Count count, Fill fill) {
    Csr C;
    C.nrows = nrows;
    C.ncols = ncols;
    C.rp.assign(static_cast<size_t>(nrows) + 1, 0);
    parallel_ranges(nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) C.rp[i + 1] = count(i);
    });
    for (i64 i = 0; i < nrows; ++i) C.rp[i + 1] += C.rp[i];
    C.ci.resize(static_cast<size_t>(C.rp[nrows]));
    C.v.resize(static_cast<size_t>(C.rp[nrows]));
    parallel_ranges(nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) fill(i, C.ci.data() + C.rp[i], C.v.data() + C.rp[i]);
    });
    return C;
}

enum : char { kFree = 0, kC = 1, kF = 2 };

// Promote F-points without a strong C-neighbour, in index order (the pass is
// order dependent, src/amg.cpp:56-84), then number the C-points.
CfSplit finish_split(const Csr& S, std::vector<char>& st) {
    const i64 n = S.nrows;
    // Promotions only ever add C-points, so an F-point that already has a
    // strong C-neighbour keeps it: find the candidates in parallel, then run
    // the order-dependent pass over the candidates only (same result).
    auto lacks_c = [&](i64 i) {
        for (i64 k = S.rp[i]; k < S.rp[i + 1]; ++k)
            if (st[S.ci[k]] == kC) return false;
        return true;
    };
    std::vector<std::vector<i64>> cand(static_cast<size_t>(host_threads()));
    parallel_ranges(n, [&](i64 b, i64 e, int t) {
        for (i64 i = b; i < e; ++i)
            if (st[i] == kF && lacks_c(i)) cand[static_cast<size_t>(t)].push_back(i);
    });
    for (const auto& list : cand) // chunks hold ascending index ranges, in chunk order
        for (const i64 i : list)
            if (lacks_c(i)) st[i] = kC;
    CfSplit sp;
    sp.is_coarse.resize(static_cast<size_t>(n));
    sp.coarse_index.assign(static_cast<size_t>(n), -1);
    for (i64 i = 0; i < n; ++i) {
        sp.is_coarse[i] = st[i] == kC;
        if (sp.is_coarse[i]) sp.coarse_index[i] = sp.n_coarse++;
    }
    return sp;
}

// Row classification shared by both interpolations (src/amg.cpp:162-205):
// strong C-neighbours, beta (strong F + weak C), weak sum (all weak), a_ii.
struct RowClass {
    double aii = 0.0, beta = 0.0, weak = 0.0;
    std::vector<std::pair<i64, double>> strong_c;
};

void classify(const Csr& A, const Csr& S, const CfSplit& sp, i64 i, RowClass& rc) {
    rc.aii = rc.beta = rc.weak = 0.0;
    rc.strong_c.clear();
    i64 s = S.rp[i];
    const i64 se = S.rp[i + 1];
    for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
        const i64 j = A.ci[k];
        const double v = A.v[k];
        while (s < se && S.ci[s] < j) ++s;
        const bool strong = s < se && S.ci[s] == j;
        if (j == i) {
            rc.aii = v;
        } else if (strong) {
            if (sp.is_coarse[j])
                rc.strong_c.emplace_back(j, v);
            else
                rc.beta += v;
        } else {
            rc.weak += v;
            if (sp.is_coarse[j]) rc.beta += v;
        }
    }
}

// 0 ok, 1 no strong C neighbour (invalid), 2 zero denominator (numeric)
int direct_weights(const RowClass& rc, std::vector<std::pair<i64, double>>& w) {
    w.clear();
    if (rc.strong_c.empty()) return 1;
    const double denom = rc.aii + rc.weak;
    if (denom == 0.0) return 2;
    const double shift = rc.beta / static_cast<double>(rc.strong_c.size());
    for (auto [j, a] : rc.strong_c) w.emplace_back(j, -(a + shift) / denom);
    return 0;
}

[[noreturn]] void direct_fail(int code, i64 i) {
    if (code == 1)
        fail_invalid("interp_direct: F-point " + std::to_string(i) +
                     " has no strong C-neighbor (coarsening repair failed)");
    fail_numeric("interp_direct: zero denominator at row " + std::to_string(i));
}

} // namespace

Csr strength(const Csr& A, double theta) {
    if (A.nrows != A.ncols) fail_invalid("strength: matrix must be square");
    if (!(theta > 0.0 && theta <= 1.0)) fail_invalid("strength: theta must lie in (0, 1]");
    std::vector<double> cut(static_cast<size_t>(A.nrows));
    auto row_cut = [&](i64 i) {
        double m = 0.0;
        for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k)
            if (A.ci[k] != i) m = std::max(m, std::abs(A.v[k]));
        return m == 0.0 ? -1.0 : theta * m; // -1: empty strength row
    };
    return assemble(
        A.nrows, A.ncols,
        [&](i64 i) {
            const double c = cut[i] = row_cut(i);
            if (c < 0.0) return i64{0};
            i64 cnt = 0;
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k)
                cnt += A.ci[k] != i && std::abs(A.v[k]) >= c;
            return cnt;
        },
        [&](i64 i, i32* c, double* v) {
            if (cut[i] < 0.0) return;
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k)
                if (A.ci[k] != i && std::abs(A.v[k]) >= cut[i]) *c++ = A.ci[k], *v++ = 1.0;
        });
}

CfSplit coarsen_rs_greedy(const Csr& S) {
    const Csr St = csr_transpose(S);
    std::vector<char> st(static_cast<size_t>(S.nrows), kFree);
    for (i64 i = 0; i < S.nrows; ++i) {
        if (st[i] != kFree) continue;
        st[i] = kC;
        for (i64 k = St.rp[i]; k < St.rp[i + 1]; ++k)
            if (st[St.ci[k]] == kFree) st[St.ci[k]] = kF;
    }
    return finish_split(S, st);
}

CfSplit coarsen_pmis(const Csr& S, std::uint64_t seed) {
    const i64 n = S.nrows;
    SetupTimer tm("pmis");
    const Csr St = csr_transpose(S);
    tm.mark("transpose S");
    std::vector<double> wt(static_cast<size_t>(n));
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i)
            wt[i] = static_cast<double>(St.rp[i + 1] - St.rp[i]) +
                    hash_unit(seed, static_cast<std::uint64_t>(i));
    });
    std::vector<char> st(static_cast<size_t>(n), kFree), fresh(static_cast<size_t>(n), 0);
    // Rounds are synchronous (every decision reads the state at the round's
    // start), so working on the compacted list of still-free points gives the
    // same split as sweeping all n points every round.
    std::vector<i64> live(static_cast<size_t>(n));
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) live[i] = i;
    });
    const int T = host_threads();
    std::vector<std::vector<i64>> keep(static_cast<size_t>(T)), picked(static_cast<size_t>(T));
    tm.mark("weights");
    i64 rounds = 0;
    while (!live.empty()) {
        ++rounds;
        const i64 m = static_cast<i64>(live.size());
        // Local maxima among still-free strong neighbours (both directions).
        for (auto& v : picked) v.clear();
        parallel_ranges(m, [&](i64 b, i64 e, int t) {
            for (i64 q = b; q < e; ++q) {
                const i64 i = live[q];
                bool top = true;
                for (const Csr* G : {&S, &St})
                    for (i64 k = G->rp[i]; top && k < G->rp[i + 1]; ++k) {
                        const i64 j = G->ci[k];
                        if (j != i && st[j] == kFree && wt[j] >= wt[i]) top = false;
                    }
                if (top) picked[static_cast<size_t>(t)].push_back(i);
            }
        });
        i64 found = 0;
        for (const auto& v : picked) found += static_cast<i64>(v.size());
        if (found == 0) picked[0].push_back(live[0]); // smallest free index (live stays ascending)
        for (const auto& v : picked)
            for (const i64 i : v) fresh[i] = 1, st[i] = kC;
        // A free point becomes F iff a fresh C-point strongly depends on it,
        // i.e. some i in S-row(j) is fresh (equivalent to the St scatter).
        for (auto& v : keep) v.clear();
        parallel_ranges(m, [&](i64 b, i64 e, int t) {
            for (i64 q = b; q < e; ++q) {
                const i64 j = live[q];
                if (st[j] != kFree) continue;
                bool hit = false;
                for (i64 k = S.rp[j]; k < S.rp[j + 1] && !hit; ++k) hit = fresh[S.ci[k]] != 0;
                if (hit)
                    st[j] = kF;
                else
                    keep[static_cast<size_t>(t)].push_back(j);
            }
        });
        for (const auto& v : picked)
            for (const i64 i : v) fresh[i] = 0;
        std::vector<i64> next;
        next.reserve(static_cast<size_t>(m));
        for (const auto& v : keep) next.insert(next.end(), v.begin(), v.end()); // chunks in ascending order
        live.swap(next);
    }
    tm.mark("rounds", rounds);
    CfSplit sp = finish_split(S, st);
    tm.mark("finish split");
    return sp;
}

Csr interp_direct(const Csr& A, const CfSplit& sp, const Csr& S) {
    const i64 n = A.nrows;
    // The weights are recomputed per pass (classification is one pass over the
    // row) instead of being stored per row: no per-row heap allocation.
    auto weights = [&](i64 i) -> const std::vector<std::pair<i64, double>>& {
        thread_local RowClass rc;
        thread_local std::vector<std::pair<i64, double>> w;
        classify(A, S, sp, i, rc);
        direct_weights(rc, w);
        return w;
    };
    std::vector<int> status(static_cast<size_t>(n), 0);
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        RowClass rc;
        std::vector<std::pair<i64, double>> w;
        for (i64 i = b; i < e; ++i) {
            if (sp.is_coarse[i]) continue;
            classify(A, S, sp, i, rc);
            status[i] = direct_weights(rc, w);
        }
    });
    for (i64 i = 0; i < n; ++i)
        if (status[i]) direct_fail(status[i], i);
    return assemble(
        n, sp.n_coarse,
        [&](i64 i) {
            if (sp.is_coarse[i]) return i64{1};
            i64 c = 0;
            for (auto& [j, w] : weights(i)) c += w != 0.0; // from_triplets drops exact zeros
            return c;
        },
        [&](i64 i, i32* c, double* v) {
            if (sp.is_coarse[i]) {
                *c = static_cast<i32>(sp.coarse_index[i]), *v = 1.0;
                return;
            }
            for (auto& [j, w] : weights(i))
                if (w != 0.0) *c++ = static_cast<i32>(sp.coarse_index[j]), *v++ = w;
        });
}

Csr interp_mm_ext(const Csr& A, const CfSplit& sp, const Csr& S, i64* fallback_rows) {
    // W = -[(D_FF + D_g)^-1 (A^s_FF + D_b)] [D_b^-1 A^s_FC]  (src/amg.cpp:235-346)
    const i64 n = A.nrows, nc = sp.n_coarse;
    std::vector<i64> floc(static_cast<size_t>(n), -1), fglob;
    for (i64 i = 0; i < n; ++i)
        if (!sp.is_coarse[i]) floc[i] = static_cast<i64>(fglob.size()), fglob.push_back(i);
    const i64 nf = static_cast<i64>(fglob.size());

    Vec dbeta(static_cast<size_t>(nf), 0.0), dgamma(static_cast<size_t>(nf), 0.0),
        dff(static_cast<size_t>(nf), 0.0);
    std::vector<Triplet> tff, tfc;
    for (i64 fi = 0; fi < nf; ++fi) {
        const i64 i = fglob[fi];
        i64 s = S.rp[i];
        for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const i64 j = A.ci[k];
            const double v = A.v[k];
            while (s < S.rp[i + 1] && S.ci[s] < j) ++s;
            const bool strong = s < S.rp[i + 1] && S.ci[s] == j;
            if (j == i) {
                dff[fi] = v;
            } else if (strong) {
                if (sp.is_coarse[j]) {
                    tfc.push_back({fi, sp.coarse_index[j], v});
                    dbeta[fi] += v;
                } else {
                    tff.push_back({fi, floc[j], v});
                }
            } else {
                dgamma[fi] += v;
            }
        }
    }
    const Csr Asff = csr_from_triplets(nf, nf, std::move(tff));
    const Csr Asfc = csr_from_triplets(nf, nc, std::move(tfc));

    i64 fallbacks = 0;
    std::vector<char> fb(static_cast<size_t>(nf), 0);
    for (i64 fi = 0; fi < nf; ++fi)
        if (dbeta[fi] == 0.0) fb[fi] = 1, ++fallbacks;

    std::vector<Triplet> tm1;
    for (i64 fi = 0; fi < nf; ++fi) {
        const double den = dff[fi] + dgamma[fi];
        if (den == 0.0)
            fail_numeric("interp_mm_ext: singular D_FF + D_gamma at F-row " + std::to_string(fglob[fi]));
        const double inv = 1.0 / den;
        tm1.push_back({fi, fi, dbeta[fi] * inv});
        for (i64 k = Asff.rp[fi]; k < Asff.rp[fi + 1]; ++k) tm1.push_back({fi, Asff.ci[k], Asff.v[k] * inv});
    }
    const Csr M1 = csr_from_triplets(nf, nf, std::move(tm1));
    Csr M2 = Asfc;
    for (i64 fi = 0; fi < nf; ++fi) {
        const double inv = fb[fi] ? 0.0 : 1.0 / dbeta[fi];
        for (i64 k = M2.rp[fi]; k < M2.rp[fi + 1]; ++k) M2.v[k] *= inv;
    }
    Csr W = csr_matmul(M1, M2);
    for (double& x : W.v) x = -x;

    std::vector<Triplet> t;
    RowClass rc;
    std::vector<std::pair<i64, double>> dw;
    for (i64 i = 0; i < n; ++i) {
        if (sp.is_coarse[i]) {
            t.push_back({i, sp.coarse_index[i], 1.0});
            continue;
        }
        const i64 fi = floc[i];
        if (fb[fi]) {
            classify(A, S, sp, i, rc);
            if (const int code = direct_weights(rc, dw)) direct_fail(code, i);
            for (auto [j, w] : dw) t.push_back({i, sp.coarse_index[j], w});
            continue;
        }
        for (i64 k = W.rp[fi]; k < W.rp[fi + 1]; ++k) t.push_back({i, W.ci[k], W.v[k]});
    }
    if (fallback_rows) *fallback_rows = fallbacks;
    return csr_from_triplets(n, nc, std::move(t));
}

DenseLu dense_lu_factor(const Csr& A) {
    if (A.nrows != A.ncols) fail_invalid("DenseLu: matrix must be square");
    DenseLu f;
    const i64 n = f.n = A.nrows;
    f.lu.assign(static_cast<size_t>(n * n), 0.0);
    f.piv.resize(static_cast<size_t>(n));
    for (i64 i = 0; i < n; ++i)
        for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) f.lu[i * n + A.ci[k]] = A.v[k];
    double* a = f.lu.data();
    for (i64 k = 0; k < n; ++k) {
        i64 p = k;
        for (i64 i = k + 1; i < n; ++i)
            if (std::abs(a[i * n + k]) > std::abs(a[p * n + k])) p = i;
        if (a[p * n + k] == 0.0)
            fail_numeric("DenseLu: singular coarse matrix at column " + std::to_string(k));
        f.piv[k] = p;
        if (p != k)
            for (i64 j = 0; j < n; ++j) std::swap(a[p * n + j], a[k * n + j]);
        const double pivot = a[k * n + k];
        for (i64 i = k + 1; i < n; ++i) {
            const double m = a[i * n + k] / pivot;
            a[i * n + k] = m;
            for (i64 j = k + 1; j < n; ++j) a[i * n + j] -= m * a[k * n + j];
        }
    }
    return f;
}

Vec dense_lu_solve(const DenseLu& f, const Vec& b) {
    const i64 n = f.n;
    Vec x = b;
    for (i64 k = 0; k < n; ++k) {
        if (f.piv[k] != k) std::swap(x[f.piv[k]], x[k]);
        for (i64 i = k + 1; i < n; ++i) x[i] -= f.lu[i * n + k] * x[k];
    }
    for (i64 i = n; i-- > 0;) {
        double s = x[i];
        for (i64 j = i + 1; j < n; ++j) s -= f.lu[i * n + j] * x[j];
        x[i] = s / f.lu[i * n + i];
    }
    return x;
}

HostHierarchy amg_setup(const Csr& A, const AmgParams& prm, const LevelReady& on_level) {
    if (A.nrows != A.ncols) fail_invalid("setup: matrix must be square");
    if (!(prm.theta > 0.0 && prm.theta <= 1.0)) fail_invalid("setup: theta must lie in (0, 1]");
    if (prm.coarse_size < 1) fail_invalid("setup: coarse_size must be >= 1");
    if (prm.max_levels < 1) fail_invalid("setup: max_levels must be >= 1");
    if (prm.cycles_nu < 1) fail_invalid("setup: cycles_nu must be >= 1");
    HostHierarchy h;
    h.params = prm;
    h.levels.reserve(static_cast<size_t>(prm.max_levels)); // stable level addresses for on_level
    SetupTimer tm("amg");
    Csr cur = csr_copy(A);
    tm.mark("copy A");
    for (;;) {
        h.levels.emplace_back();
        HostLevel& lev = h.levels.back();
        lev.A = std::move(cur);
        const i64 k = h.num_levels() - 1;
        if (lev.A.nrows <= prm.coarse_size || k + 1 >= prm.max_levels) break;
        const Csr S = strength(lev.A, prm.theta);
        tm.mark("strength", k);
        CfSplit sp = prm.coarsening == Coarsening::rs_greedy ? coarsen_rs_greedy(S)
                                                             : coarsen_pmis(S, prm.pmis_seed);
        tm.mark("coarsen", k);
        if (static_cast<double>(sp.n_coarse) > 0.95 * static_cast<double>(lev.A.nrows)) break;
        Csr P = prm.interpolation == Interpolation::direct
                    ? interp_direct(lev.A, sp, S)
                    : interp_mm_ext(lev.A, sp, S, &lev.mm_ext_fallback_rows);
        tm.mark("interp", k);
        Csr R = csr_transpose(P);
        tm.mark("transpose", k);
        if (prm.galerkin) {
            cur = prm.galerkin(lev.A, P, R);
            tm.mark("R*(A*P) device", k);
        } else {
            Csr AP = csr_matmul(lev.A, P);
            tm.mark("A*P", k);
            cur = csr_matmul(R, AP);
            tm.mark("R*(AP)", k);
        }
        lev.P = std::move(P);
        lev.R = std::move(R);
        lev.split = std::move(sp);
        if (on_level) on_level(k, lev, false);
    }
    if (on_level) on_level(h.num_levels() - 1, h.levels.back(), true);
    h.coarse = dense_lu_factor(h.levels.back().A);
    return h;
}

FlopsModel flops_model(const HostHierarchy& h) {
    FlopsModel fm;
    for (i64 k = 0; k + 1 < h.num_levels(); ++k) {
        const SmootherKind kind = h.params.plan.for_level(k).kind;
        const bool ilu = kind == SmootherKind::ilu || kind == SmootherKind::schur_ilut;
        fm.smoothing += static_cast<std::int64_t>(h.levels[k].A.nnz()) * (ilu ? 80 : 8);
    }
    const std::int64_t mc = h.levels.back().A.nrows;
    fm.coarse_solve = mc * mc * mc;
    fm.krylov_spmv = 2 * static_cast<std::int64_t>(h.levels.front().A.nnz());
    return fm;
}

} // namespace ilug
