#include "ilu.hpp"

#include <atomic>
#include <cmath>
#include <memory>
#include <thread>
#include <limits>
#include <queue>

namespace ilug {

namespace {

double row_norm2(const Csr& A, i64 i) {
    double s = 0.0;
    for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) s += A.v[k] * A.v[k];
    return std::sqrt(s);
}

// Zero-pivot policy (src/ilu.cpp:23-31): `error` aborts, `replace` substitutes
// sign(estimate) * max(droptol*|a_i|_2, 1e-16*|A|_F) (DBL_MIN if that is 0).
double patch_pivot(double droptol, double rownorm, double anorm_f, PivotPatch policy, i64 step) {
    if (policy == PivotPatch::error)
        fail_numeric("zero pivot at step " + std::to_string(step) +
                     " (no pivoting; rerun with pivot_patch=replace to substitute)");
    double mag = std::max(droptol * rownorm, 1e-16 * anorm_f);
    if (mag == 0.0) mag = std::numeric_limits<double>::min();
    return mag; // the estimate is always 0.0 here, so the sign is +
}

} // namespace

HostFactors ilu0(const Csr& A, PivotPatch patch) {
    if (A.nrows != A.ncols) fail_invalid("ilu0: matrix must be square");
    const i64 n = A.nrows;
    std::vector<i64> dpos(static_cast<size_t>(n), -1);
    for (i64 i = 0; i < n; ++i) {
        for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k)
            if (A.ci[k] == i) dpos[i] = k;
        if (dpos[i] < 0)
            fail_invalid("ilu0: diagonal entry (" + std::to_string(i) + "," + std::to_string(i) +
                         ") is structurally absent");
    }
    const double anorm_f = frobenius_norm(A);

    // Wavefront levels of the lower-pattern DAG.
    std::vector<i32> level(static_cast<size_t>(n), 0);
    i32 nlev = 0;
    for (i64 i = 0; i < n; ++i) {
        i32 l = 0;
        for (i64 k = A.rp[i]; k < dpos[i]; ++k) l = std::max(l, level[A.ci[k]] + 1);
        level[i] = l;
        nlev = std::max(nlev, l + 1);
    }
    std::vector<i64> lstart(static_cast<size_t>(nlev) + 1, 0), order(static_cast<size_t>(n));
    for (i64 i = 0; i < n; ++i) ++lstart[level[i] + 1];
    for (i32 l = 0; l < nlev; ++l) lstart[l + 1] += lstart[l];
    {
        std::vector<i64> cur(lstart.begin(), lstart.end() - 1);
        for (i64 i = 0; i < n; ++i) order[cur[level[i]]++] = i;
    }

    std::vector<double> w(A.v.begin(), A.v.end());
    std::atomic<i64> first_zero{n};
    // per-worker column -> position-in-row markers (-1 = not in row i's pattern)
    std::vector<std::vector<i32>> marks(static_cast<size_t>(host_threads()));
    for (i32 l = 0; l < nlev; ++l) {
        parallel_ranges(lstart[l + 1] - lstart[l], [&](i64 b, i64 e, int tid) {
            std::vector<i32>& pos = marks[static_cast<size_t>(tid)];
            if (pos.empty()) pos.assign(static_cast<size_t>(n), -1);
            for (i64 t = lstart[l] + b; t < lstart[l] + e; ++t) {
                const i64 i = order[t];
                const i64 beg = A.rp[i], end = A.rp[i + 1];
                for (i64 p = beg; p < end; ++p) pos[A.ci[p]] = static_cast<i32>(p - beg);
                for (i64 k = beg; k < dpos[i]; ++k) {
                    const i64 c = A.ci[k];
                    const double m = w[k] / w[dpos[c]];
                    w[k] = m;
                    // row c's strict upper part against row i's pattern; every
                    // match lies after k (its column exceeds c), and each w[p]
                    // receives its updates in ascending k, then ascending column:
                    // the order of the reference's merge (src/ilu.cpp)
                    for (i64 kk = dpos[c] + 1; kk < A.rp[c + 1]; ++kk) {
                        const i32 q = pos[A.ci[kk]];
                        if (q >= 0) w[beg + q] -= m * w[kk];
                    }
                }
                for (i64 p = beg; p < end; ++p) pos[A.ci[p]] = -1;
                if (w[dpos[i]] == 0.0) {
                    if (patch == PivotPatch::error) {
                        i64 cur = first_zero.load();
                        while (i < cur && !first_zero.compare_exchange_weak(cur, i)) {
                        }
                        w[dpos[i]] = 1.0; // placeholder; the factorisation is abandoned
                    } else {
                        w[dpos[i]] = patch_pivot(0.0, row_norm2(A, i), anorm_f, patch, i);
                    }
                }
            }
        }, 256);
    }
    if (first_zero.load() < n) patch_pivot(0.0, 0.0, 0.0, PivotPatch::error, first_zero.load());

    // Split into strict L and U (with diagonal), row-parallel.
    HostFactors f;
    for (Csr* M : {&f.L, &f.U}) {
        M->nrows = M->ncols = n;
        M->rp.assign(static_cast<size_t>(n) + 1, 0);
    }
    for (i64 i = 0; i < n; ++i) {
        f.L.rp[i + 1] = f.L.rp[i] + (dpos[i] - A.rp[i]);
        f.U.rp[i + 1] = f.U.rp[i] + (A.rp[i + 1] - dpos[i]);
    }
    f.L.ci.resize(static_cast<size_t>(f.L.rp[n]));
    f.L.v.resize(static_cast<size_t>(f.L.rp[n]));
    f.U.ci.resize(static_cast<size_t>(f.U.rp[n]));
    f.U.v.resize(static_cast<size_t>(f.U.rp[n]));
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            i64 pl = f.L.rp[i], pu = f.U.rp[i];
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                if (k < dpos[i])
                    f.L.ci[pl] = A.ci[k], f.L.v[pl++] = w[k];
                else
                    f.U.ci[pu] = A.ci[k], f.U.v[pu++] = w[k];
            }
        }
    });
    return f;
}

HostFactors ilut(const Csr& A, const IluParams& p) {
    if (A.nrows != A.ncols) fail_invalid("ilut: matrix must be square");
    if (!(p.droptol >= 0.0) || !std::isfinite(p.droptol))
        fail_invalid("ilut: droptol must be finite and >= 0");
    if (p.lfill < 0) fail_invalid("ilut: lfill must be >= 0");
    const i64 n = A.nrows;
    const double anorm_f = frobenius_norm(A);

    // Pipelined row-parallel ILUT. Row i's factor size is bounded a priori
    // (pattern part of A's row + lfill per triangle), so every row owns a fixed
    // slot and rows can be produced out of order by a pool of workers taking row
    // indices in ascending order. Row i reads U rows k only after they are
    // published (done[k], release/acquire) and eliminates in the serial heap
    // order, so each row's arithmetic is exactly the serial algorithm's: the
    // factors are bitwise independent of the worker count. The chain row i-1 ->
    // row i (last multiplier popped) bounds the speed-up, not correctness.
    std::vector<i64> loff(static_cast<size_t>(n) + 1, 0), uoff(static_cast<size_t>(n) + 1, 0);
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            i64 lo = 0, up = 0;
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) lo += A.ci[k] < i, up += A.ci[k] > i;
            loff[i + 1] = lo + p.lfill;
            uoff[i + 1] = 1 + up + p.lfill;
        }
    });
    for (i64 i = 0; i < n; ++i) loff[i + 1] += loff[i], uoff[i + 1] += uoff[i];
    // slot arrays: no zero fill (multi-GB at C2); each row writes its own slots
    RawVec<i32> lci(static_cast<size_t>(loff[n])), uci(static_cast<size_t>(uoff[n]));
    RawVec<double> lv(static_cast<size_t>(loff[n])), uv(static_cast<size_t>(uoff[n]));
    std::vector<i64> llen(static_cast<size_t>(n), 0), ulen(static_cast<size_t>(n), 0);
    std::unique_ptr<std::atomic<int>[]> done(new std::atomic<int>[static_cast<size_t>(n)]);
    for (i64 i = 0; i < n; ++i) done[i].store(0, std::memory_order_relaxed);
    std::atomic<i64> next{0}, first_zero{n};

    auto worker = [&]() {
        std::vector<double> w(static_cast<size_t>(n), 0.0);
        std::vector<char> live(static_cast<size_t>(n), 0), orig(static_cast<size_t>(n), 0);
        std::vector<i64> upper, kept, pat_part, fill_part;
        std::priority_queue<i64, std::vector<i64>, std::greater<i64>> pending;
        // Survivor selection (src/ilu.cpp:204-232): pattern entries pass on the
        // threshold (applied to the U part only), fill competes for lfill slots.
        auto select = [&](const std::vector<i64>& cols, bool lower, double tau) {
            pat_part.clear();
            fill_part.clear();
            for (i64 j : cols) {
                if (!live[j]) continue;
                if (!lower && std::abs(w[j]) < tau) continue;
                (orig[j] ? pat_part : fill_part).push_back(j);
            }
            const auto cap = static_cast<size_t>(p.lfill);
            if (fill_part.size() > cap) {
                std::nth_element(fill_part.begin(), fill_part.begin() + static_cast<std::ptrdiff_t>(cap),
                                 fill_part.end(), [&](i64 a, i64 b) {
                                     const double va = std::abs(w[a]), vb = std::abs(w[b]);
                                     return va != vb ? va > vb : a < b;
                                 });
                fill_part.resize(cap);
            }
            pat_part.insert(pat_part.end(), fill_part.begin(), fill_part.end());
            std::sort(pat_part.begin(), pat_part.end());
        };
        for (;;) {
            const i64 i = next.fetch_add(1, std::memory_order_relaxed);
            if (i >= n) return;
            const double tau = p.droptol * row_norm2(A, i);
            upper.clear();
            kept.clear();
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                const i64 j = A.ci[k];
                w[j] = A.v[k];
                live[j] = 1;
                orig[j] = 1;
                if (j < i)
                    pending.push(j);
                else if (j > i)
                    upper.push_back(j);
            }
            while (!pending.empty()) {
                const i64 k = pending.top();
                pending.pop();
                if (!live[k]) continue;
                for (int spin = 0; !done[k].load(std::memory_order_acquire); ++spin) {
                    if (spin < 20000)
                        __builtin_ia32_pause();
                    else
                        std::this_thread::yield();
                }
                const double m = w[k] / uv[uoff[k]];
                if (std::abs(m) < tau) {
                    w[k] = 0.0;
                    live[k] = 0;
                    continue;
                }
                w[k] = m;
                kept.push_back(k);
                for (i64 kk = uoff[k] + 1; kk < uoff[k] + ulen[k]; ++kk) {
                    const i64 j = uci[kk];
                    w[j] -= m * uv[kk];
                    if (!live[j]) {
                        live[j] = 1;
                        if (j < i)
                            pending.push(j);
                        else if (j > i)
                            upper.push_back(j);
                    }
                }
            }
            // U part first: it is all row i+1 waits for (done[i]); the L part's
            // selection is off that chain (both only read w, so the order is free)
            double d = w[i];
            if (d == 0.0) {
                if (p.pivot_patch == PivotPatch::error) {
                    i64 cur = first_zero.load();
                    while (i < cur && !first_zero.compare_exchange_weak(cur, i)) {
                    }
                    d = 1.0; // placeholder: the factorisation is abandoned below
                } else {
                    d = patch_pivot(p.droptol, row_norm2(A, i), anorm_f, p.pivot_patch, i);
                }
            }
            i64 o = uoff[i];
            uci[o] = static_cast<i32>(i), uv[o++] = d;
            select(upper, false, tau);
            for (i64 j : pat_part) uci[o] = static_cast<i32>(j), uv[o++] = w[j];
            ulen[i] = o - uoff[i];
            done[i].store(1, std::memory_order_release);

            select(kept, true, tau);
            o = loff[i];
            for (i64 j : pat_part) lci[o] = static_cast<i32>(j), lv[o++] = w[j];
            llen[i] = o - loff[i];

            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) orig[A.ci[k]] = 0;
            for (i64 j : kept) w[j] = 0.0, live[j] = 0;
            w[i] = 0.0;
            live[i] = 0;
            for (i64 j : upper) w[j] = 0.0, live[j] = 0;
        }
    };
    const int T = static_cast<int>(std::max<i64>(1, std::min<i64>(std::min(host_threads(), 16), n / 2000)));
    if (T == 1) {
        worker();
    } else {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t) pool.emplace_back(worker);
        for (auto& th : pool) th.join();
    }
    if (first_zero.load() < n) patch_pivot(0.0, 0.0, 0.0, PivotPatch::error, first_zero.load());

    HostFactors f;
    for (Csr* M : {&f.L, &f.U}) {
        M->nrows = M->ncols = n;
        M->rp.assign(static_cast<size_t>(n) + 1, 0);
    }
    for (i64 i = 0; i < n; ++i) {
        f.L.rp[i + 1] = f.L.rp[i] + llen[i];
        f.U.rp[i + 1] = f.U.rp[i] + ulen[i];
    }
    f.L.ci.resize(static_cast<size_t>(f.L.rp[n]));
    f.L.v.resize(static_cast<size_t>(f.L.rp[n]));
    f.U.ci.resize(static_cast<size_t>(f.U.rp[n]));
    f.U.v.resize(static_cast<size_t>(f.U.rp[n]));
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            std::copy(lci.begin() + loff[i], lci.begin() + loff[i] + llen[i], f.L.ci.begin() + f.L.rp[i]);
            std::copy(lv.begin() + loff[i], lv.begin() + loff[i] + llen[i], f.L.v.begin() + f.L.rp[i]);
            std::copy(uci.begin() + uoff[i], uci.begin() + uoff[i] + ulen[i], f.U.ci.begin() + f.U.rp[i]);
            std::copy(uv.begin() + uoff[i], uv.begin() + uoff[i] + ulen[i], f.U.v.begin() + f.U.rp[i]);
        }
    });
    return f;
}

HostFactors ilu_factorize(const Csr& A, const IluParams& p) {
    return p.variant == IluVariant::ilu0 ? ilu0(A, p.pivot_patch) : ilut(A, p);
}

} // namespace ilug
