#include "csr.hpp"

#include <atomic>
#include <memory>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <exception>
#include <thread>
#include <cmath>
#include <cstdlib>
#include <mutex>

namespace ilug {

int host_threads() {
    static const int n = [] {
        if (const char* e = std::getenv("ILUG_THREADS")) {
            const int v = std::atoi(e);
            if (v > 0) return v;
        }
        const unsigned hc = std::thread::hardware_concurrency();
        return hc == 0 ? 1 : static_cast<int>(std::min(hc, 64u));
    }();
    return n;
}

namespace {

// Persistent worker pool behind parallel_ranges: setup routines call it
// thousands of times (ILU(0) once per DAG level), so spawning threads per call
// cost more than the work. Workers sleep on a generation counter; the caller
// runs chunk 0 itself. A call from inside a worker, or while another host
// thread holds the pool, falls back to fresh threads (never deadlocks).
class Pool {
public:
    explicit Pool(int workers) {
        for (int w = 0; w < workers; ++w) std::thread([this, w] { loop(w + 1); }).detach();
    }
    bool try_run(i64 n, int T, const std::function<void(i64, i64, int)>& fn) {
        if (in_worker) return false;
        std::unique_lock<std::mutex> own(busy_, std::try_to_lock);
        if (!own.owns_lock()) return false;
        {
            std::lock_guard<std::mutex> g(mu_);
            fn_ = &fn;
            n_ = n;
            T_ = T;
            err_ = nullptr;
            pending_ = T - 1;
            ++gen_;
        }
        cv_.notify_all();
        run_chunk(0);
        std::unique_lock<std::mutex> g(mu_);
        done_.wait(g, [&] { return pending_ == 0; });
        fn_ = nullptr;
        if (err_) std::rethrow_exception(err_);
        return true;
    }

private:
    void run_chunk(int t) {
        const i64 b = n_ * t / T_, e = n_ * (t + 1) / T_;
        try {
            (*fn_)(b, e, t);
        } catch (...) {
            std::lock_guard<std::mutex> g(mu_);
            if (!err_) err_ = std::current_exception();
        }
    }
    void loop(int id) {
        in_worker = true;
        unsigned long long seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> g(mu_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (id >= T_) continue; // not needed for this call
            }
            run_chunk(id);
            std::lock_guard<std::mutex> g(mu_);
            if (--pending_ == 0) done_.notify_one();
        }
    }
    static thread_local bool in_worker;
    std::mutex busy_, mu_;
    std::condition_variable cv_, done_;
    const std::function<void(i64, i64, int)>* fn_ = nullptr;
    i64 n_ = 0;
    int T_ = 1, pending_ = 0;
    unsigned long long gen_ = 0;
    std::exception_ptr err_;
};
thread_local bool Pool::in_worker = false;

Pool& pool() {
    static Pool* p = new Pool(host_threads() - 1); // intentionally leaked: workers live for the process
    return *p;
}

} // namespace

void parallel_ranges(i64 n, const std::function<void(i64, i64, int)>& fn, i64 grain) {
    if (n <= 0) return;
    const int T = static_cast<int>(std::min<i64>(host_threads(), std::max<i64>(1, n / grain)));
    if (T <= 1) {
        fn(0, n, 0);
        return;
    }
    if (pool().try_run(n, T, fn)) return;
    std::vector<std::thread> threads;
    std::exception_ptr err;
    std::mutex mu;
    for (int t = 0; t < T; ++t) {
        const i64 b = n * t / T, e = n * (t + 1) / T;
        threads.emplace_back([&, b, e, t] {
            try {
                fn(b, e, t);
            } catch (...) {
                std::lock_guard<std::mutex> g(mu);
                if (!err) err = std::current_exception();
            }
        });
    }
    for (auto& th : threads) th.join();
    if (err) std::rethrow_exception(err);
}

namespace {
double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
} // namespace

SetupTimer::SetupTimer(const char* scope) : scope_(scope), on_(std::getenv("ILUG_TRACE_SETUP") != nullptr),
                                            t_(now_s()) {}

void SetupTimer::mark(const char* phase, i64 level) {
    if (!on_) return;
    const double t = now_s();
    static const double t0 = t; // the first mark of the process: absolute times are relative to it
    if (level >= 0)
        std::fprintf(stderr, "[setup] %s level %lld %-10s %8.3f s  @%.3f\n", scope_, static_cast<long long>(level),
                     phase, t - t_, t - t0);
    else
        std::fprintf(stderr, "[setup] %s %-18s %8.3f s  @%.3f\n", scope_, phase, t - t_, t - t0);
    t_ = t;
}

namespace {

[[noreturn]] void bad_triplet(const Triplet& e) {
    fail_invalid("from_triplets: index (" + std::to_string(e.i) + "," + std::to_string(e.j) + ") out of range");
}

// Serial form, the reference's exactly (src/sparse.cpp:49-86): std::sort by
// (row, col) — not stable, so three or more duplicates of one entry are summed
// in the order introsort leaves them, which only the same sort reproduces.
Csr from_triplets_serial(i64 nrows, i64 ncols, std::vector<Triplet> t, bool keep_zeros) {
    std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
        return a.i != b.i ? a.i < b.i : a.j < b.j;
    });
    Csr A;
    A.nrows = nrows;
    A.ncols = ncols;
    A.rp.assign(static_cast<size_t>(nrows) + 1, 0);
    size_t k = 0;
    while (k < t.size()) {
        const i64 i = t[k].i, j = t[k].j;
        double s = t[k].v;
        for (++k; k < t.size() && t[k].i == i && t[k].j == j; ++k) s += t[k].v;
        if (s == 0.0 && !keep_zeros) continue;
        A.ci.push_back(static_cast<i32>(j));
        A.v.push_back(s);
        ++A.rp[static_cast<size_t>(i) + 1];
    }
    for (i64 i = 0; i < nrows; ++i) A.rp[i + 1] += A.rp[i];
    return A;
}

} // namespace

Csr csr_from_triplets(i64 nrows, i64 ncols, std::vector<Triplet> t, bool keep_zeros) {
    const i64 nt = static_cast<i64>(t.size());
    // the first out-of-range triplet in input order, as the serial check reports it
    std::atomic<i64> first_bad{nt};
    parallel_ranges(nt, [&](i64 b, i64 e, int) {
        for (i64 k = b; k < e; ++k) {
            const Triplet& x = t[k];
            if (x.i < 0 || x.i >= nrows || x.j < 0 || x.j >= ncols) {
                i64 cur = first_bad.load();
                while (k < cur && !first_bad.compare_exchange_weak(cur, k)) {
                }
                return;
            }
        }
    });
    if (first_bad.load() < nt) bad_triplet(t[first_bad.load()]);
    if (nt < (i64{1} << 20)) return from_triplets_serial(nrows, ncols, std::move(t), keep_zeros);

    // Parallel form with the same result whenever no entry occurs three or more
    // times (two duplicates sum to the same value in either order): bucket
    // triplet indices by row, sort each bucket by (column, input index), sum
    // duplicates, drop exact zeros. Triple duplicates fall back to the serial
    // std::sort, whose order for them is the reference's.
    std::unique_ptr<std::atomic<i64>[]> cnt(new std::atomic<i64>[static_cast<size_t>(nrows) + 1]);
    parallel_ranges(nrows + 1, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) cnt[i].store(0, std::memory_order_relaxed);
    });
    parallel_ranges(nt, [&](i64 b, i64 e, int) {
        for (i64 k = b; k < e; ++k) cnt[t[k].i + 1].fetch_add(1, std::memory_order_relaxed);
    });
    std::vector<i64> start(static_cast<size_t>(nrows) + 1, 0);
    for (i64 i = 0; i < nrows; ++i) start[i + 1] = start[i] + cnt[i + 1].load(std::memory_order_relaxed);
    parallel_ranges(nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) cnt[i].store(start[i], std::memory_order_relaxed);
    });
    RawVec<i64> idx(static_cast<size_t>(nt));
    parallel_ranges(nt, [&](i64 b, i64 e, int) {
        for (i64 k = b; k < e; ++k) idx[cnt[t[k].i].fetch_add(1, std::memory_order_relaxed)] = k;
    });
    Csr A;
    A.nrows = nrows;
    A.ncols = ncols;
    A.rp.assign(static_cast<size_t>(nrows) + 1, 0);
    RawVec<i32> cj(static_cast<size_t>(nt));
    RawVec<double> cv(static_cast<size_t>(nt));
    std::vector<i64> kept(static_cast<size_t>(nrows), 0);
    std::atomic<bool> triple{false};
    parallel_ranges(nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            i64* lo = idx.data() + start[i];
            i64* hi = idx.data() + start[i + 1];
            std::sort(lo, hi, [&](i64 a, i64 c) { return t[a].j != t[c].j ? t[a].j < t[c].j : a < c; });
            i64 o = start[i];
            for (i64* q = lo; q < hi;) {
                const i64 j = t[*q].j;
                double s = t[*q].v;
                i64 dup = 1;
                for (++q; q < hi && t[*q].j == j; ++q, ++dup) s += t[*q].v;
                if (dup >= 3) triple.store(true, std::memory_order_relaxed);
                if (s == 0.0 && !keep_zeros) continue;
                cj[o] = static_cast<i32>(j);
                cv[o++] = s;
            }
            kept[i] = o - start[i];
        }
    });
    if (triple.load()) return from_triplets_serial(nrows, ncols, std::move(t), keep_zeros);
    for (i64 i = 0; i < nrows; ++i) A.rp[i + 1] = A.rp[i] + kept[i];
    A.ci.resize(static_cast<size_t>(A.rp[nrows]));
    A.v.resize(static_cast<size_t>(A.rp[nrows]));
    parallel_ranges(nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            std::copy(cj.begin() + start[i], cj.begin() + start[i] + kept[i], A.ci.begin() + A.rp[i]);
            std::copy(cv.begin() + start[i], cv.begin() + start[i] + kept[i], A.v.begin() + A.rp[i]);
        }
    });
    return A;
}

void csr_validate(const Csr& A, const char* what) {
    const std::string w(what);
    if (static_cast<i64>(A.rp.size()) != A.nrows + 1 || A.rp[0] != 0)
        fail_invalid(w + ": row_starts must have length nrows+1 and start at 0");
    if (A.ci.size() != A.v.size()) fail_invalid(w + ": column/value length mismatch");
    if (A.rp[A.nrows] != A.nnz()) fail_invalid(w + ": row_starts[nrows] != nnz");
    if (A.ncols > 0x7fffffff) fail_invalid(w + ": more than 2^31-1 columns");
    std::atomic<i64> bad{-1};
    parallel_ranges(A.nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            if (A.rp[i] > A.rp[i + 1]) {
                bad = i;
                return;
            }
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                const i64 j = A.ci[k];
                if (j < 0 || j >= A.ncols || (k > A.rp[i] && A.ci[k - 1] >= j)) {
                    bad = i;
                    return;
                }
            }
        }
    });
    if (bad >= 0)
        fail_invalid(w + ": invalid CSR structure at row " + std::to_string(bad.load()) +
                     " (row starts must not decrease; columns must be in range and strictly "
                     "increasing)");
}

Csr csr_from_arrays(i64 nrows, i64 ncols, const i64* rp, const i64* ci, const double* v) {
    if (nrows < 0 || ncols < 0) fail_invalid("from_csr: negative dimension");
    if (!rp) fail_invalid("from_csr: null row_starts");
    Csr A;
    A.nrows = nrows;
    A.ncols = ncols;
    A.rp.assign(rp, rp + nrows + 1);
    if (A.rp[0] != 0 || A.rp[nrows] < 0) fail_invalid("from_csr: row_starts[0] must be 0");
    const i64 nnz = A.rp[nrows];
    if (nnz > 0 && (!ci || !v)) fail_invalid("from_csr: null column/value arrays");
    A.ci.resize(static_cast<size_t>(nnz));
    A.v.assign(v, v + nnz);
    for (i64 k = 0; k < nnz; ++k) {
        if (ci[k] < 0 || ci[k] >= ncols) fail_invalid("from_csr: column index out of range");
        A.ci[k] = static_cast<i32>(ci[k]);
    }
    csr_validate(A, "from_csr");
    return A;
}

Csr csr_copy(const Csr& A) {
    Csr C;
    C.nrows = A.nrows;
    C.ncols = A.ncols;
    C.rp.resize(A.rp.size());
    C.ci.resize(A.ci.size());
    C.v.resize(A.v.size());
    auto copy = [](const auto& src, auto& dst) {
        parallel_ranges(static_cast<i64>(src.size()), [&](i64 b, i64 e, int) {
            std::copy(src.begin() + b, src.begin() + e, dst.begin() + b);
        }, 1 << 20);
    };
    copy(A.rp, C.rp);
    copy(A.ci, C.ci);
    copy(A.v, C.v);
    return C;
}

Csr csr_identity(i64 n) {
    Csr I;
    I.nrows = I.ncols = n;
    I.rp.resize(static_cast<size_t>(n) + 1);
    I.ci.resize(static_cast<size_t>(n));
    I.v.assign(static_cast<size_t>(n), 1.0);
    for (i64 i = 0; i <= n; ++i) I.rp[i] = i;
    for (i64 i = 0; i < n; ++i) I.ci[i] = static_cast<i32>(i);
    return I;
}

void csr_spmv(const Csr& A, const double* x, double* y) {
    parallel_ranges(A.nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            double s = 0.0;
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) s += A.v[k] * x[A.ci[k]];
            y[i] = s;
        }
    });
}

Csr csr_transpose(const Csr& A) {
    Csr T;
    T.nrows = A.ncols;
    T.ncols = A.nrows;
    const i64 nnz = A.nnz();
    T.ci.resize(static_cast<size_t>(nnz));
    T.v.resize(static_cast<size_t>(nnz));
    T.rp.assign(static_cast<size_t>(A.ncols) + 1, 0);
    // Column counts (atomic), offsets, an atomic-cursor scatter, then each row
    // of T sorted by source row: the same ascending source-row order as the
    // serial bucket fill, without per-thread column histograms (those were
    // threads x ncols words — gigabytes at 100 M rows).
    parallel_ranges(nnz, [&](i64 b, i64 e, int) {
        for (i64 k = b; k < e; ++k)
            std::atomic_ref<i64>(T.rp[static_cast<size_t>(A.ci[k]) + 1]).fetch_add(1, std::memory_order_relaxed);
    }, 1 << 16);
    for (i64 j = 0; j < A.ncols; ++j) T.rp[j + 1] += T.rp[j];
    RawVec<i64> cur(static_cast<size_t>(A.ncols));
    parallel_ranges(A.ncols, [&](i64 b, i64 e, int) {
        for (i64 j = b; j < e; ++j) cur[j] = T.rp[j];
    });
    parallel_ranges(A.nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i)
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                const i64 p = std::atomic_ref<i64>(cur[A.ci[k]]).fetch_add(1, std::memory_order_relaxed);
                T.ci[p] = static_cast<i32>(i);
                T.v[p] = A.v[k];
            }
    });
    parallel_ranges(A.ncols, [&](i64 b, i64 e, int) {
        std::vector<std::pair<i32, double>> tmp;
        for (i64 j = b; j < e; ++j) {
            const i64 lo = T.rp[j], hi = T.rp[j + 1];
            bool sorted = true;
            for (i64 p = lo + 1; p < hi && sorted; ++p) sorted = T.ci[p - 1] < T.ci[p];
            if (sorted) continue;
            tmp.clear();
            for (i64 p = lo; p < hi; ++p) tmp.emplace_back(T.ci[p], T.v[p]);
            std::sort(tmp.begin(), tmp.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
            for (i64 p = lo; p < hi; ++p) T.ci[p] = tmp[p - lo].first, T.v[p] = tmp[p - lo].second;
        }
    });
    return T;
}

Csr csr_matmul(const Csr& A, const Csr& B) {
    if (A.ncols != B.nrows) fail_invalid("matmul: dimension mismatch");
    Csr C;
    C.nrows = A.nrows;
    C.ncols = B.ncols;
    C.rp.assign(static_cast<size_t>(A.nrows) + 1, 0);
    const int T = std::max(1, std::min<int>(host_threads() * 4, static_cast<int>(A.nrows / 2048 + 1)));
    struct Piece {
        std::vector<i32> ci;
        std::vector<double> v;
    };
    std::vector<Piece> pieces(static_cast<size_t>(T));
    auto lo = [&](int t) { return A.nrows * t / T; };
    // Each worker keeps a dense accumulator + row marker over B's columns,
    // calloc'ed: the OS hands out zero pages lazily, so a worker only faults in
    // the pages of the columns its rows reach (a zero-filled n_coarse-sized
    // array per worker cost more than the product at 100 M rows).
    struct FreeDel {
        void operator()(void* p) const { std::free(p); }
    };
    parallel_ranges(T, [&](i64 tb, i64 te, int) {
        const size_t nc = static_cast<size_t>(std::max<i64>(B.ncols, 1));
        std::unique_ptr<double, FreeDel> work_mem(static_cast<double*>(std::calloc(nc, sizeof(double))));
        std::unique_ptr<i64, FreeDel> mark_mem(static_cast<i64*>(std::calloc(nc, sizeof(i64))));
        if (!work_mem || !mark_mem) fail_numeric("matmul: out of host memory");
        double* work = work_mem.get();
        i64* mark = mark_mem.get(); // row i marks with i + 1 (0 = untouched)
        std::vector<i32> cols;
        for (i64 t = tb; t < te; ++t) {
            Piece& pc = pieces[t];
            for (i64 i = lo(static_cast<int>(t)); i < lo(static_cast<int>(t) + 1); ++i) {
                cols.clear();
                for (i64 ka = A.rp[i]; ka < A.rp[i + 1]; ++ka) {
                    const i64 k = A.ci[ka];
                    const double aik = A.v[ka];
                    for (i64 kb = B.rp[k]; kb < B.rp[k + 1]; ++kb) {
                        const i32 j = B.ci[kb];
                        if (mark[j] != i + 1) {
                            mark[j] = i + 1;
                            cols.push_back(j);
                        }
                        work[j] += aik * B.v[kb];
                    }
                }
                std::sort(cols.begin(), cols.end());
                i64 kept = 0;
                for (i32 j : cols) {
                    const double s = work[j];
                    work[j] = 0.0;
                    if (s == 0.0) continue;
                    pc.ci.push_back(j);
                    pc.v.push_back(s);
                    ++kept;
                }
                C.rp[i + 1] = kept;
            }
        }
    }, 1);
    for (i64 i = 0; i < A.nrows; ++i) C.rp[i + 1] += C.rp[i];
    C.ci.resize(static_cast<size_t>(C.rp[A.nrows]));
    C.v.resize(static_cast<size_t>(C.rp[A.nrows]));
    parallel_ranges(T, [&](i64 tb, i64 te, int) {
        for (i64 t = tb; t < te; ++t) {
            const i64 off = C.rp[lo(static_cast<int>(t))];
            std::copy(pieces[t].ci.begin(), pieces[t].ci.end(), C.ci.begin() + off);
            std::copy(pieces[t].v.begin(), pieces[t].v.end(), C.v.begin() + off);
            Piece().ci.swap(pieces[t].ci);
            Piece().v.swap(pieces[t].v);
        }
    }, 1);
    return C;
}

std::tuple<Csr, Csr, Csr> csr_split_triangular(const Csr& A) {
    if (A.nrows != A.ncols) fail_invalid("split_triangular: matrix must be square");
    Csr L, D, U;
    for (Csr* M : {&L, &D, &U}) {
        M->nrows = A.nrows;
        M->ncols = A.ncols;
        M->rp.assign(static_cast<size_t>(A.nrows) + 1, 0);
    }
    for (i64 i = 0; i < A.nrows; ++i)
        for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            Csr& dst = A.ci[k] < i ? L : (A.ci[k] == i ? D : U);
            dst.ci.push_back(A.ci[k]);
            dst.v.push_back(A.v[k]);
            ++dst.rp[i + 1];
        }
    for (Csr* M : {&L, &D, &U})
        for (i64 i = 0; i < A.nrows; ++i) M->rp[i + 1] += M->rp[i];
    return {std::move(L), std::move(D), std::move(U)};
}

Vec csr_diag(const Csr& A) {
    if (A.nrows != A.ncols) fail_invalid("diag: matrix must be square");
    Vec d(static_cast<size_t>(A.nrows), 0.0);
    parallel_ranges(A.nrows, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i)
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k)
                if (A.ci[k] == i) {
                    d[i] = A.v[k];
                    break;
                }
    });
    return d;
}

double frobenius_norm(const Csr& A) {
    double s = 0.0;
    for (double x : A.v) s += x * x;
    return std::sqrt(s);
}

} // namespace ilug
