// K5: level-scheduled direct triangular solves and the Gauss-Seidel sweep —
// the "direct" comparison point of the paper and the reference's default
// coarse-level smoother (src/config.cpp:39).
//
// Host analysis buckets rows into wavefront levels of the dependency DAG and
// stores a level-ordered SELL-32 copy of the operator (each level padded to a
// whole number of slices, so a warp never straddles two levels). Each row is
// computed by one thread in the serial code's exact operation order
// (s = b; s -= a_ij x_j ascending; x_i = s / d), so the result is bitwise the
// sequential solve of src/trisolve.cpp:20-55 / src/smoother.cpp:113-132.
//
// Two schedules:
//  * narrow DAGs (coarse AMG levels): one 1024-thread CTA walks the levels
//    with __syncthreads between them (no grid-wide synchronisation at all);
//  * wide DAGs (finest-level factors): sync-free wavefront — warps take
//    32-row slices in level order from an atomic ticket and each row waits
//    only on its own dependencies' completion flags (acquire/release through
//    L2, epoch-stamped so nothing is reset between solves). A slice only
//    depends on slices handed out before it, so progress never depends on CTA
//    residency and no cooperative launch or global barrier is needed.
#include "levelset.hpp"

#include <cuda/atomic>

#include <algorithm>
#include <cstdlib>
#include <string>

namespace ilug {

namespace {

constexpr int kSmallBlock = 384; // the prefetched row state needs ~150 registers per thread
constexpr int kFlagBlock = 256;

// MODE 0: unit lower, strict storage: x_i = b_i - sum L_ij x_j
// MODE 1: upper with stored diagonal: x_i = (b_i - sum_{j != i} U_ij x_j) / U_ii
// MODE 2: Gauss-Seidel on A: x'_i = (b_i - sum_{j<i} a_ij x'_j - sum_{j>i} a_ij x_j) / a_ii
template <int MODE>
__device__ __forceinline__ bool is_dep(i32 j, i64 row) {
    return MODE == 1 ? j > row : j < row;
}

// One row in the serial operation order. Entries are processed in chunks of
// kChunk: all column/value loads of a chunk are issued first, then the x
// gathers (waiting on the producers' flags in the sync-free schedule), then
// the ordered accumulation — a row costs ~2 memory latencies per chunk instead
// of 2 per entry.
template <int MODE, bool FLAGS, int kChunk = FLAGS ? 16 : 8>
__device__ __forceinline__ void level_row(const SellView& M, i64 p, i64 row, const double* __restrict__ b,
                                          double* x, const double* __restrict__ xold, unsigned* flags,
                                          unsigned E) {
    const int len = M.rowlen[p];
    const i64 base = M.slice_ptr[p >> 5] + (p & 31);
    double s = b[row], d = 1.0;
    for (int t0 = 0; t0 < len; t0 += kChunk) {
        i32 c[kChunk];
        double a[kChunk], xv[kChunk];
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            if (t0 + u < len) {
                const i64 q = base + static_cast<i64>(t0 + u) * kSlice;
                c[u] = __ldg(M.cols + q);
                a[u] = __ldg(M.vals + q);
            }
        }
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            xv[u] = 0.0;
            if (t0 + u < len && !(MODE != 0 && c[u] == row)) {
                const i32 j = c[u];
                if (is_dep<MODE>(j, row)) {
                    if (FLAGS) {
                        // relaxed polls with back-off, one acquire once seen
                        if (ld_acquire_flag(flags + j) != E) {
                            for (int spin = 0; ld_relaxed_flag(flags + j) != E; ++spin)
                                if (spin > 8) __nanosleep(64);
                            (void)ld_acquire_flag(flags + j);
                        }
                    }
                    xv[u] = __ldcg(x + j);
                } else {
                    xv[u] = xold[j]; // GS: not-yet-updated neighbour (MODE 2 only)
                }
            }
        }
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            if (t0 + u < len) {
                if (MODE != 0 && c[u] == row)
                    d = a[u];
                else
                    s = s - a[u] * xv[u];
            }
        }
    }
    x[row] = MODE == 0 ? s : s / d;
}

// Bulk (TMA-engine) prefetch of a byte range into L2; no completion tracking.
__device__ __forceinline__ void l2_prefetch(const void* p, i64 bytes) {
    const char* a = static_cast<const char*>(p);
    const uintptr_t lo = reinterpret_cast<uintptr_t>(a) & ~uintptr_t(15);
    const uintptr_t hi = (reinterpret_cast<uintptr_t>(a) + static_cast<uintptr_t>(bytes) + 15) & ~uintptr_t(15);
    for (uintptr_t s = lo; s < hi; s += (1u << 20)) { // chunks of at most 1 MiB
        const unsigned len = static_cast<unsigned>(hi - s < (1u << 20) ? hi - s : (1u << 20));
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s), "r"(len) : "memory");
    }
}

template <int MODE>
__global__ void __launch_bounds__(kSmallBlock)
k_levels_cta(SellView M, const i64* __restrict__ level_ptr, int nlev, const double* __restrict__ b,
             double* x, const double* __restrict__ xold) {
    // Level L+2's operator slices are one contiguous range of the level-ordered
    // SELL: one thread asks the copy engine to pull them into L2 while the CTA
    // works on level L, so a level's loads are L2 hits, not DRAM misses.
    auto prefetch_level = [&](int L) {
        if (L >= nlev) return;
        const i64 s0 = level_ptr[L] >> 5, s1 = level_ptr[L + 1] >> 5;
        const i64 e0 = M.slice_ptr[s0], e1 = M.slice_ptr[s1];
        if (e1 > e0) {
            l2_prefetch(M.vals + e0, (e1 - e0) * 8);
            l2_prefetch(M.cols + e0, (e1 - e0) * 4);
        }
        l2_prefetch(M.perm + level_ptr[L], (level_ptr[L + 1] - level_ptr[L]) * 4);
    };
    if (threadIdx.x == 0) {
        prefetch_level(0);
        prefetch_level(1);
    }
    // Software pipeline: everything a row needs except x (its perm entry,
    // length, slice base, b value and first kPre column/value pairs) is loaded
    // for level L+1 before the barrier that ends level L, so the critical path
    // per level is one gather of x plus the ordered accumulation.
    constexpr int kPre = 16;
    struct Next {
        i64 p = -1, row = -1, base = 0;
        int len = 0;
        double bv = 0.0;
        i32 c[kPre];
        double a[kPre];
    } nx;
    auto fetch = [&](int L) {
        nx.p = -1;
        if (L >= nlev) return;
        const i64 p = level_ptr[L] + threadIdx.x;
        if (p >= level_ptr[L + 1]) return;
        nx.p = p;
        nx.row = M.perm[p];
        if (nx.row < 0) return;
        nx.len = M.rowlen[p];
        nx.base = M.slice_ptr[p >> 5] + (p & 31);
        nx.bv = b[nx.row];
#pragma unroll
        for (int u = 0; u < kPre; ++u)
            if (u < nx.len) {
                const i64 q = nx.base + static_cast<i64>(u) * kSlice;
                nx.c[u] = __ldg(M.cols + q);
                nx.a[u] = __ldg(M.vals + q);
            }
    };
    fetch(0);
    for (int L = 0; L < nlev; ++L) {
        if (threadIdx.x == 0) prefetch_level(L + 2);
        if (nx.p >= 0 && nx.row >= 0) {
            const i64 row = nx.row;
            double s = nx.bv, d = 1.0, xv[kPre];
#pragma unroll
            for (int u = 0; u < kPre; ++u) {
                xv[u] = 0.0;
                if (u < nx.len && !(MODE != 0 && nx.c[u] == row))
                    xv[u] = (MODE == 2 && nx.c[u] > row) ? xold[nx.c[u]] : __ldcg(x + nx.c[u]);
            }
#pragma unroll
            for (int u = 0; u < kPre; ++u)
                if (u < nx.len) {
                    if (MODE != 0 && nx.c[u] == row)
                        d = nx.a[u];
                    else
                        s = s - nx.a[u] * xv[u];
                }
            for (int t0 = kPre; t0 < nx.len; t0 += 8) { // long rows: the tail in batched chunks
                i32 c[8];
                double a[8], xt[8];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (t0 + u < nx.len) {
                        const i64 q = nx.base + static_cast<i64>(t0 + u) * kSlice;
                        c[u] = __ldg(M.cols + q);
                        a[u] = __ldg(M.vals + q);
                    }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    xt[u] = 0.0;
                    if (t0 + u < nx.len && !(MODE != 0 && c[u] == row))
                        xt[u] = (MODE == 2 && c[u] > row) ? xold[c[u]] : __ldcg(x + c[u]);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (t0 + u < nx.len) {
                        if (MODE != 0 && c[u] == row)
                            d = a[u];
                        else
                            s = s - a[u] * xt[u];
                    }
            }
            x[row] = MODE == 0 ? s : s / d;
        }
        // rows beyond the first blockDim.x of a wide level
        const i64 end = level_ptr[L + 1];
        for (i64 p = level_ptr[L] + threadIdx.x + blockDim.x; p < end; p += blockDim.x) {
            const i64 row = M.perm[p];
            if (row >= 0) level_row<MODE, false, 8>(M, p, row, b, x, xold, nullptr, 0u);
        }
        fetch(L + 1);
        __syncthreads();
    }
}

__global__ void k_epoch_bump(unsigned* epoch, unsigned* ticket) {
    *epoch = *epoch + 1u;
    *ticket = 0u;
}

template <int MODE>
__global__ void __launch_bounds__(kFlagBlock)
k_levels_flags(SellView M, i64 nslices, const double* __restrict__ b, double* x,
               const double* __restrict__ xold, unsigned* flags, const unsigned* __restrict__ epoch_p,
               unsigned* ticket) {
    const unsigned E = *epoch_p;
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned s = 0;
        if (lane == 0) s = atomicAdd(ticket, 1u);
        s = __shfl_sync(0xffffffffu, s, 0);
        if (s >= nslices) return;
        const i64 p = static_cast<i64>(s) * kSlice + lane;
        const i64 row = M.perm[p];
        if (row < 0) continue;
        level_row<MODE, true>(M, p, row, b, x, xold, flags, E);
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> f(flags[row]);
        f.store(E, cuda::memory_order_release);
    }
}

template <int MODE>
const void* cta_kernel() {
    return reinterpret_cast<const void*>(k_levels_cta<MODE>);
}
template <int MODE>
const void* flag_kernel() {
    return reinterpret_cast<const void*>(k_levels_flags<MODE>);
}

} // namespace

void LevelPlan::build(const Csr& T, Kind kind, cudaStream_t st, const double* dev_vals) {
    kind_ = kind;
    const i64 n = T.nrows;
    std::vector<i32> lev(static_cast<size_t>(n), 0);
    int nl = n > 0 ? 1 : 0;
    if (kind == Kind::upper) {
        for (i64 i = n; i-- > 0;) {
            i32 l = 0;
            for (i64 k = T.rp[i]; k < T.rp[i + 1]; ++k)
                if (T.ci[k] > i) l = std::max(l, lev[T.ci[k]] + 1);
            lev[i] = l;
            nl = std::max(nl, l + 1);
        }
    } else {
        for (i64 i = 0; i < n; ++i) {
            i32 l = 0;
            for (i64 k = T.rp[i]; k < T.rp[i + 1]; ++k)
                if (T.ci[k] < i) l = std::max(l, lev[T.ci[k]] + 1);
            lev[i] = l;
            nl = std::max(nl, l + 1);
        }
    }
    nlev_ = nl;
    std::vector<i64> cnt(static_cast<size_t>(nl) + 1, 0);
    for (i64 i = 0; i < n; ++i) ++cnt[lev[i] + 1];
    std::vector<i64> lp(static_cast<size_t>(nl) + 1, 0); // padded SELL row offsets
    max_level_rows_ = 0;
    for (int l = 0; l < nl; ++l) {
        lp[l + 1] = lp[l] + (cnt[l + 1] + kSlice - 1) / kSlice * kSlice;
        max_level_rows_ = std::max(max_level_rows_, cnt[l + 1]);
    }
    std::vector<i32> perm(static_cast<size_t>(lp[nl]), -1);
    std::vector<i64> cur(lp.begin(), lp.end() - 1);
    for (i64 i = 0; i < n; ++i) perm[cur[lev[i]]++] = static_cast<i32>(i);
    level_ptr_.upload(lp.data(), nl + 1, st);

    DBuf<i64> rp;
    DBuf<i32> ci;
    DBuf<double> v;
    rp.upload(T.rp.data(), n + 1, st);
    ci.upload(T.ci.data(), T.nnz(), st);
    if (!dev_vals) v.upload(T.v.data(), T.nnz(), st);
    sell_from_device_csr(M_, T, rp.p, ci.p, dev_vals ? dev_vals : v.p, Part::all, perm, st);

    // Narrow DAG (average level width below two CTAs' worth): one CTA.
    // One CTA only for tiny systems: with __syncthreads per level every level
    // costs its full row latency; the sync-free schedule overlaps the loads of
    // later levels with the wait on earlier ones, which wins as soon as there
    // is more than a CTA's worth of rows.
    single_cta_ = n <= 4 * kSmallBlock || n / std::max(nl, 1) <= kSmallBlock;
    if (const char* force = std::getenv("ILUG_LEVELSET")) { // test hook: cta | flags
        if (std::string(force) == "cta") single_cta_ = true;
        if (std::string(force) == "flags" && n > 0) single_cta_ = false;
    }
    if (!single_cta_) {
        flags_.alloc(n + 2); // [0, n) row flags, n epoch, n+1 ticket
        ILUG_CUDA(cudaMemsetAsync(flags_.p, 0, static_cast<size_t>(n + 2) * sizeof(unsigned), st));
        const i64 slices = M_.nrows_pad / kSlice;
        grid_ = static_cast<int>(std::min<i64>((slices + kFlagBlock / 32 - 1) / (kFlagBlock / 32),
                                               static_cast<i64>(device_sm_count()) * 8));
    } else {
        grid_ = 1;
    }
    ILUG_CUDA(cudaStreamSynchronize(st));
}

void LevelPlan::solve(const double* b, double* x, const double* xold, cudaStream_t st) const {
    if (M_.nrows == 0) return;
    SellView mv = view(M_);
    const int mode = kind_ == Kind::lower_unit ? 0 : (kind_ == Kind::upper ? 1 : 2);
    if (single_cta_) {
        const i64* lp = level_ptr_.p;
        int nl = nlev_;
        void* args[] = {&mv, &lp, &nl, &b, &x, &xold};
        const void* fn = mode == 0 ? cta_kernel<0>() : mode == 1 ? cta_kernel<1>() : cta_kernel<2>();
        ILUG_CUDA(cudaLaunchKernel(fn, dim3(1), dim3(kSmallBlock), args, 0, st));
        return;
    }
    const i64 n = M_.nrows;
    unsigned* flags = flags_.p;
    unsigned* epoch = flags_.p + n;
    unsigned* ticket = flags_.p + n + 1;
    k_epoch_bump<<<1, 1, 0, st>>>(epoch, ticket);
    ILUG_LAUNCH_CHECK();
    i64 ns = M_.nrows_pad / kSlice;
    const unsigned* ep = epoch;
    void* args[] = {&mv, &ns, &b, &x, &xold, &flags, &ep, &ticket};
    const void* fn = mode == 0 ? flag_kernel<0>() : mode == 1 ? flag_kernel<1>() : flag_kernel<2>();
    ILUG_CUDA(cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid_)), dim3(kFlagBlock), args, 0, st));
}

} // namespace ilug
