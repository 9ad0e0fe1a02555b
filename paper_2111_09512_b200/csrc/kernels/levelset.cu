// K5: level-scheduled direct triangular solves and the Gauss-Seidel sweep —
// the "direct" comparison point of the paper and the reference's default
// coarse-level smoother (src/config.cpp:39).
//
// Host analysis buckets rows into wavefront levels of the dependency DAG and
// stores a level-ordered SELL-32 copy of the operator (each level padded to a
// whole number of slices, so a warp never straddles two levels). Every row is
// computed in the serial code's exact operation order (s = b; s -= a_ij x_j
// ascending; x_i = s / d), so the result is bitwise the sequential solve of
// src/trisolve.cpp:20-55 / src/smoother.cpp:113-132.
//
// Schedules (LevelPlan::build picks by the average rows per level):
//  * narrow DAGs (<= 512 rows per level: coarse AMG levels): k_levels_warp,
//    one thread-block cluster walks the levels with barrier.cluster between
//    them; a warp per row (products in parallel, ordered shuffle-chain sum);
//  * wide DAGs (finest-level factors): k_levels_vflags, sync-free — warps take
//    32-row slices in level order from an atomic ticket, thread per row, and
//    the solution entries themselves are the completion flags (sentinel-
//    filled x, relaxed 64-bit publish/poll). A slice only depends on slices
//    handed out before it, so progress never depends on CTA residency.
//  * A/B and test forms: k_levels_cta (one CTA, thread per row, ILUG_LEVELSET=
//    cta1) and k_levels_flags (separate epoch-stamped flags, =flags).
#include "levelset.hpp"

#include <cooperative_groups.h>
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
// Set by a sync-free kernel whose dependency wait exceeded its bound (a
// scheduling fault, never a slow producer); read and cleared by
// levelset_check_error() at the callers' sync points.
__device__ unsigned g_levelset_timeout;

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
        if (FLAGS) {
            // every producer flag of the chunk polled at once (relaxed, all in
            // flight), then one acquire fence for the chunk: ~1 round trip per
            // chunk instead of one serial acquire (LD.STRONG + CCTL.IVALL) per
            // dependency
            bool ready = false;
            for (int spin = 0; !ready; ++spin) {
                ready = true;
#pragma unroll
                for (int u = 0; u < kChunk; ++u)
                    if (t0 + u < len && !(MODE != 0 && c[u] == row) && is_dep<MODE>(c[u], row))
                        ready &= ld_relaxed_flag(flags + c[u]) == E;
                if (!ready && spin > 8) __nanosleep(64);
                if (!ready && spin > (1 << 24)) { // seconds: a scheduling bug, not a slow producer
                    atomicExch(&g_levelset_timeout, 1u);
                    break;
                }
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
#pragma unroll
        for (int u = 0; u < kChunk; ++u) {
            xv[u] = 0.0;
            if (t0 + u < len && !(MODE != 0 && c[u] == row))
                xv[u] = is_dep<MODE>(c[u], row) ? __ldcg(x + c[u]) : xold[c[u]]; // xold: GS (MODE 2) only
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

__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

// Level-synchronous schedule on one thread-block cluster (1..16 CTAs on one
// GPC): the cluster's threads split each level's rows, and a hardware cluster
// barrier (barrier.cluster arrive.release / wait.acquire, ~0.2 us) separates
// the levels, so a level costs one row latency plus the barrier, with up to 16
// SMs of load bandwidth instead of one. x crosses CTAs through L2 (__ldcg),
// ordered by the barrier's release/acquire at cluster scope.
template <int MODE>
__global__ void __launch_bounds__(kSmallBlock)
k_levels_cta(SellView M, const i64* __restrict__ level_ptr, int nlev, const double* __restrict__ b,
             double* x, const double* __restrict__ xold) {
    const unsigned crank = cluster_rank(), csize = cluster_size();
    const i64 gtid = static_cast<i64>(crank) * blockDim.x + threadIdx.x;
    const i64 gthreads = static_cast<i64>(csize) * blockDim.x;
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
    if (gtid == 0) {
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
        const i64 p = level_ptr[L] + gtid;
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
        if (gtid == 0) prefetch_level(L + 2);
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
        // rows beyond the cluster's first gthreads of a wide level
        const i64 end = level_ptr[L + 1];
        for (i64 p = level_ptr[L] + gtid + gthreads; p < end; p += gthreads) {
            const i64 row = M.perm[p];
            if (row >= 0) level_row<MODE, false, 8>(M, p, row, b, x, xold, nullptr, 0u);
        }
        fetch(L + 1);
        if (csize > 1) {
            asm volatile("barrier.cluster.arrive.release.aligned;\n"
                         "barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            __syncthreads();
        }
    }
}

// ---------------------------------------------------------------------------
// Cluster schedule, warp per row (the default for narrow DAGs: coarse AMG
// levels' Gauss-Seidel, factor solves with few rows per level).
//
// A thread-per-row kernel on one SM issues a row's ~40 dependent
// gather/multiply/subtract steps serially with almost no other warps to hide
// their latency (ncu: ~1000 issued instructions per level per warp at 85
// cycles each, 15-40 us per level). Here a warp takes a row: lane t loads
// entry t (and t+32), gathers its x value and forms the product a_t * x_t —
// the same rounded product the serial loop forms — and the ordered
// accumulation s = b - p_0 - p_1 - ... runs as a chain of shuffles, so the
// result is still bitwise the serial one. The warps of a thread-block cluster
// (up to 16 CTAs on one GPC) split each level's rows; a hardware cluster
// barrier (barrier.cluster arrive.release / wait.acquire) separates levels.
// Row metadata is loaded two levels ahead and the first row's columns/values
// one level ahead, so a level costs one x gather plus the shuffle chain.
constexpr int kWarpBlock = 512;       // narrow levels (fewer warps per barrier)
constexpr int kWarpBlockWide = 1024;  // levels with more rows than 2 per warp of a 512-thread cluster
constexpr int kMaxSmemLevels = 6000; // level_ptr staged in (static) shared memory

struct RowMeta {
    i64 row = -1; // -1: no row / padding
    i64 base = 0;
    int len = 0;
};
struct RowData {
    i32 c0 = -1, c1 = -1;
    double a0 = 0.0, a1 = 0.0, bv = 0.0;
    double xo0 = 0.0, xo1 = 0.0; // SX, GS: xold at columns > row, prefetched with the row
};

// Q rows per warp at once (one per prefetch slot): every slot's x gathers are
// issued before any slot's shuffle chain, so the slots' memory latencies
// overlap. Entries 0..63 come from the prefetched registers; longer rows load
// the rest inline.
template <int MODE, int Q, bool SX = false>
__device__ __forceinline__ void warp_rows(const SellView& M, const RowMeta (&m)[Q], const RowData (&r)[Q], int lane,
                                          double* x, const double* __restrict__ xold, double* sx = nullptr) {
    const unsigned full = 0xffffffffu;
    double s[Q], d[Q];
    int maxlen = 0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        s[q] = r[q].bv;
        d[q] = 1.0;
        if (m[q].row >= 0) maxlen = max(maxlen, m[q].len);
    }
    for (int t0 = 0; t0 < maxlen; t0 += 32) {
        double prod[Q];
        unsigned dm[Q];
        int cnt[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const i64 row = m[q].row;
            const bool valid = row >= 0 && t0 < m[q].len; // warp-uniform
            const int t = t0 + lane;
            const bool act = valid && t < m[q].len;
            i32 c;
            double a, xo = 0.0;
            if (t0 == 0) {
                c = r[q].c0, a = r[q].a0, xo = r[q].xo0;
            } else if (t0 == 32) {
                c = r[q].c1, a = r[q].a1, xo = r[q].xo1;
            } else {
                c = act ? __ldg(M.cols + m[q].base + static_cast<i64>(t) * kSlice) : -1;
                a = act ? __ldg(M.vals + m[q].base + static_cast<i64>(t) * kSlice) : 0.0;
                if (SX && act && !is_dep<MODE>(c, row) && c != row) xo = __ldg(xold + c);
            }
            const bool isd = act && MODE != 0 && c == row;
            double xv = 0.0;
            if (act && !isd) {
                if (SX) // the solution lives in shared memory; GS's old values were prefetched
                    xv = is_dep<MODE>(c, row) ? sx[c] : xo;
                else
                    xv = is_dep<MODE>(c, row) ? __ldcg(x + c) : __ldg(xold + c); // xold: GS only
            }
            prod[q] = a * xv; // the serial loop's rounded product
            dm[q] = __ballot_sync(full, isd);
            if (dm[q]) d[q] = __shfl_sync(full, a, __ffs(dm[q]) - 1);
            cnt[q] = valid ? min(32, m[q].len - t0) : 0;
        }
#pragma unroll
        for (int q = 0; q < Q; ++q)
            for (int u = 0; u < cnt[q]; ++u) {
                const double pu = __shfl_sync(full, prod[q], u);
                if (!((dm[q] >> u) & 1u)) s[q] = s[q] - pu;
            }
    }
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < Q; ++q)
            if (m[q].row >= 0) {
                const double v = MODE == 0 ? s[q] : s[q] / d[q];
                if (SX)
                    sx[m[q].row] = v;
                else
                    x[m[q].row] = v;
            }
    }
}

// SX (one CTA, n <= kSmemXRows): the solution is kept in shared memory, so a
// row's dependency gathers are shared-memory reads (~30 cycles) instead of L2
// round trips; the rows' matrix entries and GS's old neighbour values do not
// depend on the sweep and are prefetched a level ahead as before. x is written
// back once at the end.
constexpr i64 kSmemXRows = 16384;

template <int MODE, int BLOCK, int Q, bool SX = false>
__global__ void __launch_bounds__(BLOCK, 1)
k_levels_warp(SellView M, const i64* __restrict__ level_ptr, int nlev, const double* __restrict__ b, double* x,
              const double* __restrict__ xold, i64 n) {
    __shared__ i64 slp[kMaxSmemLevels + 1];
    extern __shared__ double sx[]; // SX: the solution vector
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned csize = cluster_size();
    const i64 gw = static_cast<i64>(cluster_rank()) * (BLOCK / 32) + warp;
    const i64 GW = static_cast<i64>(csize) * (BLOCK / 32);
    for (int l = threadIdx.x; l <= nlev; l += blockDim.x) slp[l] = level_ptr[l];
    __syncthreads();

    // slot q of level L: the level's row gw + q * GW
    auto load_meta = [&](int L, int q, RowMeta& m) {
        m.row = -1;
        if (L >= nlev) return;
        const i64 p = slp[L] + gw + q * GW;
        if (p >= slp[L + 1]) return;
        m.row = M.perm[p];
        m.len = M.rowlen[p];
        m.base = M.slice_ptr[p >> 5] + (p & 31);
    };
    auto load_data = [&](const RowMeta& m, RowData& r) {
        if (m.row < 0) return;
        r.c0 = lane < m.len ? __ldg(M.cols + m.base + static_cast<i64>(lane) * kSlice) : -1;
        r.a0 = lane < m.len ? __ldg(M.vals + m.base + static_cast<i64>(lane) * kSlice) : 0.0;
        r.c1 = lane + 32 < m.len ? __ldg(M.cols + m.base + static_cast<i64>(lane + 32) * kSlice) : -1;
        r.a1 = lane + 32 < m.len ? __ldg(M.vals + m.base + static_cast<i64>(lane + 32) * kSlice) : 0.0;
        r.bv = b[m.row];
        if (SX && MODE == 2) { // GS's old values at columns > row (independent of the sweep)
            r.xo0 = r.c0 > m.row ? __ldg(xold + r.c0) : 0.0;
            r.xo1 = r.c1 > m.row ? __ldg(xold + r.c1) : 0.0;
        }
    };

    RowMeta mc[Q], m1[Q], m2[Q];
    RowData dc[Q], d1[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
        load_meta(0, q, mc[q]);
        load_data(mc[q], dc[q]);
        load_meta(1, q, m1[q]);
    }
    for (int L = 0; L < nlev; ++L) {
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            load_data(m1[q], d1[q]);  // level L+1's rows, one level ahead
            load_meta(L + 2, q, m2[q]); // two ahead
        }
        warp_rows<MODE, Q, SX>(M, mc, dc, lane, x, xold, sx);
        // further rows of a level wider than the cluster's warps x slots
        for (i64 p = slp[L] + gw + Q * GW; p < slp[L + 1]; p += GW) {
            RowMeta m[1];
            RowData r[1];
            m[0].row = M.perm[p];
            if (m[0].row < 0) continue;
            m[0].len = M.rowlen[p];
            m[0].base = M.slice_ptr[p >> 5] + (p & 31);
            load_data(m[0], r[0]);
            warp_rows<MODE, 1, SX>(M, m, r, lane, x, xold, sx);
        }
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            mc[q] = m1[q];
            dc[q] = d1[q];
            m1[q] = m2[q];
        }
        if (csize > 1) {
            asm volatile("barrier.cluster.arrive.release.aligned;\n"
                         "barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            __syncthreads();
        }
    }
    if (SX) // rows are computed once each; padding rows of the plan never touch sx
        for (i64 i = threadIdx.x; i < n; i += blockDim.x) x[i] = sx[i];
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

// ---------------------------------------------------------------------------
// Sync-free schedule with the solution values as their own flags (default for
// wide DAGs). x is filled with a signalling-NaN sentinel that arithmetic never
// produces (GPU results are quiet NaNs), every row publishes its value with a
// single relaxed 64-bit store, and a row polls its dependencies' x entries
// directly: the value it is waiting for is the value it needs, so there is no
// separate flag, no acquire fence and no release fence on the critical path
// (one L2 round trip per level instead of ~4 plus two MEMBARs; the separate
// flag form measured 7.5-18.7 us per level at C2 vs 2.5 us for cuSPARSE SpSV).
// A row whose result has the sentinel's exact bits (only possible when an
// empty row copies that sNaN from b) publishes the canonical NaN instead.
constexpr unsigned long long kXSentinel = 0x7FF0DEAD5EA1ED01ull; // signalling NaN

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(double* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void k_fill_sentinel(double* x, i64 n) {
    const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) reinterpret_cast<unsigned long long*>(x)[i] = kXSentinel;
}

// HOIST: the row length and slice start are loaded with perm[p] (a padding
// slot runs len = 0 and publishes nothing) instead of after the padding test,
// which the compiler otherwise turns into two dependent round trips.
template <int MODE, bool HOIST = true, int kChunk = 16>
__global__ void __launch_bounds__(kFlagBlock)
k_levels_vflags(SellView M, i64 nslices, const double* __restrict__ b, double* x, const double* __restrict__ xold,
                unsigned* ticket) {
    const int lane = threadIdx.x & 31;
    for (;;) {
        unsigned sl = 0;
        if (lane == 0) sl = atomicAdd(ticket, 1u);
        sl = __shfl_sync(0xffffffffu, sl, 0);
        if (sl >= nslices) return;
        const i64 p = static_cast<i64>(sl) * kSlice + lane;
        int len = HOIST ? M.rowlen[p] : 0;
        i64 base = HOIST ? M.slice_ptr[p >> 5] + (p & 31) : 0;
        i64 row = M.perm[p];
        const bool valid = row >= 0;
        if (!HOIST) {
            if (!valid) continue;
            len = M.rowlen[p];
            base = M.slice_ptr[p >> 5] + (p & 31);
        } else if (!valid) {
            len = 0, row = 0;
        }
        double s = b[row], d = 1.0;
        for (int t0 = 0; t0 < len; t0 += kChunk) {
            i32 c[kChunk];
            double a[kChunk], xv[kChunk];
#pragma unroll
            for (int u = 0; u < kChunk; ++u)
                if (t0 + u < len) {
                    const i64 q = base + static_cast<i64>(t0 + u) * kSlice;
                    c[u] = __ldg(M.cols + q);
                    a[u] = __ldg(M.vals + q);
                }
            // dependencies: poll the values themselves (all of the chunk in flight)
            unsigned pend = 0;
#pragma unroll
            for (int u = 0; u < kChunk; ++u) {
                xv[u] = 0.0;
                if (t0 + u < len && !(MODE != 0 && c[u] == row)) {
                    if (is_dep<MODE>(c[u], row)) {
                        const unsigned long long v = ld_relaxed_u64(x + c[u]);
                        xv[u] = __longlong_as_double(static_cast<long long>(v));
                        if (v == kXSentinel) pend |= 1u << u;
                    } else {
                        xv[u] = __ldg(xold + c[u]); // GS (MODE 2) only
                    }
                }
            }
            long long spins = 0;
            while (pend) {
                if (++spins > (1ll << 26)) { // seconds: a scheduling bug, not a slow producer
                    atomicExch(&g_levelset_timeout, 1u);
                    break;
                }
                __nanosleep(32);
#pragma unroll
                for (int u = 0; u < kChunk; ++u)
                    if ((pend >> u) & 1u) {
                        const unsigned long long v = ld_relaxed_u64(x + c[u]);
                        if (v != kXSentinel) {
                            xv[u] = __longlong_as_double(static_cast<long long>(v));
                            pend &= ~(1u << u);
                        }
                    }
            }
#pragma unroll
            for (int u = 0; u < kChunk; ++u)
                if (t0 + u < len) {
                    if (MODE != 0 && c[u] == row)
                        d = a[u];
                    else
                        s = s - a[u] * xv[u];
                }
        }
        const double r = MODE == 0 ? s : s / d;
        unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(r));
        if (bits == kXSentinel) bits = 0x7FFFFFFFFFFFFFFFull; // the canonical NaN
        if (valid) st_relaxed_u64(x + row, bits);
    }
}

// Sub-warp form of the value-flag schedule: W lanes per row, a ticket per
// group of 32/W rows of one slice. Lane j of a row's sub-warp holds entries
// j, j+W, j+2W, ... (E of them per pass: a row of up to W*E entries is one
// pass, so all its dependency polls are in flight together and no second
// chunk waits behind the first); the products a_t x_t are formed in the
// lanes and the row's leader lane subtracts them from b in ascending column
// order through a shuffle chain — the reference's serial operation order, so
// the result stays bitwise. Fewer registers per row than the thread-per-row
// form (whose 16-entry chunk split the 17-19-entry ILUT rows into two
// dependent polling rounds).
template <int MODE, int W, int E = 32 / W>
__global__ void __launch_bounds__(kFlagBlock)
k_levels_vsub(SellView M, i64 ngroups, const double* __restrict__ b, double* x, const double* __restrict__ xold,
              unsigned* ticket, unsigned sleep_ns) {
    constexpr int RPG = 32 / W; // rows per group (per warp); E: entries per lane per pass
    const int lane = threadIdx.x & 31;
    const int sub = lane / W, j = lane % W;
    for (;;) {
        unsigned g = 0;
        if (lane == 0) g = atomicAdd(ticket, 1u);
        g = __shfl_sync(0xffffffffu, g, 0);
        if (g >= ngroups) return;
        const i64 sl = g / W;
        const int q = static_cast<int>(g % W) * RPG + sub;
        const i64 p = sl * kSlice + q;
        int len = M.rowlen[p];
        const i64 base = M.slice_ptr[sl] + q;
        i64 row = M.perm[p];
        const bool valid = row >= 0;
        if (!valid) len = 0, row = 0;
        double s = j == 0 ? b[row] : 0.0, d = 1.0;
        // passes: every lane of the warp runs the same number (shuffles are warp-wide)
        int maxlen = len;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
        for (int t0 = 0; t0 < maxlen; t0 += W * E) {
            i32 c[E];
            double a[E], pr[E];
            int kind[E]; // 0 product, 1 diagonal (pr = a_ii), 2 none
            unsigned pend = 0;
#pragma unroll
            for (int u = 0; u < E; ++u) {
                const int t = t0 + j + W * u;
                kind[u] = 2;
                pr[u] = 0.0;
                if (t < len) {
                    const i64 qq = base + static_cast<i64>(t) * kSlice;
                    c[u] = __ldg(M.cols + qq);
                    a[u] = __ldg(M.vals + qq);
                }
            }
#pragma unroll
            for (int u = 0; u < E; ++u) {
                const int t = t0 + j + W * u;
                if (t < len) {
                    if (MODE != 0 && c[u] == row) {
                        kind[u] = 1;
                    } else if (is_dep<MODE>(c[u], row)) {
                        const unsigned long long v = ld_relaxed_u64(x + c[u]);
                        pr[u] = __longlong_as_double(static_cast<long long>(v));
                        kind[u] = 0;
                        if (v == kXSentinel) pend |= 1u << u;
                    } else {
                        pr[u] = __ldg(xold + c[u]); // GS (MODE 2) only
                        kind[u] = 0;
                    }
                }
            }
            long long spins = 0;
            while (pend) {
                if (++spins > (1ll << 26)) {
                    atomicExch(&g_levelset_timeout, 1u);
                    break;
                }
                __nanosleep(sleep_ns);
#pragma unroll
                for (int u = 0; u < E; ++u)
                    if ((pend >> u) & 1u) {
                        const unsigned long long v = ld_relaxed_u64(x + c[u]);
                        if (v != kXSentinel) {
                            pr[u] = __longlong_as_double(static_cast<long long>(v));
                            pend &= ~(1u << u);
                        }
                    }
            }
            // one shuffle per slot: products in the lanes, +0.0 in empty and
            // diagonal slots (s - 0.0 == s exactly); the diagonal (U: entry 0,
            // GS: anywhere) is fetched once from the lane that holds it
            bool has_d = false;
            double dl = 0.0;
#pragma unroll
            for (int u = 0; u < E; ++u) {
                if (MODE != 0 && kind[u] == 1) dl = a[u], has_d = true;
                pr[u] = kind[u] == 0 ? a[u] * pr[u] : 0.0;
            }
            if (MODE != 0) {
                const unsigned bal = __ballot_sync(0xffffffffu, has_d);
                const unsigned mine = (bal >> (sub * W)) & ((W == 32 ? 0u : (1u << W)) - 1u);
                const double dv = __shfl_sync(0xffffffffu, dl, sub * W + (mine ? __ffs(mine) - 1 : 0));
                if (mine) d = dv;
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < E; ++u) {
                if (t0 + W * u >= maxlen) break; // no row of the warp has entries in this slot
#pragma unroll
                for (int jj = 0; jj < W; ++jj) {
                    const double v = __shfl_sync(0xffffffffu, pr[u], sub * W + jj);
                    if (j == 0 && t0 + W * u + jj < len) s = s - v;
                }
            }
        }
        if (j == 0 && valid) {
            const double r = MODE == 0 ? s : s / d;
            unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(r));
            if (bits == kXSentinel) bits = 0x7FFFFFFFFFFFFFFFull;
            st_relaxed_u64(x + row, bits);
        }
    }
}

// ---------------------------------------------------------------------------
// Cluster form of the value-flag schedule (small operators; ILUG_LEVELSET_DSM): the
// solution lives in the distributed shared memory of one thread-block
// cluster — row c in CTA c >> shift at c & (2^shift - 1) — and rows publish /
// poll their values there (a cross-CTA DSMEM round trip, ~215 cycles, instead
// of an L2 one). Rows are dealt round-robin in level order to the W-lane
// sub-groups of the cluster (each walks its rows in level order; all are
// co-resident), the next row's metadata and entries are loaded while the
// current one waits; products and the ordered shuffle chain are the sub-warp
// form's, so the result is bitwise the serial one.
namespace cg = cooperative_groups;
constexpr int kDsmBlock = 512;

__device__ __forceinline__ unsigned long long ld_dsm(const double* p) {
    return static_cast<unsigned long long>(*reinterpret_cast<const volatile long long*>(p));
}
__device__ __forceinline__ void st_dsm(double* p, unsigned long long v) {
    *reinterpret_cast<volatile long long*>(p) = static_cast<long long>(v);
}

template <int MODE, int W>
__global__ void __launch_bounds__(kDsmBlock, 1)
k_levels_dsm(SellView M, i64 n, int shift, const double* __restrict__ b, double* x, const double* __restrict__ xold) {
    constexpr int E = 4; // one pass: rows of up to W * 4 entries (the plan checks)
    extern __shared__ __align__(16) double sx[];
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank(), csize = cluster.num_blocks();
    const int chunk = 1 << shift;
    const unsigned cmask = static_cast<unsigned>(chunk - 1);
    for (int i = threadIdx.x; i < chunk; i += blockDim.x) reinterpret_cast<unsigned long long*>(sx)[i] = kXSentinel;
    cluster.sync();
    auto xptr = [&](i32 c) -> double* {
        return cluster.map_shared_rank(sx, static_cast<unsigned>(c) >> shift) + (static_cast<unsigned>(c) & cmask);
    };
    constexpr int RPG = 32 / W;
    const int lane = threadIdx.x & 31;
    const int sub = lane / W, j = lane % W;
    const i64 G = static_cast<i64>(csize) * (kDsmBlock / 32) * RPG;
    const i64 g0 = (static_cast<i64>(rank) * (kDsmBlock / 32) + (threadIdx.x >> 5)) * RPG + sub;
    const i64 npad = M.nrows_pad;
    const i64 rounds = (npad + G - 1) / G;
    struct Row {
        int len;
        i32 row;
        bool valid;
        i32 c[E];
        double a[E];
    };
    auto load = [&](i64 p, Row& r) {
        r.len = 0, r.row = 0, r.valid = false;
        i64 base = 0;
        if (p < npad) {
            const i32 rw = M.perm[p];
            if (rw >= 0) r.valid = true, r.row = rw, r.len = M.rowlen[p], base = M.slice_ptr[p >> 5] + (p & 31);
        }
#pragma unroll
        for (int u = 0; u < E; ++u) {
            const int t = j + W * u;
            if (t < r.len) {
                const i64 qq = base + static_cast<i64>(t) * kSlice;
                r.c[u] = __ldg(M.cols + qq);
                r.a[u] = __ldg(M.vals + qq);
            }
        }
    };
    Row cur, nxt;
    load(g0, cur);
    for (i64 k = 0; k < rounds; ++k) {
        load(g0 + (k + 1) * G, nxt);
        const int len = cur.len;
        const i32 row = cur.row;
        double s = j == 0 && cur.valid ? b[row] : 0.0, d = 1.0;
        int maxlen = len;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
        double pr[E];
        int kind[E];
        unsigned pend = 0;
#pragma unroll
        for (int u = 0; u < E; ++u) {
            const int t = j + W * u;
            kind[u] = 2;
            pr[u] = 0.0;
            if (t < len) {
                if (MODE != 0 && cur.c[u] == row) {
                    kind[u] = 1;
                } else if (is_dep<MODE>(cur.c[u], row)) {
                    const unsigned long long v = ld_dsm(xptr(cur.c[u]));
                    pr[u] = __longlong_as_double(static_cast<long long>(v));
                    kind[u] = 0;
                    if (v == kXSentinel) pend |= 1u << u;
                } else {
                    pr[u] = __ldg(xold + cur.c[u]); // GS (MODE 2) only
                    kind[u] = 0;
                }
            }
        }
        long long spins = 0;
        while (pend) {
            if (++spins > (1ll << 26)) {
                atomicExch(&g_levelset_timeout, 1u);
                break;
            }
#pragma unroll
            for (int u = 0; u < E; ++u)
                if ((pend >> u) & 1u) {
                    const unsigned long long v = ld_dsm(xptr(cur.c[u]));
                    if (v != kXSentinel) {
                        pr[u] = __longlong_as_double(static_cast<long long>(v));
                        pend &= ~(1u << u);
                    }
                }
        }
        bool has_d = false;
        double dl = 0.0;
#pragma unroll
        for (int u = 0; u < E; ++u) {
            if (MODE != 0 && kind[u] == 1) dl = cur.a[u], has_d = true;
            pr[u] = kind[u] == 0 ? cur.a[u] * pr[u] : 0.0;
        }
        if (MODE != 0) {
            const unsigned bal = __ballot_sync(0xffffffffu, has_d);
            const unsigned mine = (bal >> (sub * W)) & ((W == 32 ? 0u : (1u << W)) - 1u);
            const double dv = __shfl_sync(0xffffffffu, dl, sub * W + (mine ? __ffs(mine) - 1 : 0));
            if (mine) d = dv;
        }
        __syncwarp();
#pragma unroll
        for (int u = 0; u < E; ++u) {
            if (W * u >= maxlen) break;
#pragma unroll
            for (int jj = 0; jj < W; ++jj) {
                const double v = __shfl_sync(0xffffffffu, pr[u], sub * W + jj);
                if (j == 0 && W * u + jj < len) s = s - v;
            }
        }
        if (j == 0 && cur.valid) {
            const double r = MODE == 0 ? s : s / d;
            unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(r));
            if (bits == kXSentinel) bits = 0x7FFFFFFFFFFFFFFFull;
            st_dsm(xptr(row), bits);
        }
        cur = nxt;
    }
    cluster.sync();
    const i64 r0 = static_cast<i64>(rank) << shift;
    for (int i = threadIdx.x; i < chunk && r0 + i < n; i += blockDim.x) x[r0 + i] = sx[i];
}

template <int MODE>
const void* dsm_kernel(int max_row) {
    return max_row <= 32 ? reinterpret_cast<const void*>(k_levels_dsm<MODE, 8>)
                         : reinterpret_cast<const void*>(k_levels_dsm<MODE, 32>);
}
// ILUG_LEVELSET_DSM: unset = the cluster form for operators of up to 10 K rows
// (the small coarse levels, where it measured 5-45 % faster per GS sweep:
// C2 levels 4-8, C1 levels 3-6; wider levels need more than one cluster's SMs:
// C2 level 2 3.07 vs 2.0 ms; profiles/r02_gs_dsm3.txt); 1 = wherever it fits;
// 0 = never
int dsm_mode(i64 n) {
    const char* e = std::getenv("ILUG_LEVELSET_DSM");
    if (e && e[0] == '0') return 0;
    if (e && e[0] == '1') return 1;
    return n <= 10000 ? 1 : 0;
}

int vf_sub_override() { // ILUG_VF_SUB (A/B): 0 / 1 thread per row (16- / 8-entry chunks), 2 / 4 / 8 / 83 / 16 / 88 / 164 / 168 / 324 lanes (x entries)
    const char* e = std::getenv("ILUG_VF_SUB");
    return e ? std::atoi(e) : -1;
}
unsigned vf_sleep_ns() {
    const char* e = std::getenv("ILUG_VF_SLEEP");
    return e ? static_cast<unsigned>(std::atoi(e)) : 32u;
}
int vf_warps_per_sm() { // resident-warp cap of the sync-free grid (0: occupancy-limited)
    const char* e = std::getenv("ILUG_VF_WARPS");
    return e ? std::atoi(e) : 0;
}
template <int MODE>
const void* vsub_kernel(int w) {
    switch (w) {
    case 2: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 2>);
    case 8: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 8>);
    case 83: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 8, 3>); // 24 entries per pass
    case 16: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 16>);
    case 88: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 8, 8>);   // 64 entries per pass
    case 164: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 16, 4>); // 64
    case 168: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 16, 8>); // 128
    case 324: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 32, 4>); // 128
    default: return reinterpret_cast<const void*>(k_levels_vsub<MODE, 4>);
    }
}

// lanes per row of a sub-warp form code (0: a thread-per-row form)
int vsub_lanes(int w) {
    switch (w) {
    case 2: case 4: case 8: case 16: return w;
    case 83: case 88: return 8;
    case 164: case 168: return 16;
    case 324: return 32;
    default: return 0;
    }
}

__global__ void k_ticket_reset(unsigned* ticket) { *ticket = 0u; }

template <int MODE>
const void* vflag_kernel() {
    // ILUG_LEVELSET_HOIST=1: hoisted row metadata (A/B; bitwise the same). Off
    // by default: C2 direct solve 3.87/4.28 s hoisted vs 3.84/4.61 s without
    // in an interleaved A/B (no clear gain; the hoisted MODE 0 form spills
    // 32 B), unlike the sweep kernels where the hoist measured +2-9 %.
    const char* e = std::getenv("ILUG_LEVELSET_HOIST");
    if (e && e[0] == '1') return reinterpret_cast<const void*>(k_levels_vflags<MODE>);
    return reinterpret_cast<const void*>(k_levels_vflags<MODE, false>);
}

template <int MODE>
const void* cta_kernel() {
    return reinterpret_cast<const void*>(k_levels_cta<MODE>);
}
template <int MODE, int BLOCK = kWarpBlock, int Q = 1>
const void* warp_kernel() {
    return reinterpret_cast<const void*>(k_levels_warp<MODE, BLOCK, Q>);
}
template <int MODE>
const void* warp_kernel_sx() {
    return reinterpret_cast<const void*>(k_levels_warp<MODE, kWarpBlockWide, 1, true>);
}
template <int MODE>
const void* flag_kernel() {
    return reinterpret_cast<const void*>(k_levels_flags<MODE>);
}

} // namespace

namespace {

// Largest cluster of k_levels_warp CTAs (512 threads, one per SM) the device
// can co-schedule on one GPC.
i64 max_cluster_ctas() {
    static const i64 c = [] {
        const void* fns[] = {warp_kernel<0>(),       warp_kernel<1>(),       warp_kernel<2>(),
                             warp_kernel<0, kWarpBlockWide>(), warp_kernel<1, kWarpBlockWide>(),
                             warp_kernel<2, kWarpBlockWide>(), warp_kernel<0, kWarpBlock, 2>(),
                             warp_kernel<1, kWarpBlock, 2>(), warp_kernel<2, kWarpBlock, 2>()};
        for (const void* fn : fns)
            if (cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
                (void)cudaGetLastError();
        for (int want : {16, 8, 4, 2}) {
            bool ok = true;
            for (int f = 0; f < 9; ++f) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(static_cast<unsigned>(want));
                cfg.blockDim = dim3(f >= 3 && f < 6 ? kWarpBlockWide : kWarpBlock);
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = static_cast<unsigned>(want);
                attr[0].val.clusterDim.y = attr[0].val.clusterDim.z = 1;
                cfg.attrs = attr;
                cfg.numAttrs = 1;
                int nclusters = 0;
                if (cudaOccupancyMaxActiveClusters(&nclusters, fns[f], &cfg) != cudaSuccess || nclusters < 1) {
                    (void)cudaGetLastError();
                    ok = false;
                }
            }
            if (ok) return static_cast<i64>(want);
        }
        return i64{1};
    }();
    return c;
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
    sell_from_device_csr(M_, T, rp.p, ci.p, dev_vals ? dev_vals : v.p, Part::all, perm, st, false);

    // Level-synchronous on one cluster (warp per row) unless the levels
    // are wider than the cluster's warps can take in one pass on average (then
    // the sync-free flag schedule uses the whole GPU). Cluster size: enough
    // CTAs for the widest level's slices, capped by what one GPC co-schedules.
    const i64 cmax = max_cluster_ctas();
    const i64 avg = n / std::max(nl, 1);
    // value-flag form by row length and direction (tools/probe_spsv.cpp,
    // profiles/r02_k5_*.txt): short rows (7-point ILU(0), <= 8 entries) thread
    // per row — 8-entry chunks for L (C4: 12.3 ms vs 18.8 cuSPARSE), 16-entry
    // chunks for U; longer rows 8 lanes per row with one shuffle per entry slot
    // (C2 ILUT: L 4.6 ms, U 7.6 ms vs cuSPARSE 6.9 / 12.9) — 3 entries per lane
    // for L rows up to 24 entries, 4 otherwise
    i64 max_row = 0;
    for (i64 i = 0; i < n; ++i) max_row = std::max(max_row, T.rp[i + 1] - T.rp[i]);
    // rows longer than one 32-entry pass (coarse AMG operators: 36-115 entries
    // at C2) take every entry in ONE pass, or the next pass's values/columns
    // load only after the previous pass's dependencies arrived — a memory round
    // trip per pass on every level's critical path (C2 GS levels 2-6: 2.97 /
    // 2.29 / 1.48 / 0.68 / 0.22 -> 2.0 / 1.28 / 0.78 / 0.35 / 0.14 ms,
    // profiles/r02_gs_forms5.txt): 16 lanes x 8 entries where levels are wide
    // (> 200 rows on average: C2 levels 1-2), a whole warp x 4 entries (one row
    // per warp) where they are narrower (C1/C3 level 1, ~198 rows per level:
    // 0.55 vs 0.64 ms, profiles/r02_gs_forms_c1.txt)
    if (max_row <= 8)
        vf_form_ = kind == Kind::lower_unit ? 1 : 0;
    else if (max_row <= 32)
        vf_form_ = kind == Kind::lower_unit && max_row <= 24 ? 83 : 8;
    else
        vf_form_ = avg > 200 ? 168 : 324;
    // measured: the cluster kernel wins up to a few hundred rows per level
    // (coarse-level GS at 128^3: 258 rows/level 3.3 vs 4.6 ms), the value-flag
    // kernel beyond (ILUT factors at 128^3, 1564 rows/level: 4.9 vs 10.6 ms L)
    // with the sub-warp value-flag kernel the sync-free schedule wins on every
    // coarse AMG level's Gauss-Seidel, down to a 59-row operator (C2 levels 1-8:
    // 0.026-2.35 ms vs 0.031-13.6 ms per sweep; C1 levels 1-6 likewise,
    // profiles/r02_gs_forms4.txt); the cluster kernel keeps the short-row
    // (7-point ILU(0)) DAGs with narrow levels and the tiny ones
    single_cta_ = max_row <= 8 && (n <= 4 * kSmallBlock || avg <= 512);
    // wide levels (> 2 rows per warp of a 512-thread cluster): 1024-thread
    // CTAs. ILUG_LEVELSET_WIDE=slots2 takes 512-thread CTAs with two rows per
    // warp prefetched and processed together instead (measured slower at the
    // C2 level-1 GS: 33.5 vs 27.0 ms per presmooth — rows past the prefetched
    // slots serialise within the warp either way).
    slots_ = 1;
    block_ = avg > cmax * (kWarpBlock / 32) * 2 ? kWarpBlockWide : kWarpBlock;
    if (const char* w = std::getenv("ILUG_LEVELSET_WIDE"))
        if (std::string(w) == "slots2" && block_ == kWarpBlockWide) block_ = kWarpBlock, slots_ = 2;
    old_cta_ = false;
    if (const char* force = std::getenv("ILUG_LEVELSET")) { // test hook: cta | cta1 | flags
        if (std::string(force) == "cta" || std::string(force) == "cta1") single_cta_ = true;
        if (std::string(force) == "cta1") old_cta_ = true;
        if (std::string(force) == "flags" && n > 0) single_cta_ = false;
    }
    cluster_ = 1;
    if (nl > kMaxSmemLevels) old_cta_ = true; // level pointers do not fit the warp kernel's shared memory
    // shared-memory solution (one CTA): ILUG_LEVELSET=sx forces it where it fits (A/B)
    sx_ = false;
    if (const char* force = std::getenv("ILUG_LEVELSET"))
        if (std::string(force) == "sx" && n > 0 && n <= kSmemXRows && nl <= kMaxSmemLevels) single_cta_ = true, sx_ = true;
    if (single_cta_ && !old_cta_)
        cluster_ = static_cast<int>(
            std::clamp<i64>((max_level_rows_ + block_ / 32 * slots_ - 1) / (block_ / 32 * slots_), 1, cmax));
    value_flags_ = true;
    if (const char* force = std::getenv("ILUG_LEVELSET"))
        if (std::string(force) == "flags") value_flags_ = false; // the separate-flag form (A/B, tests)
    dsm_cs_ = 0;
    dsm_max_row_ = static_cast<int>(max_row);
    if (dsm_mode(n) && !single_cta_ && value_flags_ && n > 0 && max_row <= 128) {
        const int mode = kind == Kind::lower_unit ? 0 : (kind == Kind::upper ? 1 : 2);
        const void* fn = mode == 0 ? dsm_kernel<0>(dsm_max_row_) : mode == 1 ? dsm_kernel<1>(dsm_max_row_)
                                                                             : dsm_kernel<2>(dsm_max_row_);
        for (int cs : {8, 16}) {
            int shift = 0;
            while ((i64{1} << shift) * cs < n) ++shift;
            const int smem = static_cast<int>((i64{1} << shift) * static_cast<i64>(sizeof(double)));
            if (smem > 200 * 1024) continue;
            // the attribute is per kernel, shared by every plan: the largest size any plan uses
            if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess ||
                (cs > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)) {
                (void)cudaGetLastError();
                continue;
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<unsigned>(cs));
            cfg.blockDim = dim3(kDsmBlock);
            cfg.dynamicSmemBytes = static_cast<size_t>(smem);
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = static_cast<unsigned>(cs);
            at[0].val.clusterDim.y = at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nc = 0;
            if (cudaOccupancyMaxActiveClusters(&nc, fn, &cfg) == cudaSuccess && nc >= 1) {
                dsm_cs_ = cs, dsm_shift_ = shift, dsm_smem_ = smem;
                break;
            }
            (void)cudaGetLastError();
        }
    }
    if (const char* force = std::getenv("ILUG_LEVELSET"))
        if (std::string(force) == "vflags" && n > 0) single_cta_ = false;
    if (!single_cta_) {
        flags_.alloc(n + 3); // [0, n) row flags, n epoch, n+1 ticket, n+2 wait timeout
        ILUG_CUDA(cudaMemsetAsync(flags_.p, 0, static_cast<size_t>(n + 3) * sizeof(unsigned), st));
        const i64 slices = M_.nrows_pad / kSlice;
        grid_ = static_cast<int>(std::min<i64>((slices + kFlagBlock / 32 - 1) / (kFlagBlock / 32),
                                               static_cast<i64>(device_sm_count()) * 8));
    } else {
        grid_ = 1;
    }
    ILUG_CUDA(cudaStreamSynchronize(st));
}

void LevelPlan::refill(const i64* rp, const i32* ci, const double* v, cudaStream_t st) {
    sell_refill(M_, rp, ci, v, Part::all, st);
}

void LevelPlan::solve(const double* b, double* x, const double* xold, cudaStream_t st) const {
    if (M_.nrows == 0) return;
    SellView mv = view(M_);
    const int mode = kind_ == Kind::lower_unit ? 0 : (kind_ == Kind::upper ? 1 : 2);
    if (single_cta_) {
        const i64* lp = level_ptr_.p;
        int nl = nlev_;
        void* args[] = {&mv, &lp, &nl, &b, &x, &xold};
        if (old_cta_) { // the one-CTA register-pipelined kernel (A/B, tests)
            const void* fn = mode == 0 ? cta_kernel<0>() : mode == 1 ? cta_kernel<1>() : cta_kernel<2>();
            ILUG_CUDA(cudaLaunchKernel(fn, dim3(1), dim3(kSmallBlock), args, 0, st));
            return;
        }
        i64 nn = M_.nrows;
        void* wargs[] = {&mv, &lp, &nl, &b, &x, &xold, &nn};
        if (sx_) { // one CTA, the solution in shared memory
            const void* fn = mode == 0 ? warp_kernel_sx<0>() : mode == 1 ? warp_kernel_sx<1>() : warp_kernel_sx<2>();
            const int dyn = static_cast<int>(nn * static_cast<i64>(sizeof(double)));
            ILUG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
            ILUG_CUDA(cudaLaunchKernel(fn, dim3(1), dim3(kWarpBlockWide), wargs, static_cast<size_t>(dyn), st));
            return;
        }
        const bool wide = block_ == kWarpBlockWide, two = slots_ == 2;
        const void* fn =
            mode == 0   ? (wide ? warp_kernel<0, kWarpBlockWide>() : two ? warp_kernel<0, kWarpBlock, 2>() : warp_kernel<0>())
            : mode == 1 ? (wide ? warp_kernel<1, kWarpBlockWide>() : two ? warp_kernel<1, kWarpBlock, 2>() : warp_kernel<1>())
                        : (wide ? warp_kernel<2, kWarpBlockWide>() : two ? warp_kernel<2, kWarpBlock, 2>() : warp_kernel<2>());
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(cluster_));
        cfg.blockDim = dim3(static_cast<unsigned>(block_));
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(cluster_);
        attr[0].val.clusterDim.y = attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        ILUG_CUDA(cudaLaunchKernelExC(&cfg, fn, wargs));
        return;
    }
    const i64 n = M_.nrows;
    unsigned* flags = flags_.p;
    unsigned* epoch = flags_.p + n;
    unsigned* ticket = flags_.p + n + 1;
    i64 ns = M_.nrows_pad / kSlice;
    if (value_flags_ && x != b && x != xold) {
        if (dsm_cs_ > 0 && vf_sub_override() < 0) { // the cluster (DSMEM) form
            const void* fn = mode == 0 ? dsm_kernel<0>(dsm_max_row_) : mode == 1 ? dsm_kernel<1>(dsm_max_row_)
                                                                                 : dsm_kernel<2>(dsm_max_row_);
            i64 nn = n;
            int sh = dsm_shift_;
            void* dargs[] = {&mv, &nn, &sh, &b, &x, &xold};
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(static_cast<unsigned>(dsm_cs_));
            cfg.blockDim = dim3(kDsmBlock);
            cfg.dynamicSmemBytes = static_cast<size_t>(dsm_smem_);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = static_cast<unsigned>(dsm_cs_);
            at[0].val.clusterDim.y = at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            ILUG_CUDA(cudaLaunchKernelExC(&cfg, fn, dargs));
            return;
        }
        // the solution entries are the flags: fill x with the sentinel, reset the ticket
        k_fill_sentinel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(x, n);
        k_ticket_reset<<<1, 1, 0, st>>>(ticket);
        ILUG_LAUNCH_CHECK();
        const int ov = vf_sub_override();
        const int w = ov >= 0 ? ov : vf_form_;
        int grid = grid_;
        if (const int cap = vf_warps_per_sm(); cap > 0)
            grid = std::max(1, std::min(grid, device_sm_count() * cap / (kFlagBlock / 32)));
        if (const int lanes = vsub_lanes(w); lanes > 0) {
            i64 ng = ns * lanes;
            unsigned sl = vf_sleep_ns();
            void* args[] = {&mv, &ng, &b, &x, &xold, &ticket, &sl};
            const void* fn = mode == 0 ? vsub_kernel<0>(w) : mode == 1 ? vsub_kernel<1>(w) : vsub_kernel<2>(w);
            ILUG_CUDA(cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(kFlagBlock), args, 0, st));
            return;
        }
        void* args[] = {&mv, &ns, &b, &x, &xold, &ticket};
        const void* fn = w == 1 ? (mode == 0   ? reinterpret_cast<const void*>(k_levels_vflags<0, false, 8>)
                                   : mode == 1 ? reinterpret_cast<const void*>(k_levels_vflags<1, false, 8>)
                                               : reinterpret_cast<const void*>(k_levels_vflags<2, false, 8>))
                                : mode == 0 ? vflag_kernel<0>() : mode == 1 ? vflag_kernel<1>() : vflag_kernel<2>();
        ILUG_CUDA(cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid)), dim3(kFlagBlock), args, 0, st));
        return;
    }
    k_epoch_bump<<<1, 1, 0, st>>>(epoch, ticket);
    ILUG_LAUNCH_CHECK();
    const unsigned* ep = epoch;
    void* args[] = {&mv, &ns, &b, &x, &xold, &flags, &ep, &ticket};
    const void* fn = mode == 0 ? flag_kernel<0>() : mode == 1 ? flag_kernel<1>() : flag_kernel<2>();
    ILUG_CUDA(cudaLaunchKernel(fn, dim3(static_cast<unsigned>(grid_)), dim3(kFlagBlock), args, 0, st));
}

void levelset_check_error(cudaStream_t st) {
    ILUG_CUDA(cudaStreamSynchronize(st));
    unsigned v = 0;
    ILUG_CUDA(cudaMemcpyFromSymbol(&v, g_levelset_timeout, sizeof v));
    if (v) {
        const unsigned zero = 0;
        ILUG_CUDA(cudaMemcpyToSymbol(g_levelset_timeout, &zero, sizeof zero));
        fail_numeric("level-scheduled solve: a dependency wait timed out (scheduling fault); the result is invalid");
    }
}

} // namespace ilug
