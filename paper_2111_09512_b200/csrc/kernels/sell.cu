// SELL-32 construction and the thread-per-row product family (K2/K3/K6).
//
// One warp = one 32-row slice; lane l owns row 32*s + l and walks its entries
// t = 0..len-1 at slice_ptr[s] + 32*t + l. Loads of values/columns are streamed
// (L1 no-allocate, one 256 B / 128 B transaction per warp per t), the gathered
// x entries go through the read-only cache where stencil neighbours hit.
// Accumulation is ascending-column from 0.0 with separate multiply/add
// (--fmad=false): bitwise equal to src/sparse.cpp:162-174.
#include "ops.hpp"

#include <cub/cub.cuh>

#include <atomic>
#include <climits>
#include <cstring>
#include <vector>
#include <mutex>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace ilug {

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
    const std::string msg = std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                            cudaGetErrorString(e) + ") in " + what + " at " + file + ":" +
                            std::to_string(line);
    // Launch/argument errors are caller errors (2); faults and OOM are numeric (3).
    if (e == cudaErrorInvalidValue || e == cudaErrorInvalidConfiguration ||
        e == cudaErrorInvalidDevicePointer || e == cudaErrorNoDevice ||
        e == cudaErrorInsufficientDriver)
        fail_invalid(msg);
    fail_numeric(msg);
}

namespace {
std::atomic<int> g_defer{0};
std::mutex g_defer_mu;
std::vector<void*> g_deferred;
size_t g_deferred_bytes = 0;
// When to flush parked frees: only once memory is actually short (less than
// a quarter of the device free, checked after 16 GB are parked). A flush
// mid-setup costs up to a second (cudaFree of many large buffers holds the
// allocator, stalling every setup thread's cudaMalloc); dev_malloc still
// flushes and retries when an allocation runs out of memory.
bool defer_should_flush(size_t parked) {
    if (parked <= (size_t{16} << 30)) return false;
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
        (void)cudaGetLastError();
        return true;
    }
    return fr < tot / 4;
}
bool defer_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("ILUG_DEFER_FREE");
        return !(e && e[0] == '0');
    }();
    return on;
}
void free_all(std::vector<void*>& v) {
    for (void* q : v) cudaFree(q);
    v.clear();
}
} // namespace

void dev_free(void* p, size_t bytes) {
    if (g_defer.load(std::memory_order_acquire) > 0 && defer_enabled()) {
        std::vector<void*> flush;
        {
            std::lock_guard<std::mutex> g(g_defer_mu);
            g_deferred.push_back(p);
            g_deferred_bytes += bytes;
            if (defer_should_flush(g_deferred_bytes)) flush.swap(g_deferred), g_deferred_bytes = 0;
        }
        if (!flush.empty()) {
            SetupTimer tm("defer");
            free_all(flush);
            tm.mark("cap flush");
        }
        return;
    }
    cudaFree(p);
}
cudaError_t dev_malloc(void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaErrorMemoryAllocation) return e;
    (void)cudaGetLastError(); // clear the sticky-free error state of the failed call
    std::vector<void*> flush;
    {
        std::lock_guard<std::mutex> g(g_defer_mu);
        flush.swap(g_deferred);
        g_deferred_bytes = 0;
    }
    if (flush.empty()) return e;
    free_all(flush);
    return cudaMalloc(p, bytes);
}

DeferFrees::DeferFrees() { g_defer.fetch_add(1, std::memory_order_acq_rel); }
DeferFrees::~DeferFrees() {
    if (g_defer.fetch_sub(1, std::memory_order_acq_rel) != 1) return;
    std::vector<void*> flush;
    {
        std::lock_guard<std::mutex> g(g_defer_mu);
        flush.swap(g_deferred);
        g_deferred_bytes = 0;
    }
    free_all(flush);
}

int device_sm_count() {
    int dev = 0, n = 0;
    ILUG_CUDA(cudaGetDevice(&dev));
    ILUG_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    return n;
}

namespace {

constexpr int kBlock = 256;

inline unsigned grid_for(i64 threads, int block = kBlock) {
    return static_cast<unsigned>((threads + block - 1) / block);
}

// ---------------------------------------------------------------- SELL packing
__global__ void k_sell_fill(i64 nrows_pad, i64 nrows, const i32* __restrict__ perm, const i64* __restrict__ rp,
                            const i32* __restrict__ ci, const double* __restrict__ v, int part,
                            const i64* __restrict__ slice_ptr, i32* __restrict__ cols,
                            double* __restrict__ vals) {
    const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (p >= nrows_pad) return;
    const i64 row = perm ? perm[p] : p;
    if (row < 0 || row >= nrows) return;
    i64 dst = slice_ptr[p >> 5] + (p & 31);
    for (i64 k = rp[row]; k < rp[row + 1]; ++k) {
        const i32 j = ci[k];
        const bool keep = part == 0 || (part == 1 && j < row) || (part == 2 && j > row);
        if (!keep) continue;
        cols[dst] = j;
        vals[dst] = v[k];
        dst += kSlice;
    }
}

__global__ void k_sell_unpack(i64 nrows_pad, i64 nrows, const i32* __restrict__ perm,
                              const i64* __restrict__ slice_ptr,
                              const std::uint16_t* __restrict__ rowlen, const i32* __restrict__ cols,
                              const double* __restrict__ vals, const i64* __restrict__ out_rp,
                              i32* __restrict__ out_ci, double* __restrict__ out_v) {
    const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (p >= nrows_pad) return;
    const i64 row = perm ? perm[p] : p;
    if (row < 0 || row >= nrows) return;
    const i64 base = slice_ptr[p >> 5] + (p & 31);
    i64 o = out_rp[row];
    for (int t = 0; t < rowlen[p]; ++t, ++o) {
        out_ci[o] = cols[base + static_cast<i64>(t) * kSlice];
        out_v[o] = vals[base + static_cast<i64>(t) * kSlice];
    }
}

// ------------------------------------------------------------ row products
// Epilogues receive (row, s) with s the ascending-order row sum. pre(row)
// loads the row's vector operands. Read-modify-write epilogues (kEarly) have it
// called BEFORE the row loop, so the output's read overlaps the streamed and
// gathered loads instead of adding a dependent round trip at the end of every
// thread (measured: U sweep with accumulate 668 -> see profiles); for plain
// epilogues the early load measured slower (register pressure in the loop), so
// it stays after the loop. The arithmetic is the same either way.
struct None {};
struct EpiStore {
    static constexpr bool kEarly = false;
    double* y;
    __device__ None pre(i64) const { return {}; }
    __device__ void operator()(i64 r, double s, None) const { y[r] = s; }
};
struct EpiAdd {
    static constexpr bool kEarly = true;
    double* acc;
    __device__ double pre(i64 r) const { return acc[r]; }
    __device__ void operator()(i64 r, double s, double a) const { acc[r] = a + s; }
};
struct EpiResidual {
    static constexpr bool kEarly = false;
    const double* b;
    double* r;
    __device__ double pre(i64 i) const { return __ldg(b + i); }
    __device__ void operator()(i64 i, double s, double bi) const { r[i] = bi - s; }
};
struct EpiDiv {
    static constexpr bool kEarly = false;
    const double* rhs;
    const double* d;
    double* out;
    __device__ double2 pre(i64 i) const { return make_double2(__ldg(rhs + i), __ldg(d + i)); }
    __device__ void operator()(i64 i, double s, double2 p) const { out[i] = (p.x - s) / p.y; }
};
struct EpiBoth {
    static constexpr bool kEarly = false;
    const double* rhs;
    const double* d;
    double* out;
    double* out2;
    __device__ double2 pre(i64 i) const { return make_double2(__ldg(rhs + i), __ldg(d + i)); }
    __device__ void operator()(i64 i, double s, double2 p) const {
        const double t = p.x - s;
        out[i] = t;
        out2[i] = t / p.y;
    }
};
struct EpiAcc {
    static constexpr bool kEarly = true;
    const double* rhs;
    double* acc;
    __device__ double2 pre(i64 i) const { return make_double2(__ldg(rhs + i), acc[i]); }
    __device__ void operator()(i64 i, double s, double2 p) const { acc[i] = p.y + (p.x - s); }
};
struct Pre3 {
    double a, b, c;
};
struct EpiAccDiv {
    static constexpr bool kEarly = true;
    const double* rhs;
    const double* d;
    double* acc;
    __device__ Pre3 pre(i64 i) const { return {__ldg(rhs + i), __ldg(d + i), acc[i]}; }
    __device__ void operator()(i64 i, double s, Pre3 p) const { acc[i] = p.c + (p.a - s) / p.b; }
};
struct EpiScaleAcc { // jacobi_like_sweep out of place: out = x + invd * (b - Ax)
    static constexpr bool kEarly = false;
    const double* rhs;
    const double* sc;
    const double* xin;
    double* out;
    __device__ Pre3 pre(i64 i) const { return {__ldg(rhs + i), __ldg(sc + i), __ldg(xin + i)}; }
    __device__ void operator()(i64 i, double s, Pre3 p) const { out[i] = p.c + p.b * (p.a - s); }
};
struct EpiScaleInit { // poly_gs: term = invd * r; acc = term
    static constexpr bool kEarly = false;
    const double* rhs;
    const double* sc;
    double* term;
    double* acc;
    __device__ double2 pre(i64 i) const { return make_double2(__ldg(rhs + i), __ldg(sc + i)); }
    __device__ void operator()(i64 i, double s, double2 p) const {
        const double t = p.y * (p.x - s);
        term[i] = t;
        acc[i] = t;
    }
};
struct EpiNegScaleAcc { // poly_gs: term = -invd * t; acc += term
    static constexpr bool kEarly = true;
    const double* sc;
    double* term;
    double* acc;
    __device__ double2 pre(i64 i) const { return make_double2(__ldg(sc + i), acc[i]); }
    __device__ void operator()(i64 i, double s, double2 p) const {
        const double t = -p.x * s;
        term[i] = t;
        acc[i] = p.y + t;
    }
};

// Small operators (coarse AMG levels): a warp per row. A thread-per-row
// kernel on a level of a few thousand rows of 30-40 entries is pure latency —
// ~10 dependent batches per row, 23-33 us per launch whatever the size (ncu,
// C2 V-cycle: 135 such launches, 2.8 ms of 22.5 ms). Here lane t loads entry t
// and its x, forms the product a_t * x_t (the serial loop's rounded product),
// and the in-order sum s = 0 + p_0 + p_1 + ... runs as a shuffle chain, so the
// result is bitwise the thread-per-row kernel's. Lane 0 applies the epilogue.
template <class Epi, bool HOIST = true>
__global__ void __launch_bounds__(kBlock) k_rowdot_warp(SellView M, i64 nrows, const double* __restrict__ x,
                                                         Epi epi) {
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const i64 w0 = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) >> 5;
    const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
    for (i64 p = w0; p < M.nrows_pad; p += nw) {
        // HOIST: row metadata in the same round trip as perm (see k_rowdot)
        int len = HOIST ? M.rowlen[p] : 0;
        i64 base = HOIST ? M.slice_ptr[p >> 5] + (p & 31) : 0;
        i64 row = M.perm ? M.perm[p] : p;
        const bool valid = row >= 0 && row < nrows;
        if (!HOIST) {
            if (!valid) continue;
            len = M.rowlen[p];
            base = M.slice_ptr[p >> 5] + (p & 31);
        } else if (!valid) {
            len = 0, row = 0;
        }
        decltype(epi.pre(row)) pr{};
        if (lane == 0) pr = epi.pre(row);
        double s = 0.0;
        for (int t0 = 0; t0 < len; t0 += 32) {
            const int t = t0 + lane;
            double prod = 0.0;
            if (t < len) {
                const i64 q = base + static_cast<i64>(t) * kSlice;
                prod = ld_stream(M.vals + q) * ld_gather(x + ld_stream(M.cols + q));
            }
            const int cnt = min(32, len - t0);
            for (int u = 0; u < cnt; ++u) s = s + __shfl_sync(full, prod, u);
        }
        if (lane == 0 && valid) epi(row, s, pr);
    }
}
constexpr i64 kWarpRowMax = 65536; // operators up to this many rows take k_rowdot_warp

// Wider variant: eight entries per batch with predicated loads, so a row of up
// to eight entries (the L factor's 7.5 on average at C2) costs one streamed
// round trip plus one gather round trip.
template <class Epi>
__global__ void __launch_bounds__(kBlock) k_rowdot8(SellView M, i64 nrows, const double* __restrict__ x,
                                                     Epi epi) {
    const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (p >= M.nrows_pad) return;
    const i64 row = M.perm ? M.perm[p] : p;
    if (row < 0 || row >= nrows) return;
    decltype(epi.pre(row)) pr{};
    if constexpr (Epi::kEarly) pr = epi.pre(row); // issued before the row loop
    const int len = M.rowlen[p];
    const double* vp = M.vals + M.slice_ptr[p >> 5] + (p & 31);
    const int* cp = M.cols + M.slice_ptr[p >> 5] + (p & 31);
    double s = 0.0;
    for (int t = 0; t < len; t += 8) {
        double a[8], xv[8];
        int c[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (t + u < len) {
                a[u] = ld_stream(vp + (t + u) * kSlice);
                c[u] = ld_stream(cp + (t + u) * kSlice);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (t + u < len) xv[u] = ld_gather(x + c[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (t + u < len) s = s + a[u] * xv[u];
    }
    if constexpr (!Epi::kEarly) pr = epi.pre(row);
    epi(row, s, pr);
}

// Distributed form: columns < nloc gather from the local vector, columns >= nloc
// from the received halo buffer (halo exchange before the launch). The entry
// order is the global column order, so the sum is the single-process one.
template <class Epi>
__global__ void __launch_bounds__(kBlock) k_rowdot_split(SellView M, i64 nrows, const double* __restrict__ x,
                                                          const double* __restrict__ halo, i32 nloc, Epi epi) {
    const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (p >= M.nrows_pad) return;
    int len = M.rowlen[p]; // row metadata in the same round trip as perm (see k_rowdot HOIST)
    const i64 sp = M.slice_ptr[p >> 5];
    i64 row = M.perm ? M.perm[p] : p;
    const bool valid = row >= 0 && row < nrows;
    if (!valid) len = 0, row = 0;
    decltype(epi.pre(row)) pr{};
    if constexpr (Epi::kEarly) pr = epi.pre(row); // issued before the row loop
    const double* vp = M.vals + sp + (p & 31);
    const int* cp = M.cols + sp + (p & 31);
    double s = 0.0;
    int t = 0;
    for (; t + 4 <= len; t += 4) {
        double a[4], xv[4];
        int c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = ld_stream(vp + (t + u) * kSlice);
            c[u] = ld_stream(cp + (t + u) * kSlice);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = c[u] < nloc ? ld_gather(x + c[u]) : ld_gather(halo + (c[u] - nloc));
#pragma unroll
        for (int u = 0; u < 4; ++u) s = s + a[u] * xv[u];
    }
    for (; t < len; ++t) {
        const int c = ld_stream(cp + t * kSlice);
        s = s + ld_stream(vp + t * kSlice) * (c < nloc ? ld_gather(x + c) : ld_gather(halo + (c - nloc)));
    }
    if constexpr (!Epi::kEarly) pr = epi.pre(row);
    if (valid) epi(row, s, pr);
}

// HOIST: the row length and slice start (valid for every p < nrows_pad,
// padding slots included) are loaded together with perm[p]: a padding slot
// runs the row with len = 0 and skips the epilogue instead of exiting early,
// so there is no branch for the compiler to sink the loads past and the row's
// metadata costs one memory round trip instead of two (SASS without it:
// LDG perm -> EXIT -> LDG rowlen/slice_ptr).
// D8: the columns come from the dictionary-coded byte stream (Sell::codes),
// col = row + offtab[code] with the table in shared memory — 9 instead of 12
// streamed bytes per entry, the same entries in the same order (bitwise).
template <class Epi, bool HINT, bool PTAIL = true, bool HOIST = true, bool EARLY = Epi::kEarly, bool D8 = false>
__global__ void __launch_bounds__(kBlock) k_rowdot(SellView M, i64 nrows, const double* __restrict__ x,
                                                    Epi epi) {
    __shared__ i32 s_off[D8 ? kOffTab : 1];
    if constexpr (D8) {
        for (int i = threadIdx.x; i < kOffTab; i += blockDim.x) s_off[i] = __ldg(M.offtab + i);
        __syncthreads();
    }
    const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (p >= M.nrows_pad) return;
    int len = 0;
    i64 sp = 0;
    if constexpr (HOIST) {
        len = M.rowlen[p];
        sp = M.slice_ptr[p >> 5];
    }
    i64 row = M.perm ? M.perm[p] : p;
    const bool valid = row >= 0 && row < nrows;
    if constexpr (HOIST) {
        if (!valid) len = 0, row = 0;
    } else {
        if (!valid) return;
    }
    decltype(epi.pre(row)) pr{};
    if constexpr (EARLY) pr = epi.pre(row); // issued before the row loop
    if constexpr (!HOIST) {
        len = M.rowlen[p];
        sp = M.slice_ptr[p >> 5];
    }
    const double* vp = M.vals + sp + (p & 31);
    const int* cp = M.cols + sp + (p & 31);
    const std::uint8_t* dp = D8 ? M.codes + sp + (p & 31) : nullptr;
    const int r32 = static_cast<int>(row);
    unsigned long long pf = 0, pl = 0;
    if (HINT) pf = l2_policy_first(), pl = l2_policy_last();
    auto lv = [&](int t) { return HINT ? ld_stream(vp + t * kSlice, pf) : ld_stream(vp + t * kSlice); };
    auto lc = [&](int t) -> int {
        if constexpr (D8) return r32 + s_off[ld_stream(dp + t * kSlice)];
        else return HINT ? ld_stream(cp + t * kSlice, pf) : ld_stream(cp + t * kSlice);
    };
    auto lx = [&](int c) { return HINT ? ld_gather(x + c, pl) : ld_gather(x + c); };
    double s = 0.0;
    int t = 0;
    // Four entries in flight per lane: issue the streamed loads, then the
    // gathers, then accumulate in order (the order of the sum never changes).
    for (; t + 4 <= len; t += 4) {
        double a[4];
        int c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = lv(t + u);
            c[u] = lc(t + u);
        }
        double xv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) xv[u] = lx(c[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) s = s + a[u] * xv[u];
    }
    if constexpr (PTAIL) {
        // the last len % 4 entries as one predicated batch: their loads are in
        // flight together instead of one dependent round trip per entry
        if (t < len) {
            double a[3], xv[3];
            int c[3];
#pragma unroll
            for (int u = 0; u < 3; ++u)
                if (t + u < len) {
                    a[u] = lv(t + u);
                    c[u] = lc(t + u);
                }
#pragma unroll
            for (int u = 0; u < 3; ++u)
                if (t + u < len) xv[u] = lx(c[u]);
#pragma unroll
            for (int u = 0; u < 3; ++u)
                if (t + u < len) s = s + a[u] * xv[u];
        }
    } else {
        for (; t < len; ++t) s = s + lv(t) * lx(lc(t));
    }
    if constexpr (!EARLY) pr = epi.pre(row);
    if (valid) epi(row, s, pr);
}

// ---------------------------------------------------------------------------
// TMA-pipelined form (B200 bulk-copy engine): a persistent grid of 12 warps
// per SM; every warp owns a 2-stage shared-memory ring and works through the
// slices s = warp, warp + W, ... For the next slice, lane 0 arms an mbarrier
// and issues two cp.async.bulk copies (the slice's values and columns, one
// contiguous 32*width block each) while every lane prefetches its next row's
// metadata (perm, length) and epilogue operand; then the current slice is
// computed from shared memory: the only global loads left on the row's
// critical path are the x gathers. The sum order is unchanged (ascending t
// from 0.0), so the result is bitwise the plain kernel's.
constexpr int kTmaWarps = 12;
constexpr int kTmaWmax = 20; // widest slice the ring holds (C2 ILUT factors: 18)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

template <class Epi>
__global__ void __launch_bounds__(kTmaWarps * 32, 1) k_rowdot_tma(SellView M, i64 nrows, const double* __restrict__ x,
                                                                  Epi epi) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr unsigned VB = 32 * kTmaWmax * 8, CB = 32 * kTmaWmax * 4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* ring = smem + static_cast<size_t>(warp) * 2 * (VB + CB);
    unsigned long long* bar =
        reinterpret_cast<unsigned long long*>(smem + static_cast<size_t>(kTmaWarps) * 2 * (VB + CB)) + 2 * warp;
    if (lane == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const i64 ns = M.nrows_pad / kSlice;
    const i64 nw = static_cast<i64>(gridDim.x) * kTmaWarps;
    i64 s = static_cast<i64>(blockIdx.x) * kTmaWarps + warp;
    if (s >= ns) return;
    using Pre = decltype(epi.pre(i64{0}));
    // issue slice sl into stage stg: bulk copies + this lane's row metadata and epilogue operand
    auto issue = [&](i64 sl, int stg, int& len, i64& row, bool& valid, Pre& pre) {
        const i64 sp = M.slice_ptr[sl];
        const unsigned w = static_cast<unsigned>((M.slice_ptr[sl + 1] - sp) / kSlice);
        if (lane == 0 && w > 0) {
            unsigned char* vb = ring + stg * (VB + CB);
            mbar_expect_tx(&bar[stg], w * 32u * 12u);
            bulk_g2s(vb, M.vals + sp, w * 32u * 8u, &bar[stg]);
            bulk_g2s(vb + VB, M.cols + sp, w * 32u * 4u, &bar[stg]);
        }
        const i64 p = sl * kSlice + lane;
        len = M.rowlen[p];
        row = M.perm ? M.perm[p] : p;
        valid = row >= 0 && row < nrows;
        if (!valid) len = 0, row = 0;
        pre = epi.pre(row);
        return w;
    };
    int len, nlen = 0;
    i64 row, nrow = 0;
    bool valid, nvalid = false;
    Pre pre, npre{};
    unsigned w = issue(s, 0, len, row, valid, pre), nwid = 0;
    unsigned phase[2] = {0u, 0u};
    int stage = 0;
    while (s < ns) {
        const i64 sn = s + nw;
        if (sn < ns) nwid = issue(sn, stage ^ 1, nlen, nrow, nvalid, npre);
        if (w > 0) {
            mbar_wait(&bar[stage], phase[stage]);
            phase[stage] ^= 1u;
        }
        const double* sv = reinterpret_cast<const double*>(ring + stage * (VB + CB)) + lane;
        const int* sc = reinterpret_cast<const int*>(ring + stage * (VB + CB) + VB) + lane;
        double acc = 0.0;
        int t = 0;
        for (; t + 8 <= len; t += 8) {
            double xv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) xv[u] = ld_gather(x + sc[(t + u) * kSlice]);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc = acc + sv[(t + u) * kSlice] * xv[u];
        }
        if (t < len) {
            double xv[7];
#pragma unroll
            for (int u = 0; u < 7; ++u)
                if (t + u < len) xv[u] = ld_gather(x + sc[(t + u) * kSlice]);
#pragma unroll
            for (int u = 0; u < 7; ++u)
                if (t + u < len) acc = acc + sv[(t + u) * kSlice] * xv[u];
        }
        if (valid) epi(row, acc, pre);
        __syncwarp(); // every lane is done with this stage before it is refilled
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        s = sn;
        stage ^= 1;
        w = nwid, len = nlen, row = nrow, valid = nvalid, pre = npre;
    }
}

size_t rowdot_tma_smem() {
    return static_cast<size_t>(kTmaWarps) * 2 * (32 * kTmaWmax * 12) + kTmaWarps * 2 * sizeof(unsigned long long);
}
bool rowdot_tma() { // ILUG_ROWDOT_TMA=1: the bulk-copy pipelined sweep (A/B)
    const char* e = std::getenv("ILUG_ROWDOT_TMA");
    return e && e[0] == '1';
}

// Kernel variant knobs for A/B experiments (tools/probe_sweep.py):
// ILUG_L2_HINTS=1 enables the L2 eviction-priority hints (measured neutral on
// B200 at C2, so off by default); ILUG_ROWDOT=4|8 picks the batch width.
// Also measured and dropped (tools/probe_step.py, same-process A/B at C2):
// programmatic dependent launch with the first four values/columns of a row
// loaded before griddepcontrol.wait — U sweep 665 vs 608 us (the peeled head
// and the tighter register budget cost more than the tail overlap gains).
bool l2_hints() {
    const char* e = std::getenv("ILUG_L2_HINTS");
    return e && e[0] == '1';
}
bool serial_tail() { // ILUG_TAIL=serial: the row tail one entry at a time (A/B)
    const char* e = std::getenv("ILUG_TAIL");
    return e && e[0] == 's';
}
// Threads per CTA of the sweep kernel: 256. ILUG_ROWDOT_BLOCK=64|128 (A/B):
// 128-thread CTAs for the short-row L factor looked 3 % faster in one run but
// lost in an interleaved same-process A/B (L sweep 355-387 us at 256 vs
// 372-472 us at 128, tools/probe_sweep.py).
int rowdot_block(const Sell&) {
    if (const char* e = std::getenv("ILUG_ROWDOT_BLOCK")) {
        const int v = std::atoi(e);
        return v == 64 || v == 128 ? v : 256;
    }
    return 256;
}
bool warp_rows_enabled() { // ILUG_WARP_ROWS=0: small operators keep the thread-per-row kernel (A/B)
    const char* e = std::getenv("ILUG_WARP_ROWS");
    return !(e && e[0] == '0');
}
bool rowdot_early() { // ILUG_ROWDOT_EARLY=1: every epilogue's inputs loaded before the row loop (A/B)
    const char* e = std::getenv("ILUG_ROWDOT_EARLY");
    return e && e[0] == '1';
}
bool rowdot_late_acc() { // ILUG_ROWDOT_LATE_ACC=1: read-modify-write epilogues load after the row loop (A/B)
    const char* e = std::getenv("ILUG_ROWDOT_LATE_ACC");
    return e && e[0] == '1';
}
bool rowdot_hoist() { // ILUG_ROWDOT_HOIST=0: row metadata loaded after the padding check (A/B)
    const char* e = std::getenv("ILUG_ROWDOT_HOIST");
    return !(e && e[0] == '0');
}
int rowdot_width() { // measured at C2: width 4 beats 8 (64 regs halve occupancy)
    const char* e = std::getenv("ILUG_ROWDOT");
    return e && e[0] == '8' ? 8 : 4;
}

template <class Epi>
void launch_rowdot(const Sell& M, const double* x, Epi epi, cudaStream_t st) {
    if (M.nrows_pad == 0) return;
    if (rowdot_tma() && M.max_row <= kTmaWmax && M.nrows_pad > kWarpRowMax) {
        static bool attr = [] {
            ILUG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_rowdot_tma<Epi>),
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(rowdot_tma_smem())));
            return true;
        }();
        (void)attr;
        k_rowdot_tma<Epi><<<device_sm_count(), kTmaWarps * 32, rowdot_tma_smem(), st>>>(view(M), M.nrows, x, epi);
        ILUG_LAUNCH_CHECK();
        return;
    }
    if (M.nrows_pad <= kWarpRowMax && warp_rows_enabled()) {
        const i64 warps = M.nrows_pad;
        const unsigned g = static_cast<unsigned>(std::min<i64>((warps * 32 + kBlock - 1) / kBlock,
                                                               static_cast<i64>(device_sm_count()) * 8));
        if (rowdot_hoist())
            k_rowdot_warp<Epi><<<g, kBlock, 0, st>>>(view(M), M.nrows, x, epi);
        else
            k_rowdot_warp<Epi, false><<<g, kBlock, 0, st>>>(view(M), M.nrows, x, epi);
        ILUG_LAUNCH_CHECK();
        return;
    }
    if (rowdot_width() == 8)
        k_rowdot8<Epi><<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, x, epi);
    else if (l2_hints())
        k_rowdot<Epi, true><<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, x, epi);
    else if (serial_tail())
        k_rowdot<Epi, false, false><<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, x, epi);
    else if (rowdot_block(M) == 128)
        k_rowdot<Epi, false><<<grid_for(M.nrows_pad, 128), 128, 0, st>>>(view(M), M.nrows, x, epi);
    else if (rowdot_block(M) == 64)
        k_rowdot<Epi, false><<<grid_for(M.nrows_pad, 64), 64, 0, st>>>(view(M), M.nrows, x, epi);
    else if (rowdot_early())
        k_rowdot<Epi, false, true, true, true><<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, x, epi);
    else if (Epi::kEarly && rowdot_late_acc())
        k_rowdot<Epi, false, true, true, false><<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, x, epi);
    else if (!rowdot_hoist())
        k_rowdot<Epi, false, true, false><<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, x, epi);
    else if (M.codes.p)
        k_rowdot<Epi, false, true, true, Epi::kEarly, true>
            <<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, x, epi);
    else
        k_rowdot<Epi, false><<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, x, epi);
    ILUG_LAUNCH_CHECK();
}

} // namespace

// ------------------------------------------------------------ staged uploads
void h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    constexpr size_t kChunk = size_t{64} << 20;
    static std::mutex mu;
    static void* buf[2] = {nullptr, nullptr};
    static cudaEvent_t ev[2];
    static bool ok = false, tried = false;
    std::lock_guard<std::mutex> g(mu);
    if (!tried) {
        tried = true;
        ok = cudaHostAlloc(&buf[0], kChunk, cudaHostAllocDefault) == cudaSuccess &&
             cudaHostAlloc(&buf[1], kChunk, cudaHostAllocDefault) == cudaSuccess &&
             cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) (void)cudaGetLastError();
    }
    if (!ok) {
        ILUG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    const char* in = static_cast<const char*>(src);
    char* out = static_cast<char*>(dst);
    int k = 0;
    for (size_t off = 0; off < bytes; off += kChunk, k ^= 1) {
        const size_t len = std::min(kChunk, bytes - off);
        ILUG_CUDA(cudaEventSynchronize(ev[k])); // the DMA that last read buf[k] is done
        char* b = static_cast<char*>(buf[k]);
        constexpr i64 kPiece = i64{1} << 20;
        parallel_ranges((static_cast<i64>(len) + kPiece - 1) / kPiece, [&](i64 lo, i64 hi, int) {
            const size_t a = static_cast<size_t>(lo * kPiece), e = std::min(len, static_cast<size_t>(hi * kPiece));
            std::memcpy(b + a, in + off + a, e - a);
        }, 4);
        ILUG_CUDA(cudaMemcpyAsync(out + off, b, len, cudaMemcpyHostToDevice, s));
        ILUG_CUDA(cudaEventRecord(ev[k], s));
    }
}

void d2h_staged(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    constexpr size_t kChunk = size_t{64} << 20;
    static std::mutex mu;
    static void* buf[2] = {nullptr, nullptr};
    static cudaEvent_t ev[2];
    static bool ok = false, tried = false;
    std::lock_guard<std::mutex> g(mu);
    if (!tried) {
        tried = true;
        ok = cudaHostAlloc(&buf[0], kChunk, cudaHostAllocDefault) == cudaSuccess &&
             cudaHostAlloc(&buf[1], kChunk, cudaHostAllocDefault) == cudaSuccess &&
             cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) == cudaSuccess &&
             cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) == cudaSuccess;
        if (!ok) (void)cudaGetLastError();
    }
    if (!ok) {
        ILUG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        ILUG_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const char* in = static_cast<const char*>(src);
    char* out = static_cast<char*>(dst);
    const size_t nchunk = (bytes + kChunk - 1) / kChunk;
    // chunk c lands in buf[c & 1]; chunk c+1's DMA runs while chunk c is copied out
    auto issue = [&](size_t c) {
        const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
        ILUG_CUDA(cudaMemcpyAsync(buf[c & 1], in + off, len, cudaMemcpyDeviceToHost, s));
        ILUG_CUDA(cudaEventRecord(ev[c & 1], s));
    };
    issue(0);
    for (size_t c = 0; c < nchunk; ++c) {
        if (c + 1 < nchunk) issue(c + 1);
        ILUG_CUDA(cudaEventSynchronize(ev[c & 1]));
        const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
        const char* b = static_cast<const char*>(buf[c & 1]);
        constexpr i64 kPiece = i64{1} << 20;
        parallel_ranges((static_cast<i64>(len) + kPiece - 1) / kPiece, [&](i64 lo, i64 hi, int) {
            const size_t a = static_cast<size_t>(lo * kPiece), e = std::min(len, static_cast<size_t>(hi * kPiece));
            std::memcpy(out + off + a, b + a, e - a);
        }, 4);
    }
}

// --------------------------------------------------------------- builders
i64 sell_sigma() {
    const char* e = std::getenv("ILUG_SELL_SIGMA");
    return e ? std::max<i64>(1, std::atoll(e)) : i64{1024};
}

namespace {

// rowlen per SELL row and slice offsets; `len_of(row)` gives the part length.
template <typename LenOf>
void layout(Sell& out, i64 nrows_pad, const std::vector<i32>& perm, LenOf len_of, cudaStream_t st) {
    out.split_slices = -1;
    std::vector<std::uint16_t> rl(static_cast<size_t>(nrows_pad), 0);
    const i64 ns = nrows_pad / kSlice;
    std::vector<i64> sp(static_cast<size_t>(ns) + 1, 0);
    std::vector<i64> width(static_cast<size_t>(ns), 0);
    std::vector<i64> nnz_part(static_cast<size_t>(std::max<i64>(ns, 1)), 0);
    std::vector<int> mx(static_cast<size_t>(std::max<i64>(ns, 1)), 0);
    bool too_long = false;
    parallel_ranges(ns, [&](i64 b, i64 e, int) {
        for (i64 s = b; s < e; ++s) {
            i64 w = 0, tot = 0;
            for (i64 l = 0; l < kSlice; ++l) {
                const i64 p = s * kSlice + l;
                const i64 row = perm.empty() ? p : perm[p];
                const i64 len = (row < 0 || row >= out.nrows) ? 0 : len_of(row);
                if (len > 65535) too_long = true;
                rl[p] = static_cast<std::uint16_t>(len);
                w = std::max(w, len);
                tot += len;
            }
            width[s] = w;
            nnz_part[s] = tot;
            mx[s] = static_cast<int>(w);
        }
    });
    if (too_long) fail_invalid("SELL: a row has more than 65535 entries");
    for (i64 s = 0; s < ns; ++s) sp[s + 1] = sp[s] + width[s] * kSlice;
    out.nrows_pad = nrows_pad;
    out.padded = sp[ns];
    out.nnz = 0;
    out.max_row = 0;
    for (i64 s = 0; s < ns; ++s) out.nnz += nnz_part[s], out.max_row = std::max(out.max_row, mx[s]);
    // Everything on the builder's stream: the fill kernel that follows runs on
    // it, and a legacy-stream copy/memset is NOT ordered with a non-blocking
    // stream (a pageable-memory cudaMemcpyAsync may still be in flight when it
    // returns) — that race corrupted large operators built on a solver stream.
    out.slice_ptr.upload(sp.data(), ns + 1, st);
    out.rowlen.upload(rl.data(), nrows_pad, st);
    out.cols.alloc(out.padded);
    out.vals.alloc(out.padded);
    if (out.padded > 0) {
        ILUG_CUDA(cudaMemsetAsync(out.cols.p, 0, static_cast<size_t>(out.padded) * sizeof(i32), st));
        ILUG_CUDA(cudaMemsetAsync(out.vals.p, 0, static_cast<size_t>(out.padded) * sizeof(double), st));
    }
    if (!perm.empty())
        out.perm.upload(perm.data(), nrows_pad, st);
    else
        out.perm.release();
}

// ---- device-side SELL-C-sigma layout (the host `layout` + `sigma_order`
// without the host round trip: row lengths, the per-window stable sort by
// decreasing length, the >= 3 % padding rule, slice widths and offsets all on
// the GPU; the same permutation as the host path, so the same layout)
__global__ void k_len_rows(i64 n, const i64* __restrict__ rp, i64 skip, i32* __restrict__ len) {
    const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (i < n) len[i] = static_cast<i32>(rp[i + 1] - rp[i] - skip);
}
__global__ void k_len_part(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci, int pc,
                           i32* __restrict__ len) {
    const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    i32 c = 0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) c += pc == 1 ? ci[k] < i : ci[k] > i;
    len[i] = c;
}
__global__ void k_iota_i32(i64 n, i32* __restrict__ a) {
    const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (i < n) a[i] = static_cast<i32>(i);
}
__global__ void k_window_offsets(i64 nw, i64 sigma, i64 n, int* __restrict__ off) {
    const i64 w = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (w <= nw) off[w] = static_cast<int>(std::min(n, w * sigma));
}
// per slice: width (max length) of the natural and of the sorted order
__global__ void k_slice_widths(i64 ns, i64 n, const i32* __restrict__ len, const i32* __restrict__ slen,
                               i64* __restrict__ wnat, i64* __restrict__ wsort, i64* __restrict__ snnz) {
    const i64 s = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (s >= ns) return;
    i32 a = 0, b = 0;
    i64 t = 0;
    for (int l = 0; l < kSlice; ++l) {
        const i64 p = s * kSlice + l;
        if (p < n) a = max(a, len[p]), b = max(b, slen ? slen[p] : 0), t += len[p];
    }
    wnat[s] = a;
    if (wsort) wsort[s] = b;
    if (snnz) snnz[s] = t;
}
__global__ void k_layout_rows(i64 pad, i64 n, const i32* __restrict__ len, const i32* __restrict__ order,
                              i32* __restrict__ perm, std::uint16_t* __restrict__ rowlen) {
    const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (p >= pad) return;
    const i32 row = p < n ? (order ? order[p] : static_cast<i32>(p)) : -1;
    if (perm) perm[p] = row;
    rowlen[p] = static_cast<std::uint16_t>(row >= 0 ? len[row] : 0);
}
__global__ void k_slice_ptr_from_widths(i64 ns, const i64* __restrict__ w, i64* __restrict__ sp) {
    const i64 s = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (s < ns) sp[s + 1] = w[s] * kSlice;
    if (s == 0) sp[0] = 0;
}

template <class It, class Op>
i64 dev_reduce(It in, i64 n, Op op, i64 init, cudaStream_t st) {
    DBuf<i64> out(1);
    size_t tmp = 0;
    ILUG_CUDA(cub::DeviceReduce::Reduce(nullptr, tmp, in, out.p, static_cast<int>(n), op, init, st));
    DBuf<unsigned char> t(static_cast<i64>(tmp) + 1);
    ILUG_CUDA(cub::DeviceReduce::Reduce(t.p, tmp, in, out.p, static_cast<int>(n), op, init, st));
    i64 h = 0;
    ILUG_CUDA(cudaMemcpyAsync(&h, out.p, sizeof h, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    return h;
}
struct MaxI64 {
    __host__ __device__ i64 operator()(i64 a, i64 b) const { return a > b ? a : b; }
};
struct SumI64 {
    __host__ __device__ i64 operator()(i64 a, i64 b) const { return a + b; }
};

// len: the selected part's length of every row (device). Fills out's layout
// fields exactly as layout(sigma_order(...)) does on the host.
void layout_device(Sell& out, i64 n, const i32* len, cudaStream_t st) {
    out.split_slices = -1;
    const i64 pad = (n + kSlice - 1) / kSlice * kSlice;
    const i64 ns = pad / kSlice;
    DBuf<i64> wnat(std::max<i64>(ns, 1)), wsort;
    DBuf<i32> keys_out, order;
    const i64 sigma = sell_sigma();
    bool sorted = false;
    if (sigma > 1 && n >= 2 * kSlice) {
        const i64 nw = (n + sigma - 1) / sigma;
        DBuf<int> off(nw + 1);
        DBuf<i32> iota(n);
        keys_out.alloc(n);
        order.alloc(n);
        k_window_offsets<<<grid_for(nw + 1), kBlock, 0, st>>>(nw, sigma, n, off.p);
        k_iota_i32<<<grid_for(n), kBlock, 0, st>>>(n, iota.p);
        ILUG_LAUNCH_CHECK();
        size_t tmp = 0;
        ILUG_CUDA(cub::DeviceSegmentedSort::StableSortPairsDescending(
            nullptr, tmp, len, keys_out.p, iota.p, order.p, static_cast<int>(n), static_cast<int>(nw), off.p,
            off.p + 1, st));
        DBuf<unsigned char> t(static_cast<i64>(tmp) + 1);
        ILUG_CUDA(cub::DeviceSegmentedSort::StableSortPairsDescending(
            t.p, tmp, len, keys_out.p, iota.p, order.p, static_cast<int>(n), static_cast<int>(nw), off.p,
            off.p + 1, st));
        wsort.alloc(ns);
        k_slice_widths<<<grid_for(ns), kBlock, 0, st>>>(ns, n, len, keys_out.p, wnat.p, wsort.p, nullptr);
        ILUG_LAUNCH_CHECK();
        const i64 pn = dev_reduce(wnat.p, ns, SumI64{}, 0, st), ps = dev_reduce(wsort.p, ns, SumI64{}, 0, st);
        ILUG_CUDA(cudaStreamSynchronize(st)); // t, iota, off die here
        sorted = !(static_cast<double>(ps) > 0.97 * static_cast<double>(pn));
    }
    if (!sorted) {
        k_slice_widths<<<grid_for(std::max<i64>(ns, 1)), kBlock, 0, st>>>(ns, n, len, nullptr, wnat.p, nullptr,
                                                                           nullptr);
        ILUG_LAUNCH_CHECK();
    }
    const i64* w = sorted ? wsort.p : wnat.p;
    out.nrows_pad = pad;
    out.max_row = static_cast<int>(ns > 0 ? dev_reduce(w, ns, MaxI64{}, 0, st) : 0);
    if (out.max_row > 65535) fail_invalid("SELL: a row has more than 65535 entries");
    out.slice_ptr.alloc(ns + 1);
    k_slice_ptr_from_widths<<<grid_for(std::max<i64>(ns, 1)), kBlock, 0, st>>>(ns, w, out.slice_ptr.p);
    ILUG_LAUNCH_CHECK();
    if (ns > 0) {
        size_t tmp = 0;
        ILUG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, out.slice_ptr.p + 1, out.slice_ptr.p + 1,
                                                static_cast<int>(ns), st));
        DBuf<unsigned char> t(static_cast<i64>(tmp) + 1);
        ILUG_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, out.slice_ptr.p + 1, out.slice_ptr.p + 1,
                                                static_cast<int>(ns), st));
        ILUG_CUDA(cudaMemcpyAsync(&out.padded, out.slice_ptr.p + ns, sizeof(i64), cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
    } else {
        out.padded = 0;
    }
    out.rowlen.alloc(pad);
    if (sorted) out.perm.alloc(pad); else out.perm.release();
    if (pad > 0) {
        k_layout_rows<<<grid_for(pad), kBlock, 0, st>>>(pad, n, len, sorted ? order.p : nullptr,
                                                         sorted ? out.perm.p : nullptr, out.rowlen.p);
        ILUG_LAUNCH_CHECK();
    }
    if (ns > 0) { // stored entries: per-slice sums of the lengths, then one reduction
        DBuf<i64> snnz(ns);
        k_slice_widths<<<grid_for(ns), kBlock, 0, st>>>(ns, n, len, nullptr, wnat.p, nullptr, snnz.p);
        ILUG_LAUNCH_CHECK();
        out.nnz = dev_reduce(static_cast<const i64*>(snnz.p), ns, SumI64{}, 0, st);
    } else {
        out.nnz = 0;
    }
    out.cols.alloc(out.padded);
    out.vals.alloc(out.padded);
    if (out.padded > 0) {
        ILUG_CUDA(cudaMemsetAsync(out.cols.p, 0, static_cast<size_t>(out.padded) * sizeof(i32), st));
        ILUG_CUDA(cudaMemsetAsync(out.vals.p, 0, static_cast<size_t>(out.padded) * sizeof(double), st));
    }
}

i64 part_len(const Csr& A, i64 row, int pc) {
    if (pc == 0) return A.rp[row + 1] - A.rp[row];
    i64 c = 0;
    for (i64 k = A.rp[row]; k < A.rp[row + 1]; ++k) c += pc == 1 ? A.ci[k] < row : A.ci[k] > row;
    return c;
}

// SELL-C-sigma row order: within windows of sigma rows, rows sorted by
// decreasing length so each 32-row slice holds rows of similar length (less
// padding streamed). Returns an empty vector (natural order) when sorting would
// cut the padded size by less than 3 % — then the extra perm read is not worth it.
// sigma comes from ILUG_SELL_SIGMA (default 1024; 1 disables).
template <typename LenOf>
std::vector<i32> sigma_order(i64 n, LenOf len_of) {
    const i64 sigma = sell_sigma();
    if (sigma <= 1 || n < 2 * kSlice) return {};
    const i64 pad = (n + kSlice - 1) / kSlice * kSlice;
    std::vector<i32> len(static_cast<size_t>(n));
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) len[i] = static_cast<i32>(len_of(i));
    });
    std::vector<i32> perm(static_cast<size_t>(pad), -1);
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) perm[i] = static_cast<i32>(i);
    });
    const i64 wins = (n + sigma - 1) / sigma;
    parallel_ranges(wins, [&](i64 b, i64 e, int) {
        for (i64 w = b; w < e; ++w) {
            auto lo = perm.begin() + w * sigma, hi = perm.begin() + std::min(n, (w + 1) * sigma);
            std::stable_sort(lo, hi, [&](i32 a, i32 c) { return len[a] > len[c]; });
        }
    }, 1);
    auto padded = [&](bool sorted) {
        const i64 ns = pad / kSlice;
        const int T = host_threads();
        std::vector<i64> part(static_cast<size_t>(T) + 1, 0);
        parallel_ranges(ns, [&](i64 b, i64 e, int t) {
            i64 tot = 0;
            for (i64 s = b; s < e; ++s) {
                i32 w = 0;
                for (i64 l = 0; l < kSlice; ++l) {
                    const i64 p = s * kSlice + l;
                    if (p < n) w = std::max(w, len[sorted ? perm[p] : p]);
                }
                tot += w;
            }
            part[static_cast<size_t>(t)] += tot;
        });
        i64 tot = 0;
        for (i64 v : part) tot += v;
        return tot;
    };
    if (padded(true) > 0.97 * static_cast<double>(padded(false))) return {};
    return perm;
}

// ------------------------------------------------------- SELL-D8 coding
// Distinct column offsets c - row of a SELL matrix: each CTA gathers its rows'
// offsets into a shared-memory open-addressing set (plain reads first, CAS
// only on an empty slot, so the hot keys cost no atomics), then merges its
// keys into a global set; more than 255 distinct offsets anywhere leaves the
// matrix uncoded.
constexpr int kGSet = 1024, kCSet = 512;
constexpr i32 kNoKey = INT_MIN;
__device__ __forceinline__ unsigned off_hash(i32 v) { return (static_cast<unsigned>(v) * 2654435761u) >> 16; }

__global__ void k_fill_i32(i32* a, int n, i32 v) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) a[i] = v;
}

// insert v into set[cap] (probing); returns 1 if newly inserted, 0 if present, -1 if full
template <int CAP>
__device__ int set_insert(volatile i32* set, i32 v) {
    unsigned h = off_hash(v) & (CAP - 1);
    for (int probe = 0; probe < CAP; ++probe) {
        i32 cur = set[h];
        if (cur == v) return 0;
        if (cur == kNoKey) {
            cur = atomicCAS(const_cast<i32*>(set) + h, kNoKey, v);
            if (cur == kNoKey) return 1;
            if (cur == v) return 0;
        }
        h = (h + 1) & (CAP - 1);
    }
    return -1;
}

__global__ void k_offsets_collect(SellView M, i64 nrows, i32* gset, unsigned* gstat) {
    __shared__ i32 set[kCSet];
    __shared__ int full;
    for (int i = threadIdx.x; i < kCSet; i += blockDim.x) set[i] = kNoKey;
    if (threadIdx.x == 0) full = 0;
    __syncthreads();
    const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (p < M.nrows_pad) {
        const i64 row = M.perm ? M.perm[p] : p;
        if (row >= 0 && row < nrows) {
            const int len = M.rowlen[p];
            const i64 base = M.slice_ptr[p >> 5] + (p & 31);
            for (int t = 0; t < len && !full; ++t)
                if (set_insert<kCSet>(set, static_cast<i32>(M.cols[base + static_cast<i64>(t) * kSlice] - row)) < 0)
                    full = 1;
        }
    }
    __syncthreads();
    if (full) {
        if (threadIdx.x == 0) atomicOr(gstat + 1, 1u);
        return;
    }
    for (int i = threadIdx.x; i < kCSet; i += blockDim.x) {
        const i32 v = set[i];
        if (v == kNoKey) continue;
        const int r = set_insert<kGSet>(gset, v);
        if (r > 0) atomicAdd(gstat, 1u);
        if (r < 0) atomicOr(gstat + 1, 1u);
    }
}

__global__ void k_offsets_encode(SellView M, i64 nrows, const i32* __restrict__ tab, int ntab,
                                 std::uint8_t* __restrict__ codes) {
    __shared__ i32 t_s[kOffTab];
    for (int i = threadIdx.x; i < kOffTab; i += blockDim.x) t_s[i] = i < ntab ? tab[i] : INT_MAX;
    __syncthreads();
    const i64 p = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (p >= M.nrows_pad) return;
    const i64 row = M.perm ? M.perm[p] : p;
    if (row < 0 || row >= nrows) return;
    const int len = M.rowlen[p];
    const i64 base = M.slice_ptr[p >> 5] + (p & 31);
    for (int t = 0; t < len; ++t) {
        const i64 q = base + static_cast<i64>(t) * kSlice;
        const i32 off = static_cast<i32>(M.cols[q] - row);
        int lo = 0, hi = ntab - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (t_s[mid] < off)
                lo = mid + 1;
            else
                hi = mid;
        }
        codes[q] = static_cast<std::uint8_t>(lo);
    }
}

} // namespace

bool device_layout() { // ILUG_SELL_DEVICE_LAYOUT=0: the host layout path (A/B; read at every build)
    const char* e = std::getenv("ILUG_SELL_DEVICE_LAYOUT");
    return !(e && e[0] == '0');
}

bool sell_d8_enabled() { // ILUG_SELL_D8=0: int32 column stream only (A/B; read at every build)
    const char* e = std::getenv("ILUG_SELL_D8");
    return !(e && e[0] == '0');
}

void sell_encode(Sell& M, cudaStream_t st) {
    M.codes.release();
    M.offtab.release();
    if (!sell_d8_enabled() || M.nrows_pad == 0 || M.padded == 0 || M.nnz == 0) return;
    DBuf<i32> gset(kGSet);
    DBuf<unsigned> gstat(2);
    k_fill_i32<<<(kGSet + 255) / 256, 256, 0, st>>>(gset.p, kGSet, kNoKey);
    ILUG_CUDA(cudaMemsetAsync(gstat.p, 0, 2 * sizeof(unsigned), st));
    k_offsets_collect<<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, gset.p, gstat.p);
    ILUG_LAUNCH_CHECK();
    unsigned stat[2] = {0, 0};
    std::vector<i32> keys(kGSet);
    ILUG_CUDA(cudaMemcpyAsync(stat, gstat.p, sizeof stat, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaMemcpyAsync(keys.data(), gset.p, kGSet * sizeof(i32), cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    if (stat[1] || stat[0] == 0 || stat[0] >= static_cast<unsigned>(kOffTab)) return;
    std::vector<i32> tab;
    for (i32 k : keys)
        if (k != kNoKey) tab.push_back(k);
    std::sort(tab.begin(), tab.end());
    const int ntab = static_cast<int>(tab.size());
    tab.resize(kOffTab, 0);
    M.offtab.upload(tab.data(), kOffTab, st);
    M.codes.alloc(M.padded);
    ILUG_CUDA(cudaMemsetAsync(M.codes.p, 0, static_cast<size_t>(M.padded), st));
    k_offsets_encode<<<grid_for(M.nrows_pad), kBlock, 0, st>>>(view(M), M.nrows, M.offtab.p, ntab, M.codes.p);
    ILUG_LAUNCH_CHECK();
    ILUG_CUDA(cudaStreamSynchronize(st)); // the host table dies here
}

void sell_from_device_csr(Sell& out, const Csr& pattern, const i64* rp, const i32* ci,
                          const double* v, Part part, const std::vector<i32>& perm_in,
                          cudaStream_t s, bool encode) {
    out.nrows = pattern.nrows;
    out.ncols = pattern.ncols;
    const int pc = part == Part::all ? 0 : (part == Part::strict_lower ? 1 : 2);
    const std::vector<i32> perm_host =
        perm_in.empty() ? sigma_order(pattern.nrows, [&](i64 r) { return part_len(pattern, r, pc); })
                        : perm_in;
    const i64 pad = perm_host.empty() ? (pattern.nrows + kSlice - 1) / kSlice * kSlice
                                      : static_cast<i64>(perm_host.size());
    layout(out, pad, perm_host, [&](i64 row) { return part_len(pattern, row, pc); }, s);
    if (pad > 0 && pattern.nnz() > 0) {
        k_sell_fill<<<grid_for(pad), kBlock, 0, s>>>(pad, out.nrows, out.perm.p, rp, ci, v, pc,
                                                     out.slice_ptr.p, out.cols.p, out.vals.p);
        ILUG_LAUNCH_CHECK();
    }
    if (encode)
        sell_encode(out, s);
    else
        out.codes.release(), out.offtab.release();
}

void sell_from_device_rows(Sell& out, i64 nrows, i64 ncols, const RawVec<i64>& rp_host, i64 skip, const i64* rp,
                           const i32* ci, const double* v, Part part, cudaStream_t s) {
    SetupTimer tm("sell-dev");
    out.nrows = nrows;
    out.ncols = ncols;
    const int pc = part == Part::all ? 0 : (part == Part::strict_lower ? 1 : 2);
    i64 pad = 0;
    if (device_layout()) {
        DBuf<i32> len(std::max<i64>(nrows, 1));
        if (nrows > 0) {
            k_len_rows<<<grid_for(nrows), kBlock, 0, s>>>(nrows, rp, skip, len.p);
            ILUG_LAUNCH_CHECK();
        }
        layout_device(out, nrows, len.p, s);
        pad = out.nrows_pad;
        tm.mark("device layout");
    } else {
        auto len = [&](i64 r) { return rp_host[r + 1] - rp_host[r] - skip; };
        const std::vector<i32> perm = sigma_order(nrows, len);
        tm.mark("sigma order");
        pad = perm.empty() ? (nrows + kSlice - 1) / kSlice * kSlice : static_cast<i64>(perm.size());
        layout(out, pad, perm, len, s);
        tm.mark("layout+upload");
    }
    if (pad > 0 && rp_host[nrows] > 0) {
        k_sell_fill<<<grid_for(pad), kBlock, 0, s>>>(pad, out.nrows, out.perm.p, rp, ci, v, pc, out.slice_ptr.p,
                                                     out.cols.p, out.vals.p);
        ILUG_LAUNCH_CHECK();
    }
    sell_encode(out, s);
}

void sell_refill(Sell& M, const i64* rp, const i32* ci, const double* v, Part part, cudaStream_t s) {
    if (M.nrows_pad == 0 || M.padded == 0) return;
    const int pc = part == Part::all ? 0 : (part == Part::strict_lower ? 1 : 2);
    k_sell_fill<<<grid_for(M.nrows_pad), kBlock, 0, s>>>(M.nrows_pad, M.nrows, M.perm.p, rp, ci, v, pc,
                                                         M.slice_ptr.p, M.cols.p, M.vals.p);
    ILUG_LAUNCH_CHECK();
}

namespace {
void sell_host_build(Sell& out, const Csr& A, Part part, const std::vector<i32>* perm_in, cudaStream_t s);
void sell_device_build(Sell& out, i64 nrows, const i64* rp, const i32* ci, const double* v, int pc, cudaStream_t s,
                       SetupTimer& tm);
// rows sorted by decreasing length inside windows of sigma (stable), padded
// with -1 to whole slices: one group of a split SELL
void append_group(std::vector<i32>& perm, std::vector<i32>&& g, const Csr& A) {
    const i64 sigma = std::max<i64>(1, sell_sigma());
    const i64 m = static_cast<i64>(g.size());
    parallel_ranges((m + sigma - 1) / sigma, [&](i64 b, i64 e, int) {
        for (i64 w = b; w < e; ++w)
            std::stable_sort(g.begin() + w * sigma, g.begin() + std::min(m, (w + 1) * sigma),
                             [&](i32 a, i32 c) { return A.rp[a + 1] - A.rp[a] > A.rp[c + 1] - A.rp[c]; });
    }, 1);
    perm.insert(perm.end(), g.begin(), g.end());
    while (perm.size() % kSlice) perm.push_back(-1);
}
} // namespace

void sell_from_host_split(Sell& out, const Csr& A, i64 nloc, cudaStream_t s) {
    bool any_halo = false;
    std::vector<char> halo(static_cast<size_t>(A.nrows), 0);
    std::atomic<bool> seen{false};
    parallel_ranges(A.nrows, [&](i64 b, i64 e, int) {
        bool local_seen = false;
        for (i64 i = b; i < e; ++i) {
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k)
                if (A.ci[k] >= nloc) {
                    halo[static_cast<size_t>(i)] = 1;
                    local_seen = true;
                    break;
                }
        }
        if (local_seen) seen.store(true, std::memory_order_relaxed);
    });
    any_halo = seen.load();
    if (!any_halo) { // one rank / no halo: the plain layout (every row is local)
        sell_host_build(out, A, Part::all, nullptr, s);
        out.split_slices = out.nrows_pad / kSlice;
        return;
    }
    std::vector<i32> inner, outer;
    inner.reserve(static_cast<size_t>(A.nrows));
    for (i64 i = 0; i < A.nrows; ++i) (halo[static_cast<size_t>(i)] ? outer : inner).push_back(static_cast<i32>(i));
    std::vector<i32> perm;
    perm.reserve(static_cast<size_t>(A.nrows + 2 * kSlice));
    append_group(perm, std::move(inner), A);
    const i64 split = static_cast<i64>(perm.size()) / kSlice;
    append_group(perm, std::move(outer), A);
    sell_host_build(out, A, Part::all, &perm, s);
    out.split_slices = split;
}

void sell_from_host(Sell& out, const Csr& A, Part part, cudaStream_t s) { sell_host_build(out, A, part, nullptr, s); }

void sell_from_device(Sell& out, i64 nrows, i64 ncols, i64 nnz, const i64* rp, const i32* ci, const double* v,
                      cudaStream_t s, Part part) {
    if (!device_layout() || nnz == 0) { // the host layout (A/B knob) or nothing to lay out: via a host copy
        Csr h;
        h.nrows = nrows;
        h.ncols = ncols;
        h.rp.resize(static_cast<size_t>(nrows) + 1);
        h.ci.resize(static_cast<size_t>(nnz));
        h.v.resize(static_cast<size_t>(nnz));
        ILUG_CUDA(cudaMemcpyAsync(h.rp.data(), rp, sizeof(i64) * (nrows + 1), cudaMemcpyDeviceToHost, s));
        if (nnz > 0) {
            ILUG_CUDA(cudaMemcpyAsync(h.ci.data(), ci, sizeof(i32) * nnz, cudaMemcpyDeviceToHost, s));
            ILUG_CUDA(cudaMemcpyAsync(h.v.data(), v, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
        }
        ILUG_CUDA(cudaStreamSynchronize(s));
        return sell_from_host(out, h, part, s);
    }
    SetupTimer tm("sell-devcsr");
    out.nrows = nrows;
    out.ncols = ncols;
    out.split_slices = -1;
    sell_device_build(out, nrows, rp, ci, v, part == Part::all ? 0 : (part == Part::strict_lower ? 1 : 2), s, tm);
}

namespace {
// Layout on the GPU from a device CSR (nrows rows; out.nrows/ncols set by the caller).
void sell_device_build(Sell& out, i64 nrows, const i64* rp, const i32* ci, const double* v, int pc, cudaStream_t s,
                       SetupTimer& tm) {
    DBuf<i32> len(std::max<i64>(nrows, 1));
    if (pc == 0)
        k_len_rows<<<grid_for(nrows), kBlock, 0, s>>>(nrows, rp, 0, len.p);
    else
        k_len_part<<<grid_for(nrows), kBlock, 0, s>>>(nrows, rp, ci, pc, len.p);
    ILUG_LAUNCH_CHECK();
    layout_device(out, nrows, len.p, s);
    out.codes.release(), out.offtab.release();
    tm.mark("device layout");
    k_sell_fill<<<grid_for(out.nrows_pad), kBlock, 0, s>>>(out.nrows_pad, out.nrows, out.perm.p, rp, ci, v, pc,
                                                           out.slice_ptr.p, out.cols.p, out.vals.p);
    ILUG_LAUNCH_CHECK();
    sell_encode(out, s);
    ILUG_CUDA(cudaStreamSynchronize(s)); // the CSR (and temporaries) may die after this
    tm.mark("fill+encode");
}

void sell_host_build(Sell& out, const Csr& A, Part part, const std::vector<i32>* perm_in, cudaStream_t s) {
    SetupTimer tm("sell-host");
    out.nrows = A.nrows;
    out.ncols = A.ncols;
    out.split_slices = -1;
    const int pc = part == Part::all ? 0 : (part == Part::strict_lower ? 1 : 2);
    if (!perm_in && device_layout() && A.nnz() > 0) { // layout on the GPU from the uploaded CSR
        DBuf<i64> rp;
        DBuf<i32> ci;
        DBuf<double> v;
        rp.upload(A.rp.data(), A.nrows + 1, s);
        ci.upload(A.ci.data(), A.nnz(), s);
        v.upload(A.v.data(), A.nnz(), s);
        tm.mark("csr upload");
        sell_device_build(out, A.nrows, rp.p, ci.p, v.p, pc, s, tm);
        return;
    }
    const std::vector<i32> perm =
        perm_in ? *perm_in : sigma_order(A.nrows, [&](i64 r) { return part_len(A, r, pc); });
    tm.mark("sigma order");
    const i64 pad = perm.empty() ? (A.nrows + kSlice - 1) / kSlice * kSlice : static_cast<i64>(perm.size());
    layout(out, pad, perm, [&](i64 row) { return part_len(A, row, pc); }, s);
    tm.mark("layout+upload");
    out.codes.release(), out.offtab.release();
    if (A.nnz() == 0 || pad == 0) return;
    DBuf<i64> rp;
    DBuf<i32> ci;
    DBuf<double> v;
    rp.upload(A.rp.data(), A.nrows + 1, s);
    ci.upload(A.ci.data(), A.nnz(), s);
    v.upload(A.v.data(), A.nnz(), s);
    ILUG_CUDA(cudaStreamSynchronize(s));
    tm.mark("csr upload");
    k_sell_fill<<<grid_for(pad), kBlock, 0, s>>>(pad, out.nrows, out.perm.p, rp.p, ci.p, v.p, pc,
                                                 out.slice_ptr.p, out.cols.p, out.vals.p);
    ILUG_LAUNCH_CHECK();
    ILUG_CUDA(cudaStreamSynchronize(s)); // temporaries die at scope exit
    tm.mark("fill");
    sell_encode(out, s);
    tm.mark("encode");
}
} // namespace

Csr sell_to_host(const Sell& M) {
    ILUG_CUDA(cudaDeviceSynchronize()); // M may still be written on another stream
    Csr A;
    A.nrows = M.nrows;
    A.ncols = M.ncols;
    std::vector<std::uint16_t> rl(static_cast<size_t>(M.nrows_pad));
    std::vector<i32> perm(static_cast<size_t>(M.perm.n));
    M.rowlen.download(rl.data());
    if (M.perm.n) M.perm.download(perm.data());
    ILUG_CUDA(cudaDeviceSynchronize());
    A.rp.assign(static_cast<size_t>(M.nrows) + 1, 0);
    for (i64 p = 0; p < M.nrows_pad; ++p) {
        const i64 row = perm.empty() ? p : perm[p];
        if (row >= 0 && row < M.nrows) A.rp[row + 1] = rl[p];
    }
    for (i64 i = 0; i < M.nrows; ++i) A.rp[i + 1] += A.rp[i];
    A.ci.resize(static_cast<size_t>(A.rp[M.nrows]));
    A.v.resize(static_cast<size_t>(A.rp[M.nrows]));
    if (A.nnz() == 0) return A;
    DBuf<i64> rp;
    DBuf<i32> ci(A.nnz());
    DBuf<double> v(A.nnz());
    rp.upload(A.rp.data(), M.nrows + 1);
    k_sell_unpack<<<grid_for(M.nrows_pad), kBlock>>>(M.nrows_pad, M.nrows, M.perm.p, M.slice_ptr.p, M.rowlen.p,
                                                     M.cols.p, M.vals.p, rp.p, ci.p, v.p);
    ILUG_LAUNCH_CHECK();
    ci.download(A.ci.data());
    v.download(A.v.data());
    ILUG_CUDA(cudaDeviceSynchronize());
    return A;
}

// -------------------------------------------------------------- launchers
void spmv(const Sell& M, const double* x, double* y, cudaStream_t st) {
    launch_rowdot(M, x, EpiStore{y}, st);
}
namespace {
// slices [s0, s1) of M as a kernel view (row metadata offset; values/columns
// are addressed through slice_ptr, so they need no offset)
SellView view_range(const Sell& M, i64 s0, i64 s1) {
    SellView v = view(M);
    v.slice_ptr += s0;
    v.rowlen += s0 * kSlice;
    if (v.perm) v.perm += s0 * kSlice;
    v.nrows_pad = (s1 - s0) * kSlice;
    return v;
}
template <class Epi>
void launch_split(const Sell& M, const double* x, const double* halo, i64 nloc, Epi epi, cudaStream_t st,
                  const HaloWait* w) {
    const i64 ns = M.nrows_pad / kSlice;
    // local-only rows first when the halo is still in flight (split SELL)
    const i64 si = w && M.split_slices >= 0 && M.perm.p ? std::min(M.split_slices, ns) : 0;
    auto run = [&](i64 s0, i64 s1) {
        if (s1 <= s0) return;
        k_rowdot_split<Epi><<<grid_for((s1 - s0) * kSlice), kBlock, 0, st>>>(view_range(M, s0, s1), M.nrows, x, halo,
                                                                            static_cast<i32>(nloc), epi);
        ILUG_LAUNCH_CHECK();
    };
    run(0, si);
    if (w) (*w)(st);
    run(si, ns);
}
} // namespace
void residual_split(const Sell& M, const double* x, const double* halo, i64 nloc, const double* b, double* r,
                    cudaStream_t st, const HaloWait* w) {
    launch_split(M, x, halo, nloc, EpiResidual{b, r}, st, w);
}
void spmv_split(const Sell& M, const double* x, const double* halo, i64 nloc, double* y, cudaStream_t st,
                const HaloWait* w) {
    launch_split(M, x, halo, nloc, EpiStore{y}, st, w);
}
void spmv_add_split(const Sell& M, const double* x, const double* halo, i64 nloc, double* acc, cudaStream_t st,
                    const HaloWait* w) {
    launch_split(M, x, halo, nloc, EpiAdd{acc}, st, w);
}
void residual_scale_step_split(const Sell& M, const double* x, const double* halo, i64 nloc, const double* rhs,
                               const double* scale, double* out, cudaStream_t st, const HaloWait* w) {
    launch_split(M, x, halo, nloc, EpiScaleAcc{rhs, scale, x, out}, st, w);
}
void residual_scale_init_split(const Sell& M, const double* x, const double* halo, i64 nloc, const double* rhs,
                               const double* scale, double* term, double* acc, cudaStream_t st,
                               const HaloWait* w) {
    launch_split(M, x, halo, nloc, EpiScaleInit{rhs, scale, term, acc}, st, w);
}
void spmv_add(const Sell& M, const double* x, double* acc, cudaStream_t st) {
    launch_rowdot(M, x, EpiAdd{acc}, st);
}
void residual(const Sell& M, const double* x, const double* b, double* r, cudaStream_t st) {
    launch_rowdot(M, x, EpiResidual{b, r}, st);
}
void sweep_div(const Sell& M, const double* x, const double* rhs, const double* div, double* out,
               cudaStream_t st) {
    launch_rowdot(M, x, EpiDiv{rhs, div, out}, st);
}
void sweep_both(const Sell& M, const double* x, const double* rhs, const double* div, double* out,
                double* out2, cudaStream_t st) {
    launch_rowdot(M, x, EpiBoth{rhs, div, out, out2}, st);
}
void sweep_acc(const Sell& M, const double* x, const double* rhs, const double* div, double* acc,
               cudaStream_t st) {
    if (div)
        launch_rowdot(M, x, EpiAccDiv{rhs, div, acc}, st);
    else
        launch_rowdot(M, x, EpiAcc{rhs, acc}, st);
}
void residual_scale_step(const Sell& M, const double* x, const double* rhs, const double* scale,
                         double* out, cudaStream_t st) {
    launch_rowdot(M, x, EpiScaleAcc{rhs, scale, x, out}, st);
}
void residual_scale_init(const Sell& M, const double* x, const double* rhs, const double* scale,
                         double* term, double* acc, cudaStream_t st) {
    launch_rowdot(M, x, EpiScaleInit{rhs, scale, term, acc}, st);
}
void neg_scale_acc(const Sell& M, const double* x, const double* scale, double* term, double* acc,
                   cudaStream_t st) {
    launch_rowdot(M, x, EpiNegScaleAcc{scale, term, acc}, st);
}

} // namespace ilug
