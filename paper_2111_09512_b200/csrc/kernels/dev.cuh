// Device-side vocabulary shared by every kernel TU: error checks, owned
// device buffers, cache-hinted loads, and the SELL-32 matrix layout.
//
// Numerics contract: all kernels are compiled with --fmad=false, so a*b+c is a
// rounded multiply followed by a rounded add exactly like the reference's x86-64
// code (gcc -O2, no -march: no FMA). Thread-per-row kernels accumulate in
// ascending column order from 0.0, which makes SpMV, residual and every sweep
// bitwise identical to src/sparse.cpp:162-174 / src/trisolve.cpp:94-147.
#pragma once

#include "../host/common.hpp"

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace ilug {

[[noreturn]] void cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define ILUG_CUDA(call)                                                   \
    do {                                                                  \
        cudaError_t e__ = (call);                                         \
        if (e__ != cudaSuccess) ::ilug::cuda_fail(e__, #call, __FILE__, __LINE__); \
    } while (0)

#define ILUG_LAUNCH_CHECK() ILUG_CUDA(cudaGetLastError())

constexpr int kSlice = 32; // SELL slice height = warp width: one row per lane

/// Host -> device copy of a large pageable buffer through pinned staging
/// buffers filled by the host worker pool (the driver's own pageable path
/// stages single-threaded, ~5 GB/s). Returns once src is no longer needed.
void h2d_staged(void* dst, const void* src, size_t bytes, cudaStream_t s);
/// Device -> host counterpart (pageable destination): DMA into pinned chunks,
/// copied out by the worker pool. Synchronous with respect to the host.
void d2h_staged(void* dst, const void* src, size_t bytes, cudaStream_t s);
constexpr size_t kStagedMin = size_t{32} << 20; // smaller copies take the plain path

/// cudaFree synchronises the whole device, so a free on one setup thread waits
/// for every kernel in flight on the others (the AMG setup would wait for the
/// ILUT factorisation kernel). Inside a DeferFrees scope (any thread) frees are
/// parked and done when the last scope closes, or when the parked bytes pass a
/// cap (ILUG_DEFER_FREE=0 disables; A/B).
void dev_free(void* p, size_t bytes);
/// cudaMalloc that, on out-of-memory, frees the parked (deferred) buffers and
/// retries once before failing
cudaError_t dev_malloc(void** p, size_t bytes);
struct DeferFrees {
    DeferFrees();
    ~DeferFrees();
    DeferFrees(const DeferFrees&) = delete;
    DeferFrees& operator=(const DeferFrees&) = delete;
};

/// Owned device allocation (cudaMalloc / dev_free), move-only.
template <typename T>
struct DBuf {
    T* p = nullptr;
    i64 n = 0;
    DBuf() = default;
    explicit DBuf(i64 count) { alloc(count); }
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
    DBuf& operator=(DBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p, n = o.n;
            o.p = nullptr, o.n = 0;
        }
        return *this;
    }
    ~DBuf() { release(); }
    void alloc(i64 count) {
        release();
        n = count;
        if (count > 0) ILUG_CUDA(dev_malloc(reinterpret_cast<void**>(&p), static_cast<size_t>(count) * sizeof(T)));
    }
    void release() {
        if (p) dev_free(p, static_cast<size_t>(n) * sizeof(T));
        p = nullptr;
        n = 0;
    }
    void upload(const T* h, i64 count, cudaStream_t s = nullptr) {
        if (count != n) alloc(count);
        const size_t bytes = static_cast<size_t>(count) * sizeof(T);
        if (bytes >= kStagedMin)
            h2d_staged(p, h, bytes, s);
        else if (count > 0)
            ILUG_CUDA(cudaMemcpyAsync(p, h, bytes, cudaMemcpyHostToDevice, s));
    }
    void download(T* h, cudaStream_t s = nullptr) const {
        const size_t bytes = static_cast<size_t>(n) * sizeof(T);
        if (bytes >= kStagedMin)
            d2h_staged(h, p, bytes, s);
        else if (n > 0)
            ILUG_CUDA(cudaMemcpyAsync(h, p, bytes, cudaMemcpyDeviceToHost, s));
    }
    i64 bytes() const { return n * static_cast<i64>(sizeof(T)); }
};

/// SELL-32 ("sliced ELLPACK", slice height 32, sigma = 1 or level-sorted):
/// slice s stores its 32 rows column-major, entry t of lane l at
/// slice_ptr[s] + 32*t + l, so a warp's t-th loads of values and columns are
/// one fully coalesced 256 B / 128 B transaction. Per-row lengths predicate the
/// loop (padding is never multiplied, so Inf/NaN propagate exactly as in CSR).
/// Optional perm: SELL row p holds original row perm[p] (-1 = padding row);
/// used for level-ordered copies where each level starts on a slice boundary.
struct Sell {
    i64 nrows = 0;   ///< logical rows (original numbering)
    i64 ncols = 0;
    i64 nrows_pad = 0; ///< SELL rows (multiple of 32)
    i64 nnz = 0;     ///< stored (unpadded) entries
    i64 padded = 0;  ///< entries incl. padding
    int max_row = 0;
    DBuf<i64> slice_ptr; ///< nrows_pad/32 + 1
    DBuf<std::uint16_t> rowlen; ///< nrows_pad
    DBuf<i32> cols;
    DBuf<double> vals;
    DBuf<i32> perm; ///< empty = identity
    /// Dictionary-coded columns (SELL-D8): when a matrix has at most 255
    /// distinct column offsets c - row (stencil operators and their ILU
    /// factors: 27 / 30 / 84 at C2), codes[q] indexes offtab and the sweep
    /// kernels read 1 byte per entry instead of 4 (col = row + offtab[code]).
    /// cols stays for the other consumers. Empty = not coded.
    DBuf<std::uint8_t> codes;
    DBuf<i32> offtab; ///< kOffTab entries (unused slots 0)
    /// Distributed rows (sell_from_host_split): slices [0, split_slices) hold
    /// only rows whose columns are all local, the rest the rows that read the
    /// halo, so the local part runs while the halo is in flight. -1: unsplit.
    i64 split_slices = -1;
    bool empty() const { return nrows == 0; }
};
constexpr int kOffTab = 256;

/// Kernel-side view (trivially copyable).
struct SellView {
    const i64* __restrict__ slice_ptr;
    const std::uint16_t* __restrict__ rowlen;
    const i32* __restrict__ cols;
    const double* __restrict__ vals;
    const i32* __restrict__ perm;
    i64 nrows_pad;
    const std::uint8_t* __restrict__ codes;
    const i32* __restrict__ offtab;
};
inline SellView view(const Sell& s) {
    return {s.slice_ptr.p, s.rowlen.p, s.cols.p, s.vals.p, s.perm.p, s.nrows_pad, s.codes.p, s.offtab.p};
}

int device_sm_count();

} // namespace ilug

#ifdef __CUDACC__
namespace ilug {
// Streaming (read-once) loads: bypass L1 allocation, keep L2 behaviour default.
__device__ __forceinline__ double ld_stream(const double* p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_stream(const int* p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned ld_stream(const std::uint8_t* p) {
    unsigned v;
    asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// Gathered vector entries: read-only path, cached (stencil reuse across rows).
__device__ __forceinline__ double ld_gather(const double* p) { return __ldg(p); }

// L2 eviction-priority variants: the streamed operator is marked evict_first so
// it does not push the gathered vector (reused by up to ~27 rows, one z-plane
// apart) out of L2; the gathered vector is marked evict_last.
__device__ __forceinline__ unsigned long long l2_policy_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_policy_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_stream(const double* p, unsigned long long pol) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ld_stream(const int* p, unsigned long long pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_gather(const double* p, unsigned long long pol) {
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
// Dependency flags (epoch-stamped, written with a release store by the
// producer). An acquire load is LD.STRONG.GPU + CCTL.IVALL (it drops the whole
// SM's L1), so spinning on acquire loads spends most of the wait invalidating
// L1 for every warp on the SM (ncu: 70 % of the device ILUT's stall samples).
// Wait instead with relaxed polls and one acquire load once the flag is seen.
// Returns false when the bounded spin runs out (a scheduling bug, not a slow
// producer: seconds of waiting).
__device__ __forceinline__ unsigned ld_relaxed_flag(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_flag(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <int SLEEP_NS = 32>
__device__ __forceinline__ bool wait_flag(const unsigned* p, unsigned E) {
    if (ld_acquire_flag(p) == E) return true;
    long long spins = 0;
    while (ld_relaxed_flag(p) != E) {
        if (++spins > (1ll << 26)) return false;
        __nanosleep(SLEEP_NS);
    }
    (void)ld_acquire_flag(p); // synchronises with the producer's release store
    return true;
}
} // namespace ilug
#endif
