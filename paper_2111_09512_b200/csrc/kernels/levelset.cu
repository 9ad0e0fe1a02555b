// K5: level-scheduled direct triangular solves and the Gauss-Seidel sweep —
// the "direct" comparison point of the paper and the reference's default
// coarse-level smoother (src/config.cpp:39).
//
// Host analysis buckets rows into wavefront levels of the dependency DAG and
// stores a level-ordered SELL-32 copy of the operator (each level padded to a
// whole number of slices, so a warp never straddles two levels). One persistent
// kernel walks the levels with a grid-wide barrier between them (cooperative
// launch guarantees co-residency; tiny systems use one CTA and __syncthreads).
// Each row is computed by one thread in the serial code's exact operation order
// (s = b; s -= a_ij x_j ascending; x_i = s / d), so the result is bitwise the
// sequential solve of src/trisolve.cpp:20-55 / src/smoother.cpp:113-132.
#include "levelset.hpp"

#include <algorithm>

namespace ilug {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ void grid_barrier(unsigned* count, unsigned* gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = *reinterpret_cast<volatile unsigned*>(gen);
        __threadfence();
        if (atomicAdd(count, 1u) == gridDim.x - 1) {
            atomicExch(count, 0u);
            __threadfence();
            atomicAdd(gen, 1u);
        } else {
            while (*reinterpret_cast<volatile unsigned*>(gen) == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}

// MODE 0: unit lower, strict storage: x_i = b_i - sum L_ij x_j
// MODE 1: upper with stored diagonal: x_i = (b_i - sum_{j != i} U_ij x_j) / U_ii
// MODE 2: Gauss-Seidel on A: x'_i = (b_i - sum_{j<i} a_ij x'_j - sum_{j>i} a_ij x_j) / a_ii
template <int MODE>
__global__ void __launch_bounds__(kBlock)
k_levels(SellView M, const i64* __restrict__ level_ptr, int nlev, const double* __restrict__ b,
         double* x, const double* __restrict__ xold, unsigned* bar) {
    const i64 nth = static_cast<i64>(gridDim.x) * blockDim.x;
    const i64 gt = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    for (int L = 0; L < nlev; ++L) {
        const i64 end = level_ptr[L + 1];
        for (i64 p = level_ptr[L] + gt; p < end; p += nth) {
            const i64 row = M.perm[p];
            if (row < 0) continue;
            const int len = M.rowlen[p];
            const i64 base = M.slice_ptr[p >> 5] + (p & 31);
            double s = b[row], d = 1.0;
            for (int t = 0; t < len; ++t) {
                const i64 q = base + static_cast<i64>(t) * kSlice;
                const i32 j = M.cols[q];
                const double a = M.vals[q];
                if (MODE == 0) {
                    s = s - a * __ldcg(x + j);
                } else if (j == row) {
                    d = a;
                } else if (MODE == 1 || j < row) {
                    s = s - a * __ldcg(x + j);
                } else {
                    s = s - a * xold[j];
                }
            }
            x[row] = MODE == 0 ? s : s / d;
        }
        if (L + 1 < nlev) {
            if (gridDim.x == 1)
                __syncthreads();
            else
                grid_barrier(bar, bar + 1);
        }
    }
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
    bar_.alloc(2);
    ILUG_CUDA(cudaMemsetAsync(bar_.p, 0, 2 * sizeof(unsigned), st));
    ILUG_CUDA(cudaStreamSynchronize(st));

    // Persistent grid: co-resident CTAs only (cooperative launch checks it).
    int per_sm = 0;
    switch (kind) {
    case Kind::lower_unit:
        ILUG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_levels<0>, kBlock, 0));
        break;
    case Kind::upper:
        ILUG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_levels<1>, kBlock, 0));
        break;
    case Kind::gauss_seidel:
        ILUG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_levels<2>, kBlock, 0));
        break;
    }
    const i64 want = (max_level_rows_ + kBlock - 1) / kBlock;
    const i64 cap = static_cast<i64>(std::max(1, per_sm)) * device_sm_count();
    grid_ = static_cast<int>(std::max<i64>(1, std::min(want, cap)));
    if (n <= 4 * kBlock * 8) grid_ = 1; // small systems: one CTA, block barriers only
}

void LevelPlan::solve(const double* b, double* x, const double* xold, cudaStream_t st) const {
    if (M_.nrows == 0) return;
    SellView mv = view(M_);
    const i64* lp = level_ptr_.p;
    int nl = nlev_;
    unsigned* bar = bar_.p;
    void* args[] = {&mv, &lp, &nl, &b, &x, &xold, &bar};
    const void* fn = kind_ == Kind::lower_unit ? reinterpret_cast<const void*>(k_levels<0>)
                     : kind_ == Kind::upper    ? reinterpret_cast<const void*>(k_levels<1>)
                                               : reinterpret_cast<const void*>(k_levels<2>);
    if (grid_ == 1) {
        ILUG_CUDA(cudaLaunchKernel(fn, dim3(1), dim3(kBlock), args, 0, st));
    } else {
        ILUG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(static_cast<unsigned>(grid_)), dim3(kBlock), args,
                                              0, st));
    }
}

} // namespace ilug
