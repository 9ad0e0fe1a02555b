// K1: scaling of the U factor on the device (north-star subsystem 1).
//
// Operates in place on the uploaded CSR of U (diagonal stored); rows are
// handled by 4-lane groups so the CSR arrays stream coalesced. Row scaling follows src/ilu.cpp:271-295 exactly (d = u_ii, diagonal set to
// 1.0, off-diagonals multiplied by the rounded reciprocal 1.0/d), row/column
// scaling src/ilu.cpp:297-333 (root = sqrt|d|, dr = sign/root, dc = 1/root,
// u_ij *= dr_i * dc_j): IEEE division and sqrt (nvcc defaults, -prec-div/-prec-sqrt)
// make both bitwise equal to the reference.
//
// Algorithmic bytes: 2*8*nnz(U) + 4*nnz(U) + 4(n+1) + 8n.
#include "ops.hpp"

namespace ilug {

namespace {

constexpr int kBlock = 256;

// Rows are handled by groups of kG lanes, each lane owning entries
// b + lane + kG*r (r < kR) of its row: the first kG*kR entries of a row are
// loaded with kR independent loads per lane before any is used (ILUT rows at
// C2 average 16.6), longer rows continue in a strided loop. Accesses stay in
// contiguous kG*8 B runs (one thread per row would touch 32 scattered sectors
// per warp access).
constexpr int kG = 4;
constexpr int kR = 4;

// Diagonal of row i: U's columns ascend and are >= i, so it is the first entry
// when stored; any other layout falls back to a scan (lane 0 of the group).
__device__ __forceinline__ double row_diag(i64 i, i64 b, i64 e, const i32* __restrict__ ci,
                                           const double* __restrict__ v) {
    if (b >= e) return 0.0;
    if (ci[b] == i) return v[b];
    for (i64 k = b + 1; k < e; ++k)
        if (ci[k] == i) return v[k];
    return 0.0;
}

__global__ void k_diag(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                       const double* __restrict__ v, double* __restrict__ d,
                       unsigned long long* __restrict__ first_zero) {
    const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double di = row_diag(i, rp[i], rp[i + 1], ci, v);
    d[i] = di;
    if (di == 0.0) atomicMin(first_zero, static_cast<unsigned long long>(i));
}

// Row scaling fused: d = u_ii -> rs, then u_ii = 1.0, u_ij *= 1.0/d.
__global__ void k_row_scale_fused(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                                  double* __restrict__ v, double* __restrict__ rs,
                                  unsigned long long* __restrict__ first_zero) {
    const i64 i = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) / kG;
    const int lane = threadIdx.x % kG;
    const bool active = i < n;
    i64 b = 0, e = 0;
    if (active) {
        b = rp[i];
        e = rp[i + 1];
    }
    int c[kR];
    double a[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const i64 k = b + lane + r * kG;
        c[r] = -1;
        a[r] = 0.0;
        if (k < e) {
            c[r] = ci[k];
            a[r] = v[k];
        }
    }
    // the diagonal is the row's first entry when stored (U: columns ascend, >= i)
    const int c0 = __shfl_sync(0xffffffffu, c[0], 0, kG);
    double di = __shfl_sync(0xffffffffu, a[0], 0, kG);
    if (!active) return;
    if (c0 != i) di = row_diag(i, b, e, ci, v); // other layouts: scan
    if (lane == 0) {
        rs[i] = di;
        if (di == 0.0) atomicMin(first_zero, static_cast<unsigned long long>(i));
    }
    const double inv = 1.0 / di;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const i64 k = b + lane + r * kG;
        if (k < e) v[k] = c[r] == i ? 1.0 : a[r] * inv;
    }
    for (i64 k = b + lane + kR * kG; k < e; k += kG) v[k] = ci[k] == i ? 1.0 : v[k] * inv;
}

// d and rs may alias (rs holds d on entry): read d before writing rs.
__global__ void k_rowcol_factors(i64 n, const double* d, double* __restrict__ dr,
                                 double* __restrict__ dc, double* rs, double* __restrict__ cs) {
    const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double di = d[i];
    const double root = sqrt(fabs(di));
    const double sign = di < 0.0 ? -1.0 : 1.0;
    dc[i] = 1.0 / root;
    dr[i] = sign / root;
    cs[i] = root;
    rs[i] = sign * root;
}

__global__ void k_rowcol_scale(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                               double* __restrict__ v, const double* __restrict__ dr,
                               const double* __restrict__ dc) {
    const i64 i = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) / kG;
    const int lane = threadIdx.x % kG;
    if (i >= n) return;
    const i64 b = rp[i], e = rp[i + 1];
    const double ri = dr[i];
    int c[kR];
    double a[kR], s[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const i64 k = b + lane + r * kG;
        c[r] = -1;
        a[r] = 0.0;
        s[r] = 0.0;
        if (k < e) {
            c[r] = ci[k];
            a[r] = v[k];
        }
    }
#pragma unroll
    for (int r = 0; r < kR; ++r)
        if (c[r] >= 0) s[r] = dc[c[r]];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const i64 k = b + lane + r * kG;
        if (k < e) v[k] = c[r] == i ? 1.0 : a[r] * (ri * s[r]);
    }
    for (i64 k = b + lane + kR * kG; k < e; k += kG) {
        const i32 j = ci[k];
        v[k] = j == i ? 1.0 : v[k] * (ri * dc[j]);
    }
}

i64 first_zero_row(i64 n, const i64* rp, const i32* ci, const double* v, double* d, cudaStream_t st) {
    DBuf<unsigned long long> fz(1);
    const unsigned long long init = ~0ull;
    ILUG_CUDA(cudaMemcpyAsync(fz.p, &init, sizeof init, cudaMemcpyHostToDevice, st));
    const unsigned g = static_cast<unsigned>((n + kBlock - 1) / kBlock);
    if (n > 0) {
        k_diag<<<g, kBlock, 0, st>>>(n, rp, ci, v, d, fz.p);
        ILUG_LAUNCH_CHECK();
    }
    unsigned long long h = 0;
    ILUG_CUDA(cudaMemcpyAsync(&h, fz.p, sizeof h, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    return h == ~0ull ? -1 : static_cast<i64>(h);
}

} // namespace

i64 extract_diag(i64 n, const i64* rp, const i32* ci, const double* v, double* d, cudaStream_t st) {
    return first_zero_row(n, rp, ci, v, d, st);
}

i64 scale_upper(i64 n, const i64* rp, const i32* ci, double* v, int kind, double* rs, double* cs,
                double* dr, double* dc, cudaStream_t st) {
    if (n == 0) return -1;
    const unsigned g = static_cast<unsigned>((n + kBlock - 1) / kBlock);
    const unsigned gg = static_cast<unsigned>((n * kG + kBlock - 1) / kBlock);
    if (kind == 1) {
        // one pass: rs = d = diag(U) (row_scale stores it as-is), then scale
        DBuf<unsigned long long> fz(1);
        const unsigned long long init = ~0ull;
        ILUG_CUDA(cudaMemcpyAsync(fz.p, &init, sizeof init, cudaMemcpyHostToDevice, st));
        k_row_scale_fused<<<gg, kBlock, 0, st>>>(n, rp, ci, v, rs, fz.p);
        ILUG_LAUNCH_CHECK();
        unsigned long long h = 0;
        ILUG_CUDA(cudaMemcpyAsync(&h, fz.p, sizeof h, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        return h == ~0ull ? -1 : static_cast<i64>(h);
    }
    // rs receives d = diag(U) first; every row's factors are needed before any
    // row is scaled (dc[j] of the columns)
    const i64 bad = first_zero_row(n, rp, ci, v, rs, st);
    if (bad >= 0) return bad;
    {
        k_rowcol_factors<<<g, kBlock, 0, st>>>(n, rs, dr, dc, rs, cs);
        ILUG_LAUNCH_CHECK();
        k_rowcol_scale<<<gg, kBlock, 0, st>>>(n, rp, ci, v, dr, dc);
        ILUG_LAUNCH_CHECK();
    }
    return -1;
}

} // namespace ilug
