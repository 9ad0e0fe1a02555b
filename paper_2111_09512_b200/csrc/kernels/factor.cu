// K1: scaling of the U factor on the device (north-star subsystem 1).
//
// Operates in place on the uploaded CSR of U (diagonal stored), one thread per
// row. Row scaling follows src/ilu.cpp:271-295 exactly (d = u_ii, diagonal set to
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

__global__ void k_diag(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                       const double* __restrict__ v, double* __restrict__ d,
                       unsigned long long* __restrict__ first_zero) {
    const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double di = 0.0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] == i) {
            di = v[k];
            break;
        }
    d[i] = di;
    if (di == 0.0) atomicMin(first_zero, static_cast<unsigned long long>(i));
}

__global__ void k_row_scale(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                            double* __restrict__ v, const double* __restrict__ d) {
    const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double inv = 1.0 / d[i];
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) v[k] = ci[k] == i ? 1.0 : v[k] * inv;
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
    const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const double ri = dr[i];
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
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
    // rs receives d = diag(U) first (row scaling stores it as row_scale as-is).
    const i64 bad = first_zero_row(n, rp, ci, v, rs, st);
    if (bad >= 0) return bad;
    const unsigned g = static_cast<unsigned>((n + kBlock - 1) / kBlock);
    if (n == 0) return -1;
    if (kind == 1) {
        k_row_scale<<<g, kBlock, 0, st>>>(n, rp, ci, v, rs);
        ILUG_LAUNCH_CHECK();
    } else {
        k_rowcol_factors<<<g, kBlock, 0, st>>>(n, rs, dr, dc, rs, cs);
        ILUG_LAUNCH_CHECK();
        k_rowcol_scale<<<g, kBlock, 0, st>>>(n, rp, ci, v, dr, dc);
        ILUG_LAUNCH_CHECK();
    }
    return -1;
}

} // namespace ilug
