// BLAS-1 building blocks and the CGS2 orthogonalisation kernels (K8), plus
// the coarse dense LU solve (K7).
//
// Reductions are deterministic: a fixed tiling (1024 rows per block), a fixed
// in-block order (per-thread sequential, then warp shuffles, then warps in
// order) and a single-block final pass over the per-block partials in order.
// Repeated runs are bitwise identical; against the reference's sequential dot
// (src/krylov.cpp:38-42) they differ only by summation order.
#include "ops.hpp"

namespace ilug {

namespace {

constexpr int kBlock = 256;
constexpr int kRows = 4;                 // rows per thread in the tiled reductions
constexpr int kTile = kBlock * kRows;    // rows per block
constexpr int kMaxVec = 64;              // dot outputs per pass of the fused CGS2 kernels

inline unsigned ew_grid(i64 n) {
    const i64 g = (n + kBlock - 1) / kBlock;
    return static_cast<unsigned>(std::max<i64>(1, std::min<i64>(g, 148 * 64)));
}

__global__ void k_div(double* __restrict__ o, const double* __restrict__ a, const double* __restrict__ d,
                      i64 n) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        o[i] = a[i] / d[i];
}
__global__ void k_acc(double* __restrict__ x, const double* __restrict__ z, i64 n) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        x[i] = x[i] + z[i];
}
__global__ void k_acc_div(double* __restrict__ x, const double* __restrict__ z,
                          const double* __restrict__ d, i64 n) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        x[i] = x[i] + z[i] / d[i];
}
__global__ void k_scale_div(double* o, const double* w, double h, i64 n) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        o[i] = w[i] / h;
}
// out = w / *h, skipped when *h == 0 (GMRES happy breakdown leaves v_{j+1} unset)
__global__ void k_scale_div_dev(double* o, const double* w, const double* h, i64 n) {
    const double hv = *h;
    if (hv == 0.0) return;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        o[i] = w[i] / hv;
}
__global__ void k_sub_into(double* __restrict__ o, const double* __restrict__ a,
                           const double* __restrict__ b, i64 n) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        o[i] = a[i] - b[i];
}
__global__ void k_add_into(double* __restrict__ o, const double* __restrict__ a,
                           const double* __restrict__ b, i64 n) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        o[i] = a[i] + b[i];
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;
}

// Sum `per` values of thread-local partials for k outputs over the block:
// red[w][j] per warp, then warps summed in order by thread j. Any k: the
// outputs are produced in chunks of kMaxVec (the per-row axpy of MODE 3/4
// always covers all k vectors before any dot is taken, so chunking the
// outputs does not change a bit); partials are written with stride pstride.
template <int MODE>
__global__ void __launch_bounds__(kBlock)
k_tiled(const double* __restrict__ V, i64 ld, int k, const double* __restrict__ hin,
        double* __restrict__ w, const double* __restrict__ w2, i64 n, double* __restrict__ partial,
        i64 pstride) {
    // MODE 0: dot(w, w2) -> 1 output; MODE 1: ||w||^2; MODE 2: V^T w (k outputs);
    // MODE 3: w -= V hin, then V^T w; MODE 4: w -= V hin, then ||w||^2;
    // MODE 5: sum_i (w_i - h v_i)^2 with h = hin[0], v = w2 (Schur h21^2).
    __shared__ double red[kBlock / 32][kMaxVec];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const i64 base = blockIdx.x * static_cast<i64>(kTile) + threadIdx.x;
    double wv[kRows];
#pragma unroll
    for (int u = 0; u < kRows; ++u) {
        const i64 i = base + u * kBlock;
        wv[u] = i < n ? w[i] : 0.0;
    }
    if (MODE == 3 || MODE == 4) {
        for (int j = 0; j < k; ++j) {
            const double hj = __ldg(hin + j); // uniform address: one broadcast per warp
#pragma unroll
            for (int u = 0; u < kRows; ++u) {
                const i64 i = base + u * kBlock;
                if (i < n) wv[u] = wv[u] - hj * V[j * ld + i];
            }
        }
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
            const i64 i = base + u * kBlock;
            if (i < n) w[i] = wv[u];
        }
    }
    if constexpr (MODE == 0 || MODE == 1 || MODE == 4 || MODE == 5) {
        double s = 0.0;
        const double h = MODE == 5 ? hin[0] : 0.0;
#pragma unroll
        for (int u = 0; u < kRows; ++u) {
            const i64 i = base + u * kBlock;
            if (MODE == 5) {
                const double dv = i < n ? wv[u] - h * w2[i] : 0.0;
                s += dv * dv;
                continue;
            }
            const double o = MODE == 0 ? (i < n ? w2[i] : 0.0) : wv[u];
            s += wv[u] * o;
        }
        s = warp_sum(s);
        if (lane == 0) red[warp][0] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < kBlock / 32; ++q) t += red[q][0];
            partial[blockIdx.x * pstride] = t;
        }
    } else {
    for (int j0 = 0; j0 < k; j0 += kMaxVec) {
        const int kc = min(kMaxVec, k - j0);
        for (int j = 0; j < kc; ++j) {
            double s = 0.0;
#pragma unroll
            for (int u = 0; u < kRows; ++u) {
                const i64 i = base + u * kBlock;
                if (i < n) s += V[(j0 + j) * ld + i] * wv[u];
            }
            s = warp_sum(s);
            if (lane == 0) red[warp][j] = s;
        }
        __syncthreads();
        for (int j = threadIdx.x; j < kc; j += blockDim.x) {
            double s = 0.0;
            for (int q = 0; q < kBlock / 32; ++q) s += red[q][j];
            partial[blockIdx.x * pstride + j0 + j] = s;
        }
        __syncthreads();
    }
    }
}

// out[j] = sum over blocks b (in order, tree within one block) of partial[b][j]
__global__ void k_finish(const double* __restrict__ partial, i64 nblocks, int nout, i64 pstride,
                         double* __restrict__ out) {
    __shared__ double sm[kBlock];
    for (int j = 0; j < nout; ++j) {
        double s = 0.0;
        for (i64 b = threadIdx.x; b < nblocks; b += blockDim.x) s += partial[b * pstride + j];
        sm[threadIdx.x] = s;
        __syncthreads();
        for (int o = kBlock / 2; o > 0; o >>= 1) {
            if (threadIdx.x < o) sm[threadIdx.x] += sm[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) out[j] = sm[0];
        __syncthreads();
    }
}

// y = base + sum_j c_j V_j, any k (c read through the uniform-address path)
__global__ void k_combine(const double* __restrict__ V, i64 ld, int k, const double* __restrict__ c,
                          const double* __restrict__ base, double* __restrict__ y, i64 n) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x) {
        double s = base ? base[i] : 0.0;
        for (int j = 0; j < k; ++j) s = s + __ldg(c + j) * V[j * ld + i];
        y[i] = s;
    }
}

// Two-stage reductions write their per-block partials into caller-owned
// workspace (reduce_ws_doubles(n) doubles): no hidden state, graph-capturable,
// and concurrent solves on different streams never share scratch.
template <int MODE>
void tiled(const double* V, i64 ld, int k, const double* hin, double* w, const double* w2, i64 n,
           double* out, int nout, double* ws, cudaStream_t st) {
    if (!ws) fail_invalid("reduction: no workspace");
    const i64 nb = std::max<i64>(1, (n + kTile - 1) / kTile);
    const i64 pstride = std::max<i64>(kMaxVec, nout); // reduce_ws_doubles(n, k) covers nb * pstride
    k_tiled<MODE><<<static_cast<unsigned>(nb), kBlock, 0, st>>>(V, ld, k, hin, w, w2, n, ws, pstride);
    ILUG_LAUNCH_CHECK();
    k_finish<<<1, kBlock, 0, st>>>(ws, nb, nout, pstride, out);
    ILUG_LAUNCH_CHECK();
}

// K7: x = LU \ P b (src/dense.cpp:40-55). Forward elimination is parallel over
// rows i > k (each x_i still receives its updates in ascending k); back
// substitution runs on one thread to keep the reference's summation order.
__global__ void k_dense_solve(i64 n, const double* __restrict__ lu, const i64* __restrict__ piv,
                              const double* __restrict__ b, double* __restrict__ x) {
    for (i64 i = threadIdx.x; i < n; i += blockDim.x) x[i] = b[i];
    __syncthreads();
    for (i64 k = 0; k < n; ++k) {
        if (threadIdx.x == 0 && piv[k] != k) {
            const double t = x[piv[k]];
            x[piv[k]] = x[k];
            x[k] = t;
        }
        __syncthreads();
        const double xk = x[k];
        for (i64 i = k + 1 + threadIdx.x; i < n; i += blockDim.x) x[i] = x[i] - lu[i * n + k] * xk;
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (i64 i = n; i-- > 0;) {
            double s = x[i];
            for (i64 j = i + 1; j < n; ++j) s = s - lu[i * n + j] * x[j];
            x[i] = s / lu[i * n + i];
        }
}

} // namespace

void vec_copy(double* d, const double* s, i64 n, cudaStream_t st) {
    if (n <= 0 || d == s) return;
    ILUG_CUDA(cudaMemcpyAsync(d, s, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToDevice, st));
}
void vec_zero(double* d, i64 n, cudaStream_t st) {
    if (n > 0) ILUG_CUDA(cudaMemsetAsync(d, 0, static_cast<size_t>(n) * sizeof(double), st));
}
void vec_div(double* o, const double* a, const double* d, i64 n, cudaStream_t st) {
    if (n <= 0) return;
    k_div<<<ew_grid(n), kBlock, 0, st>>>(o, a, d, n);
    ILUG_LAUNCH_CHECK();
}
void vec_acc(double* x, const double* z, i64 n, cudaStream_t st) {
    if (n <= 0) return;
    k_acc<<<ew_grid(n), kBlock, 0, st>>>(x, z, n);
    ILUG_LAUNCH_CHECK();
}
void vec_acc_div(double* x, const double* z, const double* d, i64 n, cudaStream_t st) {
    if (n <= 0) return;
    k_acc_div<<<ew_grid(n), kBlock, 0, st>>>(x, z, d, n);
    ILUG_LAUNCH_CHECK();
}
void vec_scale_div(double* o, const double* w, double h, i64 n, cudaStream_t st) {
    if (n <= 0) return;
    k_scale_div<<<ew_grid(n), kBlock, 0, st>>>(o, w, h, n);
    ILUG_LAUNCH_CHECK();
}
void vec_scale_div_dev(double* o, const double* w, const double* h, i64 n, cudaStream_t st) {
    if (n <= 0) return;
    k_scale_div_dev<<<ew_grid(n), kBlock, 0, st>>>(o, w, h, n);
    ILUG_LAUNCH_CHECK();
}
void vec_add_into(double* o, const double* a, const double* b, i64 n, cudaStream_t st) {
    if (n <= 0) return;
    k_add_into<<<ew_grid(n), kBlock, 0, st>>>(o, a, b, n);
    ILUG_LAUNCH_CHECK();
}
void vec_sub_into(double* o, const double* a, const double* b, i64 n, cudaStream_t st) {
    if (n <= 0) return;
    k_sub_into<<<ew_grid(n), kBlock, 0, st>>>(o, a, b, n);
    ILUG_LAUNCH_CHECK();
}
i64 reduce_ws_doubles(i64 n, i64 k) {
    return std::max<i64>(1, (n + kTile - 1) / kTile) * std::max<i64>(kMaxVec, k);
}
void dot_dev(const double* a, const double* b, i64 n, double* out, double* ws, cudaStream_t st) {
    tiled<0>(nullptr, 0, 0, nullptr, const_cast<double*>(a), b, n, out, 1, ws, st);
}
void nrm2sq_dev(const double* a, i64 n, double* out, double* ws, cudaStream_t st) {
    tiled<1>(nullptr, 0, 0, nullptr, const_cast<double*>(a), nullptr, n, out, 1, ws, st);
}
void nrm2sq_diff_dev(const double* w, const double* v, const double* h, i64 n, double* out, double* ws,
                     cudaStream_t st) {
    tiled<5>(nullptr, 0, 0, h, const_cast<double*>(w), v, n, out, 1, ws, st);
}
void multi_dot(const double* V, i64 ld, int k, const double* w, i64 n, double* h, double* ws, cudaStream_t st) {
    tiled<2>(V, ld, k, nullptr, const_cast<double*>(w), nullptr, n, h, k, ws, st);
}
void multi_axpy_dot(const double* V, i64 ld, int k, const double* hin, double* w, i64 n, double* hout,
                    double* ws, cudaStream_t st) {
    tiled<3>(V, ld, k, hin, w, nullptr, n, hout, k, ws, st);
}
void multi_axpy_nrm(const double* V, i64 ld, int k, const double* hin, double* w, i64 n, double* out,
                    double* ws, cudaStream_t st) {
    tiled<4>(V, ld, k, hin, w, nullptr, n, out, 1, ws, st);
}
void multi_combine(const double* V, i64 ld, int k, const double* c, const double* base, double* y,
                   i64 n, cudaStream_t st) {
    if (n <= 0) return;
    k_combine<<<ew_grid(n), kBlock, 0, st>>>(V, ld, k, c, base, y, n);
    ILUG_LAUNCH_CHECK();
}
void dense_lu_solve_dev(i64 n, const double* lu, const i64* piv, const double* b, double* x,
                        cudaStream_t st) {
    if (n <= 0) return;
    k_dense_solve<<<1, kBlock, 0, st>>>(n, lu, piv, b, x);
    ILUG_LAUNCH_CHECK();
}

} // namespace ilug
