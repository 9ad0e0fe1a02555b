// Sparse matrix product C = A B on the device (the AMG Galerkin product R (A P),
// SURVEY.md §8f rank 1), bitwise equal to host/csr.cpp csr_matmul and the
// reference's SparseMatrix::multiply (src/sparse.cpp:176-231).
//
// The reference accumulates row i of C in a dense accumulator: for k ascending
// in A's row, for j ascending in B's row k, acc[j] += a_ik * b_kj (acc starts at
// 0.0), then emits the touched columns in ascending order, dropping exact
// zeros. Here a warp owns a row and keeps the accumulator as an open-addressing
// hash table (column -> value) in its shared memory: the k steps run in order
// and within one step every lane adds to a distinct column (B's row has
// distinct columns), so every acc[j] receives its products in the reference's
// order with the same rounding. The surviving entries (value != 0.0; NaN kept)
// are compacted and bitonic-sorted by column. Two passes: count, then fill at
// the prefix offsets. Rows whose distinct columns overflow the table are
// queued and redone with a larger table (fewer warps per CTA).
#include "spgemm.hpp"

#include <cub/device/device_scan.cuh>

#include <climits>
#include <cstdlib>

namespace ilug {

namespace {

struct Args {
    i64 nrows;
    const i64* arp;
    const i32* aci;
    const double* av;
    const i64* brp;
    const i32* bci;
    const double* bv;
    i64* cnt;        // count pass: entries of row i (at cnt[i + 1])
    const i64* crp;  // fill pass: row starts
    i32* cci;
    double* cv;
    const i64* rows; // nullptr: all rows; else the listed rows (overflow retries)
    i64 nlist;
    i64* ovf;        // ovf[0] count, ovf[1..] rows
    i64 ovf_cap;
};

// Fibonacci hashing: the top bits of the product (CAP is a power of two)
template <int CAP>
__device__ __forceinline__ unsigned hash_col(i32 j) {
    constexpr int kLog = CAP == 512 ? 9 : CAP == 4096 ? 12 : 14;
    return (static_cast<unsigned>(j) * 2654435761u) >> (32 - kLog);
}

template <int CAP, int WARPS, bool FILL>
__global__ void __launch_bounds__(WARPS * 32) k_spgemm(Args a) {
    extern __shared__ double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per warp: vals[CAP] doubles, keys[CAP] ints (then reused for the sort)
    double* vals = smem + static_cast<size_t>(warp) * CAP;
    i32* keys = reinterpret_cast<i32*>(smem + static_cast<size_t>(WARPS) * CAP) + static_cast<size_t>(warp) * CAP;
    const unsigned full = 0xffffffffu;
    const i64 nwork = a.rows ? a.nlist : a.nrows;
    const i64 gw = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const i64 nw = (static_cast<i64>(gridDim.x) * blockDim.x) >> 5;
    for (i64 w = gw; w < nwork; w += nw) {
        const i64 i = a.rows ? a.rows[w] : w;
        for (int q = lane; q < CAP; q += 32) keys[q] = -1;
        __syncwarp();
        bool over = false;
        for (i64 ka = a.arp[i]; ka < a.arp[i + 1] && !over; ++ka) {
            const i32 k = a.aci[ka];
            const double aik = a.av[ka];
            const i64 bb = a.brp[k], be = a.brp[k + 1];
            for (i64 c0 = bb; c0 < be; c0 += 32) {
                const i64 kb = c0 + lane;
                bool bad = false;
                if (kb < be) {
                    const i32 j = a.bci[kb];
                    const double p = aik * a.bv[kb];
                    unsigned h = hash_col<CAP>(j);
                    for (int probe = 0;; ++probe) {
                        if (probe == CAP) {
                            bad = true;
                            break;
                        }
                        const i32 key = keys[h];
                        if (key == j) {
                            vals[h] = vals[h] + p;
                            break;
                        }
                        if (key == -1) {
                            const i32 old = atomicCAS(keys + h, -1, j);
                            if (old == -1) {
                                vals[h] = 0.0 + p; // acc[j] starts at 0.0
                                break;
                            }
                            if (old == j) { // not reachable: B's row holds distinct columns
                                vals[h] = vals[h] + p;
                                break;
                            }
                        }
                        h = (h + 1) & (CAP - 1);
                    }
                }
                over = __any_sync(full, bad);
                __syncwarp();
                if (over) break;
            }
        }
        if (over) {
            if (lane == 0) {
                const i64 slot = atomicAdd(reinterpret_cast<unsigned long long*>(a.ovf), 1ull);
                if (slot < a.ovf_cap) a.ovf[1 + slot] = i;
            }
            __syncwarp();
            continue;
        }
        // compact the surviving entries (value != 0.0, NaN kept) to the front
        // of the table: first collect into registers chunk by chunk
        int m = 0;
        for (int q0 = 0; q0 < CAP; q0 += 32) {
            const int q = q0 + lane;
            const i32 key = keys[q];
            const double v = key >= 0 ? vals[q] : 0.0;
            const bool keep = key >= 0 && v != 0.0;
            const unsigned bal = __ballot_sync(full, keep);
            __syncwarp();
            if (keep) {
                const int dst = m + __popc(bal & ((1u << lane) - 1u));
                // dst <= q: never overwrites an unread slot of this or a later chunk
                keys[dst] = key;
                vals[dst] = v;
            }
            m += __popc(bal);
            __syncwarp();
        }
        if (!FILL) {
            if (lane == 0) a.cnt[i + 1] = m;
            __syncwarp();
            continue;
        }
        // bitonic sort of keys[0, np) (padded with INT_MAX) carrying vals
        int np = 1;
        while (np < m) np <<= 1;
        for (int q = m + lane; q < np; q += 32) keys[q] = INT_MAX;
        __syncwarp();
        for (int size = 2; size <= np; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = lane; t < np / 2; t += 32) {
                    const int lo = 2 * t - (t & (stride - 1));
                    const int hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const i32 kl = keys[lo], kh = keys[hi];
                    if ((kl > kh) == up) {
                        keys[lo] = kh, keys[hi] = kl;
                        const double vl = vals[lo];
                        vals[lo] = vals[hi], vals[hi] = vl;
                    }
                }
                __syncwarp();
            }
        }
        const i64 o = a.crp[i];
        for (int q = lane; q < m; q += 32) {
            a.cci[o + q] = keys[q];
            a.cv[o + q] = vals[q];
        }
        __syncwarp();
    }
}

template <int CAP, int WARPS, bool FILL>
void launch(const Args& a, cudaStream_t st) {
    constexpr size_t smem = static_cast<size_t>(WARPS) * CAP * (sizeof(double) + sizeof(i32));
    auto* fn = k_spgemm<CAP, WARPS, FILL>;
    ILUG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    ILUG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, WARPS * 32, smem));
    const i64 work = a.rows ? a.nlist : a.nrows;
    const i64 grid = std::max<i64>(1, std::min<i64>(static_cast<i64>(std::max(per_sm, 1)) * device_sm_count(),
                                                    (work + WARPS - 1) / WARPS));
    fn<<<static_cast<unsigned>(grid), WARPS * 32, smem, st>>>(a);
    ILUG_LAUNCH_CHECK();
}

// Run one pass over all rows with the smallest table, then over the overflow
// rows with the larger ones. Returns false if a row overflows every tier.
template <bool FILL>
bool run_pass(Args a, DBuf<i64>& ovf, cudaStream_t st) {
    const i64 cap = ovf.n - 1;
    a.ovf = ovf.p;
    a.ovf_cap = cap;
    ILUG_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(i64), st));
    launch<512, 16, FILL>(a, st);
    for (int tier = 0; tier < 2; ++tier) {
        i64 nov = 0;
        ILUG_CUDA(cudaMemcpyAsync(&nov, ovf.p, sizeof nov, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        if (nov == 0) return true;
        if (nov > cap) return false;
        DBuf<i64> list(nov);
        ILUG_CUDA(cudaMemcpyAsync(list.p, ovf.p + 1, static_cast<size_t>(nov) * sizeof(i64),
                                  cudaMemcpyDeviceToDevice, st));
        ILUG_CUDA(cudaMemsetAsync(ovf.p, 0, sizeof(i64), st));
        Args b = a;
        b.rows = list.p;
        b.nlist = nov;
        if (tier == 0)
            launch<4096, 4, FILL>(b, st);
        else
            launch<16384, 1, FILL>(b, st);
        ILUG_CUDA(cudaStreamSynchronize(st)); // list dies at scope exit
    }
    i64 nov = 0;
    ILUG_CUDA(cudaMemcpyAsync(&nov, ovf.p, sizeof nov, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    return nov == 0;
}

} // namespace

bool spgemm_device(i64 nrows, i64 ncols, const DevCsr& A, const DevCsr& B, DevCsr& C, cudaStream_t st) {
    C.nrows = nrows;
    C.ncols = ncols;
    C.rp.alloc(nrows + 1);
    ILUG_CUDA(cudaMemsetAsync(C.rp.p, 0, static_cast<size_t>(nrows + 1) * sizeof(i64), st));
    DBuf<i64> ovf(1 + std::max<i64>(nrows / 64, 1024));
    Args a{nrows, A.rp.p, A.ci.p, A.v.p, B.rp.p, B.ci.p, B.v.p, C.rp.p, nullptr, nullptr, nullptr,
           nullptr, 0, nullptr, 0};
    if (nrows > 0 && !run_pass<false>(a, ovf, st)) return false;
    size_t tmp = 0;
    ILUG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, C.rp.p, C.rp.p, nrows + 1, st));
    DBuf<char> t(static_cast<i64>(std::max<size_t>(tmp, 1)));
    ILUG_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, C.rp.p, C.rp.p, nrows + 1, st));
    i64 nnz = 0;
    ILUG_CUDA(cudaMemcpyAsync(&nnz, C.rp.p + nrows, sizeof nnz, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    C.ci.alloc(nnz);
    C.v.alloc(nnz);
    a.cnt = nullptr;
    a.crp = C.rp.p;
    a.cci = C.ci.p;
    a.cv = C.v.p;
    if (nrows > 0 && nnz > 0 && !run_pass<true>(a, ovf, st)) return false;
    ILUG_CUDA(cudaStreamSynchronize(st));
    return true;
}

void DevCsr::upload(const Csr& h, cudaStream_t st) {
    nrows = h.nrows;
    ncols = h.ncols;
    rp.upload(h.rp.data(), h.nrows + 1, st);
    ci.upload(h.ci.data(), h.nnz(), st);
    v.upload(h.v.data(), h.nnz(), st);
}

Csr DevCsr::download(cudaStream_t st) const {
    Csr h;
    h.nrows = nrows;
    h.ncols = ncols;
    h.rp.resize(static_cast<size_t>(nrows) + 1);
    h.ci.resize(static_cast<size_t>(ci.n));
    h.v.resize(static_cast<size_t>(v.n));
    rp.download(h.rp.data(), st);
    ci.download(h.ci.data(), st);
    v.download(h.v.data(), st);
    ILUG_CUDA(cudaStreamSynchronize(st));
    return h;
}

Csr spgemm_device_host(const Csr& A, const Csr& B, cudaStream_t st) {
    if (A.ncols != B.nrows) fail_invalid("matmul: dimension mismatch");
    DevCsr dA, dB, dC;
    dA.upload(A, st);
    dB.upload(B, st);
    if (!spgemm_device(A.nrows, B.ncols, dA, dB, dC, st)) return csr_matmul(A, B);
    return dC.download(st);
}

// Off by default: with the rest of the AMG setup on the host, the operand
// uploads and the coarse-operator download eat the gain, and the products
// compete with the concurrent device factorisation for the GPU and the
// staging buffers (C2 level 0: 1.14 s device vs 1.03 s host on 16 cores, C2
// setup +2.9 s with it on; C4 level 0 with staged downloads: 2.2 s vs 5.0 s,
// setup 21.3 vs 23.6 s). The kernels are the building block for a device-resident
// hierarchy setup. ILUG_GALERKIN_DEVICE=1 enables it.
bool galerkin_on_device() {
    const char* e = std::getenv("ILUG_GALERKIN_DEVICE");
    return e && e[0] == '1';
}

Csr galerkin_device(const Csr& A, const Csr& P, const Csr& R, cudaStream_t st) {
    if (A.ncols != P.nrows || R.ncols != A.nrows) fail_invalid("matmul: dimension mismatch");
    SetupTimer tm("galerkin-device");
    DevCsr dA, dP, dAP, dR, dC;
    dA.upload(A, st);
    dP.upload(P, st);
    dR.upload(R, st);
    ILUG_CUDA(cudaStreamSynchronize(st));
    tm.mark("upload A,P,R");
    if (!spgemm_device(A.nrows, P.ncols, dA, dP, dAP, st)) return csr_matmul(R, csr_matmul(A, P));
    tm.mark("A*P");
    dA = DevCsr{};
    dP = DevCsr{};
    if (!spgemm_device(R.nrows, P.ncols, dR, dAP, dC, st)) return csr_matmul(R, dAP.download(st));
    tm.mark("R*(AP)");
    Csr out = dC.download(st);
    tm.mark("download");
    return out;
}

} // namespace ilug
