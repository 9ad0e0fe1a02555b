// ILU(0) factorisation on the device, bitwise equal to
// the reference's IKJ ILU(0) (src/ilu.cpp:56-118) and to host/ilu.cpp.
//
// One thread per row. Row i needs rows c < i of its lower pattern finished;
// instead of level barriers every row waits on its dependencies' epoch-stamped
// done flags, just before it uses each one (sync-free, like the K5 flag
// schedule). CTAs take their row block from an atomic ticket, so a block only
// ever waits on blocks that were scheduled before it: no deadlock whatever the
// residency. Each row performs the serial algorithm's operations in its order
// (multipliers by ascending k, then the merge of row c's strict upper part in
// ascending column order), with separate multiply/subtract (--fmad=false), so
// the factors are bitwise the host ones. A bounded spin turns a scheduling bug
// into an error instead of a hung GPU.
#include "ilu0.hpp"

#include <cuda/atomic>

#include <cfloat>
#include <cstdlib>

namespace ilug {

namespace {

constexpr int kBlock = 128;

__global__ void k_ilu0_bump(unsigned* epoch, unsigned* ticket) {
    *epoch = *epoch + 1u;
    *ticket = 0u;
}

__global__ void __launch_bounds__(kBlock)
k_ilu0(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci, const i64* __restrict__ dpos,
       const double* __restrict__ a, double* w, unsigned* done, const unsigned* __restrict__ epoch_p,
       unsigned* ticket, unsigned long long* first_zero, unsigned* err, int patch, double anorm_f) {
    __shared__ unsigned s_blk;
    if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned E = *epoch_p;
    const i64 i = static_cast<i64>(s_blk) * kBlock + threadIdx.x;
    if (i >= n) return;
    const i64 beg = rp[i], end = rp[i + 1], di = dpos[i];
    for (i64 k = beg; k < di; ++k) {
        const i64 c = ci[k];
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> f(done[c]);
        if (f.load(cuda::memory_order_acquire) != E) {
            long long spins = 0;
            while (f.load(cuda::memory_order_acquire) != E) {
                if (++spins > (1ll << 26)) { // seconds: a scheduling bug, not a slow row
                    atomicExch(err, 1u);
                    break;
                }
                __nanosleep(64);
            }
        }
        const double m = w[k] / w[dpos[c]];
        w[k] = m;
        // merge row c's strict upper part against row i's tail (ascending columns)
        i64 p = k + 1;
        const i64 cend = rp[c + 1];
        for (i64 kk = dpos[c] + 1; kk < cend && p < end; ++kk) {
            const i32 j = ci[kk];
            while (p < end && ci[p] < j) ++p;
            if (p < end && ci[p] == j) w[p] = w[p] - m * w[kk];
        }
    }
    if (w[di] == 0.0) {
        if (patch == 0) {
            atomicMin(first_zero, static_cast<unsigned long long>(i));
            w[di] = 1.0; // placeholder; the factorisation is abandoned
        } else {
            // patch_pivot(0.0, |a_i|_2, |A|_F): max(0 * rownorm, 1e-16 * |A|_F), DBL_MIN if 0
            double s = 0.0;
            for (i64 k = beg; k < end; ++k) s = s + a[k] * a[k];
            const double zr = 0.0 * sqrt(s), fl = 1e-16 * anorm_f;
            double mag = zr < fl ? fl : zr; // std::max(zr, fl)
            if (mag == 0.0) mag = DBL_MIN;
            w[di] = mag;
        }
    }
    cuda::atomic_ref<unsigned, cuda::thread_scope_device> fi(done[i]);
    fi.store(E, cuda::memory_order_release);
}

} // namespace

bool ilu0_on_device() {
    const char* e = std::getenv("ILUG_ILU0_DEVICE");
    return !(e && e[0] == '0');
}

HostFactors ilu0_device(const Csr& A, PivotPatch patch, cudaStream_t st) {
    if (A.nrows != A.ncols) fail_invalid("ilu0: matrix must be square");
    const i64 n = A.nrows;
    std::vector<i64> dpos(static_cast<size_t>(n), -1);
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i)
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k)
                if (A.ci[k] == i) dpos[i] = k;
    });
    for (i64 i = 0; i < n; ++i)
        if (dpos[i] < 0)
            fail_invalid("ilu0: diagonal entry (" + std::to_string(i) + "," + std::to_string(i) +
                         ") is structurally absent");
    const double anorm_f = frobenius_norm(A);
    const i64 nnz = A.nnz();
    std::vector<double> w(static_cast<size_t>(nnz));
    if (n > 0) {
        DBuf<i64> rp, dp;
        DBuf<i32> ci;
        DBuf<double> a, wd;
        rp.upload(A.rp.data(), n + 1, st);
        ci.upload(A.ci.data(), nnz, st);
        dp.upload(dpos.data(), n, st);
        a.upload(A.v.data(), nnz, st);
        wd.alloc(nnz);
        ILUG_CUDA(cudaMemcpyAsync(wd.p, a.p, static_cast<size_t>(nnz) * sizeof(double), cudaMemcpyDeviceToDevice,
                                  st));
        DBuf<unsigned> sync(n + 3); // done flags, epoch, ticket, error
        ILUG_CUDA(cudaMemsetAsync(sync.p, 0, static_cast<size_t>(n + 3) * sizeof(unsigned), st));
        DBuf<unsigned long long> fz(1);
        const unsigned long long init = ~0ull;
        ILUG_CUDA(cudaMemcpyAsync(fz.p, &init, sizeof init, cudaMemcpyHostToDevice, st));
        unsigned* epoch = sync.p + n;
        k_ilu0_bump<<<1, 1, 0, st>>>(epoch, epoch + 1);
        ILUG_LAUNCH_CHECK();
        const unsigned g = static_cast<unsigned>((n + kBlock - 1) / kBlock);
        k_ilu0<<<g, kBlock, 0, st>>>(n, rp.p, ci.p, dp.p, a.p, wd.p, sync.p, epoch, epoch + 1, fz.p, epoch + 2,
                                     patch == PivotPatch::error ? 0 : 1, anorm_f);
        ILUG_LAUNCH_CHECK();
        unsigned long long h = 0;
        unsigned bad = 0;
        ILUG_CUDA(cudaMemcpyAsync(&h, fz.p, sizeof h, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaMemcpyAsync(&bad, epoch + 2, sizeof bad, cudaMemcpyDeviceToHost, st));
        wd.download(w.data(), st);
        ILUG_CUDA(cudaStreamSynchronize(st));
        if (bad) fail_numeric("ilu0 (device): dependency wait timed out (scheduling error)");
        if (h != ~0ull)
            fail_numeric("zero pivot at step " + std::to_string(h) +
                         " (no pivoting; rerun with pivot_patch=replace to substitute)");
    }
    // split into strict L and U (with diagonal)
    HostFactors f;
    for (Csr* M : {&f.L, &f.U}) {
        M->nrows = M->ncols = n;
        M->rp.assign(static_cast<size_t>(n) + 1, 0);
    }
    for (i64 i = 0; i < n; ++i) {
        f.L.rp[i + 1] = f.L.rp[i] + (dpos[i] - A.rp[i]);
        f.U.rp[i + 1] = f.U.rp[i] + (A.rp[i + 1] - dpos[i]);
    }
    f.L.ci.resize(static_cast<size_t>(f.L.rp[n]));
    f.L.v.resize(static_cast<size_t>(f.L.rp[n]));
    f.U.ci.resize(static_cast<size_t>(f.U.rp[n]));
    f.U.v.resize(static_cast<size_t>(f.U.rp[n]));
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i) {
            i64 pl = f.L.rp[i], pu = f.U.rp[i];
            for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                if (k < dpos[i])
                    f.L.ci[pl] = A.ci[k], f.L.v[pl++] = w[k];
                else
                    f.U.ci[pu] = A.ci[k], f.U.v[pu++] = w[k];
            }
        }
    });
    return f;
}

HostFactors factorize(const Csr& A, const IluParams& p, cudaStream_t st) {
    if (p.variant == IluVariant::ilu0 && ilu0_on_device()) return ilu0_device(A, p.pivot_patch, st);
    if (p.variant == IluVariant::ilut && ilut_on_device()) return ilut_device(A, p, st);
    return ilu_factorize(A, p);
}

} // namespace ilug
