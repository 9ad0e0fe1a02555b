// ILU(0) factorisation on the device, bitwise equal to
// the reference's IKJ ILU(0) (src/ilu.cpp:56-118) and to host/ilu.cpp.
//
// One thread per row. Row i needs rows c < i of its lower pattern finished;
// instead of level barriers every row waits on its dependencies' epoch-stamped
// done flags, just before it uses each one (sync-free, like the K5 flag
// schedule). CTAs take their row block from an atomic ticket over the rows in
// wavefront (level) order, so a block holds independent rows and only ever
// waits on blocks scheduled before it: no deadlock whatever the residency. Each row performs the serial algorithm's operations in its order
// (multipliers by ascending k, then the merge of row c's strict upper part in
// ascending column order), with separate multiply/subtract (--fmad=false), so
// the factors are bitwise the host ones. A bounded spin turns a scheduling bug
// into an error instead of a hung GPU.
#include "ilu0.hpp"
#include "spgemm.hpp"

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
       unsigned* ticket, unsigned long long* first_zero, unsigned* err, int patch, double anorm_f,
       const i32* __restrict__ order) {
    __shared__ unsigned s_blk;
    if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned E = *epoch_p;
    const i64 t = static_cast<i64>(s_blk) * kBlock + threadIdx.x;
    if (t >= n) return;
    // rows in wavefront (level) order when given: a block then holds rows of one
    // level (independent) instead of a chain of x-neighbours, and a row's
    // dependencies are always in earlier blocks (no deadlock)
    const i64 i = order ? order[t] : t;
    const i64 beg = rp[i], end = rp[i + 1], di = dpos[i];
    for (i64 k = beg; k < di; ++k) {
        const i64 c = ci[k];
        if (!wait_flag<64>(done + c, E)) atomicExch(err, 1u);
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

// Warp-per-row form (rows of at most 64 entries, the common case): the row's
// values live in the lanes' registers (entries l and l+32 on lane l), and the
// merge of row c's strict upper part is a broadcast of its (column, value)
// pairs — one load round trip per dependency instead of the thread form's
// serial scan. Each entry still receives its updates in ascending k with the
// same multiply/subtract, so the factors are bitwise those of k_ilu0.
constexpr int kWarpRowsPerCta = 8;

__global__ void __launch_bounds__(kWarpRowsPerCta * 32)
k_ilu0_warp(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci, const i64* __restrict__ dpos,
            const double* __restrict__ a, double* w, unsigned* done, const unsigned* __restrict__ epoch_p,
            unsigned* ticket, unsigned long long* first_zero, unsigned* err, int patch, double anorm_f,
            const i32* __restrict__ order) {
    __shared__ unsigned s_blk;
    if (threadIdx.x == 0) s_blk = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned full = 0xffffffffu;
    const unsigned E = *epoch_p;
    const int lane = threadIdx.x & 31;
    const i64 t = static_cast<i64>(s_blk) * kWarpRowsPerCta + (threadIdx.x >> 5);
    if (t >= n) return;
    const i64 i = order ? order[t] : t;
    const i64 beg = rp[i], len = rp[i + 1] - beg, dq = dpos[i] - beg;
    // row values in registers: slot 0 = entry lane, slot 1 = entry lane + 32
    const bool h0 = lane < len, h1 = lane + 32 < len;
    const i32 j0 = h0 ? ci[beg + lane] : -1, j1 = h1 ? ci[beg + lane + 32] : -1;
    double v0 = h0 ? w[beg + lane] : 0.0, v1 = h1 ? w[beg + lane + 32] : 0.0;
    for (i64 q = 0; q < dq; ++q) {
        const int src = static_cast<int>(q & 31);
        const i32 c = __shfl_sync(full, q < 32 ? j0 : j1, src);
        if (!wait_flag<64>(done + c, E)) atomicExch(err, 1u);
        const i64 dc = dpos[c], ce = rp[c + 1];
        const double wk = __shfl_sync(full, q < 32 ? v0 : v1, src);
        const double m = wk / w[dc];
        if (lane == src) {
            if (q < 32) v0 = m;
            else v1 = m;
        }
        // row c's strict upper part, 32 entries at a time
        for (i64 cb = dc + 1; cb < ce; cb += 32) {
            const bool has = cb + lane < ce;
            const i32 jc = has ? ci[cb + lane] : -1;
            const double vc = has ? w[cb + lane] : 0.0;
            const int cnt = ce - cb < 32 ? static_cast<int>(ce - cb) : 32;
            for (int u = 0; u < cnt; ++u) {
                const i32 ju = __shfl_sync(full, jc, u);
                const double vu = __shfl_sync(full, vc, u);
                if (h0 && j0 == ju) v0 = v0 - m * vu;
                if (h1 && j1 == ju) v1 = v1 - m * vu;
            }
        }
    }
    // zero pivot (the lane holding the diagonal)
    const int dl = static_cast<int>(dq & 31);
    if (lane == dl) {
        double& d = dq < 32 ? v0 : v1;
        if (d == 0.0) {
            if (patch == 0) {
                atomicMin(first_zero, static_cast<unsigned long long>(i));
                d = 1.0; // placeholder; the factorisation is abandoned
            } else {
                double s2 = 0.0;
                for (i64 k = beg; k < beg + len; ++k) s2 = s2 + a[k] * a[k];
                const double zr = 0.0 * sqrt(s2), fl = 1e-16 * anorm_f;
                double mag = zr < fl ? fl : zr; // std::max(zr, fl)
                if (mag == 0.0) mag = DBL_MIN;
                d = mag;
            }
        }
    }
    if (h0) w[beg + lane] = v0;
    if (h1) w[beg + lane + 32] = v1;
    __syncwarp(); // every lane's row write before lane 0's release (cumulative)
    if (lane == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> fi(done[i]);
        fi.store(E, cuda::memory_order_release);
    }
}

// w (A's pattern) -> strict L and U (diagonal first) on the device, thread per row
__global__ void k_ilu0_split(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                             const i64* __restrict__ dpos, const double* __restrict__ w,
                             const i64* __restrict__ lrp, const i64* __restrict__ urp, i32* __restrict__ lci,
                             double* __restrict__ lv, i32* __restrict__ uci, double* __restrict__ uv) {
    const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    i64 pl = lrp[i], pu = urp[i];
    const i64 di = dpos[i];
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
        if (k < di)
            lci[pl] = ci[k], lv[pl++] = w[k];
        else
            uci[pu] = ci[k], uv[pu++] = w[k];
    }
}

} // namespace

namespace {

// The elimination proper, into wd (a copy of the values a). |A|_F (a serial
// sum over every value, as the reference computes it) only matters for a
// patched zero pivot, so it is computed only if one occurs: the first launch
// detects zero pivots; under pivot_patch=replace a second launch then runs
// with the norm. Without zero pivots both policies give the same factors.
bool ilu0_warp_enabled() { // ILUG_ILU0_WARP=0: the thread-per-row kernel (A/B)
    const char* e = std::getenv("ILUG_ILU0_WARP");
    return !(e && e[0] == '0');
}

void ilu0_eliminate(i64 n, const i64* rp, const i32* ci, const i64* dpos, const double* a, double* wd, i64 nnz,
                    PivotPatch patch, const Csr& A, const i32* order, cudaStream_t st) {
    i64 max_row = 0;
    for (i64 r = 0; r < A.nrows; ++r) max_row = std::max(max_row, A.rp[r + 1] - A.rp[r]);
    DBuf<unsigned> sync(n + 3); // done flags, epoch, ticket, error
    ILUG_CUDA(cudaMemsetAsync(sync.p, 0, static_cast<size_t>(n + 3) * sizeof(unsigned), st));
    DBuf<unsigned long long> fz(1);
    unsigned* epoch = sync.p + n;
    double anorm_f = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
        const unsigned long long init = ~0ull;
        ILUG_CUDA(cudaMemcpyAsync(fz.p, &init, sizeof init, cudaMemcpyHostToDevice, st));
        ILUG_CUDA(cudaMemcpyAsync(wd, a, static_cast<size_t>(nnz) * sizeof(double), cudaMemcpyDeviceToDevice, st));
        k_ilu0_bump<<<1, 1, 0, st>>>(epoch, epoch + 1);
        ILUG_LAUNCH_CHECK();
        if (max_row <= 64 && ilu0_warp_enabled()) {
            const unsigned g = static_cast<unsigned>((n + kWarpRowsPerCta - 1) / kWarpRowsPerCta);
            k_ilu0_warp<<<g, kWarpRowsPerCta * 32, 0, st>>>(n, rp, ci, dpos, a, wd, sync.p, epoch, epoch + 1, fz.p,
                                                            epoch + 2, pass, anorm_f, order);
        } else {
            const unsigned g = static_cast<unsigned>((n + kBlock - 1) / kBlock);
            k_ilu0<<<g, kBlock, 0, st>>>(n, rp, ci, dpos, a, wd, sync.p, epoch, epoch + 1, fz.p, epoch + 2, pass,
                                         anorm_f, order);
        }
        ILUG_LAUNCH_CHECK();
        unsigned long long h = 0;
        unsigned bad = 0;
        ILUG_CUDA(cudaStreamSynchronize(st)); // not inside the pageable copies (see ilut.cu)
        ILUG_CUDA(cudaMemcpyAsync(&h, fz.p, sizeof h, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaMemcpyAsync(&bad, epoch + 2, sizeof bad, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        if (bad) fail_numeric("ilu0 (device): dependency wait timed out (scheduling error)");
        if (h == ~0ull || pass == 1) return;
        if (patch == PivotPatch::error)
            fail_numeric("zero pivot at step " + std::to_string(h) +
                         " (no pivoting; rerun with pivot_patch=replace to substitute)");
        anorm_f = frobenius_norm(A);
    }
}

} // namespace

// Rows sorted by wavefront level of the lower-pattern DAG (level[i] = 1 +
// max level of its lower neighbours), stable within a level.
std::vector<i32> ilu0_level_order(const Csr& A, const std::vector<i64>& dpos) {
    const i64 n = A.nrows;
    std::vector<i32> level(static_cast<size_t>(n), 0);
    i32 nlev = n > 0 ? 1 : 0;
    for (i64 i = 0; i < n; ++i) {
        i32 l = 0;
        for (i64 k = A.rp[i]; k < dpos[i]; ++k) l = std::max(l, level[A.ci[k]] + 1);
        level[i] = l;
        nlev = std::max(nlev, l + 1);
    }
    std::vector<i64> start(static_cast<size_t>(nlev) + 1, 0);
    for (i64 i = 0; i < n; ++i) ++start[level[i] + 1];
    for (i32 l = 0; l < nlev; ++l) start[l + 1] += start[l];
    std::vector<i32> order(static_cast<size_t>(n));
    for (i64 i = 0; i < n; ++i) order[start[level[i]]++] = static_cast<i32>(i);
    return order;
}

bool ilu0_on_device() {
    const char* e = std::getenv("ILUG_ILU0_DEVICE");
    return !(e && e[0] == '0');
}

HostFactors DevFactors::to_host(cudaStream_t st) const {
    HostFactors f;
    for (int part = 0; part < 2; ++part) {
        Csr& M = part == 0 ? f.L : f.U;
        M.nrows = M.ncols = n;
        M.rp = part == 0 ? Lrp_h : Urp_h;
        const DBuf<i32>& c = part == 0 ? Lci : Uci;
        const DBuf<double>& v = part == 0 ? Lv : Uv;
        M.ci.resize(static_cast<size_t>(c.n));
        M.v.resize(static_cast<size_t>(v.n));
        c.download(M.ci.data(), st);
        v.download(M.v.data(), st);
    }
    ILUG_CUDA(cudaStreamSynchronize(st));
    return f;
}

DevFactors DevFactors::upload(const HostFactors& f, cudaStream_t st) {
    DevFactors d;
    d.n = f.U.nrows;
    d.Lrp_h = f.L.rp;
    d.Urp_h = f.U.rp;
    d.Lrp.upload(f.L.rp.data(), d.n + 1, st);
    d.Urp.upload(f.U.rp.data(), d.n + 1, st);
    d.Lci.upload(f.L.ci.data(), f.L.nnz(), st);
    d.Uci.upload(f.U.ci.data(), f.U.nnz(), st);
    d.Lv.upload(f.L.v.data(), f.L.nnz(), st);
    d.Uv.upload(f.U.v.data(), f.U.nnz(), st);
    d.diag_first = true;
    for (i64 i = 0; i < d.n && d.diag_first; ++i)
        d.diag_first = f.U.rp[i] < f.U.rp[i + 1] && f.U.ci[f.U.rp[i]] == i;
    ILUG_CUDA(cudaStreamSynchronize(st)); // host vectors may die after return
    return d;
}

DevFactors ilu0_resident(const Csr& A, PivotPatch patch, cudaStream_t st, bool keep_A, const DevCsr* Ad) {
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
    const i64 nnz = A.nnz();
    DevFactors f;
    f.n = n;
    f.diag_first = true;
    f.Lrp_h.assign(static_cast<size_t>(n) + 1, 0);
    f.Urp_h.assign(static_cast<size_t>(n) + 1, 0);
    for (i64 i = 0; i < n; ++i) {
        f.Lrp_h[i + 1] = f.Lrp_h[i] + (dpos[i] - A.rp[i]);
        f.Urp_h[i + 1] = f.Urp_h[i] + (A.rp[i + 1] - dpos[i]);
    }
    if (n == 0) {
        f.Lrp.upload(f.Lrp_h.data(), 1, st);
        f.Urp.upload(f.Urp_h.data(), 1, st);
        ILUG_CUDA(cudaStreamSynchronize(st));
        return f;
    }
    DBuf<i64> rp, dp;
    DBuf<i32> ci;
    DBuf<double> a, wd;
    if (!Ad) {
        rp.upload(A.rp.data(), n + 1, st);
        ci.upload(A.ci.data(), nnz, st);
        a.upload(A.v.data(), nnz, st);
    }
    const i64* const rpp = Ad ? Ad->rp.p : rp.p;
    const i32* const cip = Ad ? Ad->ci.p : ci.p;
    const double* const ap = Ad ? Ad->v.p : a.p;
    dp.upload(dpos.data(), n, st);
    wd.alloc(nnz);
    DBuf<i32> ord;
    {
        const std::vector<i32> o = ilu0_level_order(A, dpos);
        ord.upload(o.data(), n, st);
    }
    ilu0_eliminate(n, rpp, cip, dp.p, ap, wd.p, nnz, patch, A, ord.p, st);
    f.Lrp.upload(f.Lrp_h.data(), n + 1, st);
    f.Urp.upload(f.Urp_h.data(), n + 1, st);
    f.Lci.alloc(f.Lrp_h[n]);
    f.Lv.alloc(f.Lrp_h[n]);
    f.Uci.alloc(f.Urp_h[n]);
    f.Uv.alloc(f.Urp_h[n]);
    const unsigned g = static_cast<unsigned>((n + kBlock - 1) / kBlock);
    k_ilu0_split<<<g, kBlock, 0, st>>>(n, rpp, cip, dp.p, wd.p, f.Lrp.p, f.Urp.p, f.Lci.p, f.Lv.p, f.Uci.p,
                                       f.Uv.p);
    ILUG_LAUNCH_CHECK();
    ILUG_CUDA(cudaStreamSynchronize(st)); // temporaries die at scope exit
    if (keep_A && !Ad) f.Arp = std::move(rp), f.Aci = std::move(ci), f.Av = std::move(a);
    return f;
}

// Thread-count-independent hash of a column array (blocks hashed in
// parallel, combined in block order).
std::uint64_t csr_pattern_hash(const Csr& A) {
    const i64 nnz = A.nnz();
    constexpr i64 kB = i64{1} << 20;
    const i64 nb = (nnz + kB - 1) / kB;
    std::vector<std::uint64_t> part(static_cast<size_t>(std::max<i64>(nb, 1)), 0);
    parallel_ranges(nb, [&](i64 b, i64 e, int) {
        for (i64 blk = b; blk < e; ++blk) {
            std::uint64_t h = 1469598103934665603ull;
            for (i64 k = blk * kB; k < std::min(nnz, (blk + 1) * kB); ++k)
                h = (h ^ static_cast<std::uint32_t>(A.ci[k])) * 1099511628211ull;
            part[static_cast<size_t>(blk)] = h;
        }
    }, 1);
    std::uint64_t h = static_cast<std::uint64_t>(nnz);
    for (std::uint64_t x : part) h = (h ^ x) * 1099511628211ull + 0x9e3779b97f4a7c15ull;
    return h;
}

std::unique_ptr<Ilu0Symbolic> Ilu0Symbolic::analyse(const Csr& A, cudaStream_t st) {
    if (A.nrows != A.ncols) fail_invalid("ilu0: matrix must be square");
    auto s = std::make_unique<Ilu0Symbolic>();
    const i64 n = s->n = A.nrows;
    s->nnz = A.nnz();
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
    s->rp_h = A.rp;
    s->Lrp_h.assign(static_cast<size_t>(n) + 1, 0);
    s->Urp_h.assign(static_cast<size_t>(n) + 1, 0);
    for (i64 i = 0; i < n; ++i) {
        s->Lrp_h[i + 1] = s->Lrp_h[i] + (dpos[i] - A.rp[i]);
        s->Urp_h[i + 1] = s->Urp_h[i] + (A.rp[i + 1] - dpos[i]);
    }
    s->ci_hash = csr_pattern_hash(A);
    {
        const std::vector<i32> o = ilu0_level_order(A, dpos);
        s->order.upload(o.data(), n, st);
    }
    s->rp.upload(A.rp.data(), n + 1, st);
    s->ci.upload(A.ci.data(), s->nnz, st);
    s->dpos.upload(dpos.data(), n, st);
    s->Lrp.upload(s->Lrp_h.data(), n + 1, st);
    s->Urp.upload(s->Urp_h.data(), n + 1, st);
    ILUG_CUDA(cudaStreamSynchronize(st));
    return s;
}

DevFactors Ilu0Symbolic::factor(const Csr& A, PivotPatch patch, cudaStream_t st) const {
    SetupTimer tm("ilu0-refactor");
    if (A.nrows != n || A.nnz() != nnz || A.rp != rp_h || csr_pattern_hash(A) != ci_hash)
        fail_invalid("ilu0 refactor: the matrix pattern differs from the analysed one");
    tm.mark("pattern check");
    DevFactors f;
    f.n = n;
    f.diag_first = true;
    f.Lrp_h = Lrp_h;
    f.Urp_h = Urp_h;
    if (n == 0) {
        f.Lrp.upload(Lrp_h.data(), 1, st);
        f.Urp.upload(Urp_h.data(), 1, st);
        ILUG_CUDA(cudaStreamSynchronize(st));
        return f;
    }
    DBuf<double> a, wd;
    a.upload(A.v.data(), nnz, st);
    wd.alloc(nnz);
    ILUG_CUDA(cudaStreamSynchronize(st));
    tm.mark("upload values");
    ilu0_eliminate(n, rp.p, ci.p, dpos.p, a.p, wd.p, nnz, patch, A, order.p, st);
    tm.mark("factor kernel");
    f.Lrp.alloc(n + 1);
    f.Urp.alloc(n + 1);
    ILUG_CUDA(cudaMemcpyAsync(f.Lrp.p, Lrp.p, static_cast<size_t>(n + 1) * sizeof(i64), cudaMemcpyDeviceToDevice, st));
    ILUG_CUDA(cudaMemcpyAsync(f.Urp.p, Urp.p, static_cast<size_t>(n + 1) * sizeof(i64), cudaMemcpyDeviceToDevice, st));
    f.Lci.alloc(Lrp_h[n]);
    f.Lv.alloc(Lrp_h[n]);
    f.Uci.alloc(Urp_h[n]);
    f.Uv.alloc(Urp_h[n]);
    const unsigned g = static_cast<unsigned>((n + kBlock - 1) / kBlock);
    k_ilu0_split<<<g, kBlock, 0, st>>>(n, rp.p, ci.p, dpos.p, wd.p, f.Lrp.p, f.Urp.p, f.Lci.p, f.Lv.p, f.Uci.p,
                                       f.Uv.p);
    ILUG_LAUNCH_CHECK();
    ILUG_CUDA(cudaStreamSynchronize(st));
    return f;
}

HostFactors ilu0_device(const Csr& A, PivotPatch patch, cudaStream_t st) {
    return ilu0_resident(A, patch, st).to_host(st);
}

HostFactors ilut_device(const Csr& A, const IluParams& p, cudaStream_t st) {
    return ilut_resident(A, p, st).to_host(st);
}

HostFactors factorize(const Csr& A, const IluParams& p, cudaStream_t st) {
    if (p.variant == IluVariant::ilu0 && ilu0_on_device()) return ilu0_device(A, p.pivot_patch, st);
    if (p.variant == IluVariant::ilut && ilut_on_device()) return ilut_device(A, p, st);
    return ilu_factorize(A, p);
}

DevFactors factorize_resident(const Csr& A, const IluParams& p, cudaStream_t st, bool keep_A, const DevCsr* Ad) {
    if (p.variant == IluVariant::ilu0 && ilu0_on_device()) return ilu0_resident(A, p.pivot_patch, st, keep_A, Ad);
    if (p.variant == IluVariant::ilut && ilut_on_device()) return ilut_resident(A, p, st, keep_A, Ad);
    return DevFactors::upload(ilu_factorize(A, p), st);
}

} // namespace ilug
