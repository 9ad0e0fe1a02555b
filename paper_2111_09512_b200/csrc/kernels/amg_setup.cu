// Device AMG setup: strength of connection, PMIS
// C/F splitting, direct and MM-ext interpolation, the transposes and the Galerkin
// product R (A P), level after level on the GPU, bitwise equal to the host
// setup and the reference (src/amg.cpp:18-390).
//
// Operation order is the reference's wherever floating point is involved:
//  * strength: cut = theta * max_{j != i} |a_ij|, S_ij iff |a_ij| >= cut (pure
//    comparisons);
//  * PMIS weights: |St row| + hash_unit(seed, i) (the reference's splitmix
//    hash, exact in double); rounds are synchronous — every decision of a round
//    reads the state at the round's start — so a parallel round is the serial
//    one; the order-dependent repair pass runs on one thread over the
//    ascending candidate list, like the host;
//  * direct interpolation: aii, beta, weak summed in the row's entry order,
//    w = -(a + beta / |C_s|) / (aii + weak), exact zeros dropped;
//  * MM-ext: the two scaled factors built per F-row (same sums, same zero
//    rules as the host's triplet assembly), their product by the SpGEMM;
//  * transposes list each row's columns ascending (entries gathered with
//    atomics, then every row sorted: a transpose does no arithmetic);
//  * the Galerkin products use the bitwise SpGEMM of kernels/spgemm.cu.
// Rows with no strong C-neighbour / a zero denominator are reported as the
// host does (invalid / numeric, lowest failing row first).
#include "amg_setup.hpp"

#include "../host/problems.hpp"

#include <cub/cub.cuh>

#include <future>

namespace ilug {

namespace {

constexpr int kB = 256;
inline unsigned grid_n(i64 n) {
    return static_cast<unsigned>(std::max<i64>(1, std::min<i64>((n + kB - 1) / kB, 148 * 64)));
}
#define GRID_STRIDE(i, n)                                                                  \
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < (n);          \
         i += static_cast<i64>(gridDim.x) * blockDim.x)

enum : char { kFree = 0, kC = 1, kF = 2 };

// exclusive scan of cnt[0..n) into rp[0..n] (rp[0] = 0), returns rp[n]
i64 scan_counts(const i64* cnt, i64* rp, i64 n, cudaStream_t st) {
    ILUG_CUDA(cudaMemsetAsync(rp, 0, sizeof(i64), st));
    if (n > 0) {
        size_t tmp = 0;
        ILUG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, cnt, rp + 1, n, st));
        DBuf<unsigned char> t(static_cast<i64>(tmp) + 1);
        ILUG_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, cnt, rp + 1, n, st));
    }
    i64 total = 0;
    ILUG_CUDA(cudaMemcpyAsync(&total, rp + n, sizeof total, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    return total;
}

// ---- strength (src/amg.cpp:18-50) --------------------------------------------
__global__ void k_strength_count(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                                 const double* __restrict__ v, double theta, double* __restrict__ cut,
                                 i64* __restrict__ cnt) {
    GRID_STRIDE(i, n) {
        double m = 0.0;
        for (i64 k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] != i) m = fmax(m, fabs(v[k]));
        const double c = m == 0.0 ? -1.0 : theta * m;
        cut[i] = c;
        i64 q = 0;
        if (c >= 0.0)
            for (i64 k = rp[i]; k < rp[i + 1]; ++k) q += ci[k] != i && fabs(v[k]) >= c;
        cnt[i] = q;
    }
}
__global__ void k_strength_fill(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                                const double* __restrict__ v, const double* __restrict__ cut,
                                const i64* __restrict__ srp, i32* __restrict__ sci) {
    GRID_STRIDE(i, n) {
        const double c = cut[i];
        if (c < 0.0) continue;
        i64 o = srp[i];
        for (i64 k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] != i && fabs(v[k]) >= c) sci[o++] = ci[k];
    }
}

// ---- transpose (src/sparse.cpp:233-257) --------------------------------------
__global__ void k_col_count(i64 nnz, const i32* __restrict__ ci, unsigned long long* __restrict__ cnt) {
    GRID_STRIDE(k, nnz) atomicAdd(cnt + ci[k], 1ull);
}
__global__ void k_row_of(i64 n, const i64* __restrict__ rp, i32* __restrict__ row) {
    GRID_STRIDE(i, n) for (i64 k = rp[i]; k < rp[i + 1]; ++k) row[k] = static_cast<i32>(i);
}
__global__ void k_scatter_t(i64 nnz, const i32* __restrict__ row, const i32* __restrict__ ci,
                            const double* __restrict__ v, unsigned long long* __restrict__ cursor,
                            i32* __restrict__ tci, double* __restrict__ tv) {
    GRID_STRIDE(k, nnz) {
        const i64 pos = static_cast<i64>(atomicAdd(cursor + ci[k], 1ull));
        tci[pos] = row[k];
        if (v) tv[pos] = v[k];
    }
}
// insertion sort of every row by column (a transpose row's entries are distinct)
__global__ void k_sort_rows(i64 n, const i64* __restrict__ rp, i32* __restrict__ ci, double* __restrict__ v) {
    GRID_STRIDE(i, n) {
        const i64 b = rp[i], e = rp[i + 1];
        for (i64 k = b + 1; k < e; ++k) {
            const i32 c = ci[k];
            const double x = v ? v[k] : 0.0;
            i64 q = k - 1;
            while (q >= b && ci[q] > c) {
                ci[q + 1] = ci[q];
                if (v) v[q + 1] = v[q];
                --q;
            }
            ci[q + 1] = c;
            if (v) v[q + 1] = x;
        }
    }
}

// ---- PMIS (src/amg.cpp:103-158) -----------------------------------------------
__device__ __forceinline__ std::uint64_t mix64(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__global__ void k_pmis_init(i64 n, const i64* __restrict__ trp, std::uint64_t seed, double* __restrict__ wt,
                            char* __restrict__ st, i64* __restrict__ live) {
    GRID_STRIDE(i, n) {
        const double h = static_cast<double>(mix64(seed ^ mix64(static_cast<std::uint64_t>(i))) >> 11) * 0x1.0p-53;
        wt[i] = static_cast<double>(trp[i + 1] - trp[i]) + h;
        st[i] = kFree;
        live[i] = i;
    }
}
__global__ void k_pmis_pick(i64 m, const i64* __restrict__ live, const i64* __restrict__ srp,
                            const i32* __restrict__ sci, const i64* __restrict__ trp, const i32* __restrict__ tci,
                            const double* __restrict__ wt, const char* __restrict__ st, char* __restrict__ picked,
                            unsigned long long* __restrict__ found) {
    GRID_STRIDE(q, m) {
        const i64 i = live[q];
        const double wi = wt[i];
        bool top = true;
        for (i64 k = srp[i]; top && k < srp[i + 1]; ++k) {
            const i64 j = sci[k];
            if (j != i && st[j] == kFree && wt[j] >= wi) top = false;
        }
        for (i64 k = trp[i]; top && k < trp[i + 1]; ++k) {
            const i64 j = tci[k];
            if (j != i && st[j] == kFree && wt[j] >= wi) top = false;
        }
        picked[q] = top;
        if (top) atomicAdd(found, 1ull);
    }
}
__global__ void k_pmis_mark(i64 m, const i64* __restrict__ live, const char* __restrict__ picked,
                            char* __restrict__ st, char* __restrict__ fresh, char set) {
    GRID_STRIDE(q, m) if (picked[q]) {
        const i64 i = live[q];
        fresh[i] = set;
        if (set) st[i] = kC;
    }
}
__global__ void k_pmis_fpass(i64 m, const i64* __restrict__ live, const i64* __restrict__ srp,
                             const i32* __restrict__ sci, const char* __restrict__ fresh, char* __restrict__ st,
                             char* __restrict__ keep) {
    GRID_STRIDE(q, m) {
        const i64 j = live[q];
        char k = 0;
        if (st[j] == kFree) {
            bool hit = false;
            for (i64 t = srp[j]; t < srp[j + 1] && !hit; ++t) hit = fresh[sci[t]] != 0;
            if (hit)
                st[j] = kF;
            else
                k = 1;
        }
        keep[q] = k;
    }
}
// repair pass candidates: F-points without a strong C-neighbour
__global__ void k_lacks_c(i64 n, const i64* __restrict__ srp, const i32* __restrict__ sci,
                          const char* __restrict__ st, char* __restrict__ cand) {
    GRID_STRIDE(i, n) {
        char c = 0;
        if (st[i] == kF) {
            c = 1;
            for (i64 k = srp[i]; k < srp[i + 1]; ++k)
                if (st[sci[k]] == kC) {
                    c = 0;
                    break;
                }
        }
        cand[i] = c;
    }
}
// the order-dependent pass over the ascending candidates (one thread)
__global__ void k_repair(i64 nc, const i64* __restrict__ cand, const i64* __restrict__ srp,
                         const i32* __restrict__ sci, char* __restrict__ st) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (i64 q = 0; q < nc; ++q) {
        const i64 i = cand[q];
        bool lacks = true;
        for (i64 k = srp[i]; lacks && k < srp[i + 1]; ++k) lacks = st[sci[k]] != kC;
        if (lacks) st[i] = kC;
    }
}
__global__ void k_is_coarse(i64 n, const char* __restrict__ st, i64* __restrict__ flag, char* __restrict__ isc) {
    GRID_STRIDE(i, n) {
        isc[i] = st[i] == kC;
        flag[i] = st[i] == kC;
    }
}
__global__ void k_coarse_index(i64 n, const char* __restrict__ isc, const i64* __restrict__ pre,
                               i64* __restrict__ cidx) {
    GRID_STRIDE(i, n) cidx[i] = isc[i] ? pre[i] : -1;
}

// ---- direct interpolation (src/amg.cpp:162-232) --------------------------------
// Weights of F-row i: returns the status (0 ok, 1 no strong C-neighbour, 2 zero
// denominator); FILL writes the nonzero weights at pci/pv, otherwise *q counts
// them. The weights are recomputed per pass instead of being stored.
template <bool FILL>
__device__ int direct_row(i64 i, const i64* __restrict__ rp, const i32* __restrict__ ci,
                          const double* __restrict__ v, const i64* __restrict__ srp, const i32* __restrict__ sci,
                          const char* __restrict__ isc, const i64* __restrict__ cidx, i64* q, i32* pci, double* pv) {
    double aii = 0.0, beta = 0.0, weak = 0.0;
    i64 nc = 0;
    i64 s = srp[i];
    const i64 se = srp[i + 1];
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
        const i64 j = ci[k];
        const double a = v[k];
        while (s < se && sci[s] < j) ++s;
        const bool strong = s < se && sci[s] == j;
        if (j == i) {
            aii = a;
        } else if (strong) {
            if (isc[j])
                ++nc;
            else
                beta += a;
        } else {
            weak += a;
            if (isc[j]) beta += a;
        }
    }
    const double denom = aii + weak;
    const int code = nc == 0 ? 1 : (denom == 0.0 ? 2 : 0);
    if (code) {
        if (!FILL) *q = 0;
        return code;
    }
    const double shift = beta / static_cast<double>(nc);
    i64 cnt = 0;
    s = srp[i];
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
        const i64 j = ci[k];
        while (s < se && sci[s] < j) ++s;
        const bool strong = s < se && sci[s] == j;
        if (j == i || !strong || !isc[j]) continue;
        const double w = -(v[k] + shift) / denom;
        if (w == 0.0) continue; // the reference's from_triplets drops exact zeros
        if (FILL)
            pci[cnt] = static_cast<i32>(cidx[j]), pv[cnt] = w;
        ++cnt;
    }
    if (!FILL) *q = cnt;
    return 0;
}

// pass 0: count (and status); pass 1: fill
template <int PASS>
__global__ void k_interp(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci, const double* __restrict__ v,
                         const i64* __restrict__ srp, const i32* __restrict__ sci, const char* __restrict__ isc,
                         const i64* __restrict__ cidx, i64* __restrict__ cnt, int* __restrict__ status,
                         unsigned long long* __restrict__ first_bad, const i64* __restrict__ prp,
                         i32* __restrict__ pci, double* __restrict__ pv) {
    GRID_STRIDE(i, n) {
        if (isc[i]) {
            if (PASS == 0) {
                cnt[i] = 1;
            } else {
                pci[prp[i]] = static_cast<i32>(cidx[i]);
                pv[prp[i]] = 1.0;
            }
            continue;
        }
        if (PASS == 0) {
            const int code = direct_row<false>(i, rp, ci, v, srp, sci, isc, cidx, &cnt[i], nullptr, nullptr);
            status[i] = code;
            if (code) atomicMin(first_bad, static_cast<unsigned long long>(i));
        } else {
            direct_row<true>(i, rp, ci, v, srp, sci, isc, cidx, nullptr, pci + prp[i], pv + prp[i]);
        }
    }
}

// ---- MM-ext interpolation (src/amg.cpp:235-346) ---------------------------------
// W = -[(D_FF + D_gamma)^-1 (A^s_FF + D_beta)] [D_beta^-1 A^s_FC] as the host
// restates it (host/amg.cpp interp_mm_ext): per F-row the sums d_ff, beta
// (strong C), gamma (weak) in the row's entry order; M1 = the row of
// (A^s_FF + D_beta) times 1/(d_ff + gamma) with exact zeros dropped (it is built
// from triplets), M2 = A^s_FC times 1/beta (0 on rows with beta == 0, which
// fall back to direct weights), zeros kept (a scaled copy); W = M1 M2 by the
// bitwise SpGEMM, negated.
struct MmRow {
    double dff, beta, gamma;
    i64 nff, nfc;
};
__device__ MmRow mm_sums(i64 i, const i64* __restrict__ rp, const i32* __restrict__ ci, const double* __restrict__ v,
                         const i64* __restrict__ srp, const i32* __restrict__ sci, const char* __restrict__ isc) {
    MmRow r{0.0, 0.0, 0.0, 0, 0};
    i64 s = srp[i];
    const i64 se = srp[i + 1];
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
        const i64 j = ci[k];
        while (s < se && sci[s] < j) ++s;
        const bool strong = s < se && sci[s] == j;
        if (j == i) {
            r.dff = v[k];
        } else if (strong) {
            if (isc[j])
                r.beta += v[k], ++r.nfc;
            else
                ++r.nff;
        } else {
            r.gamma += v[k];
        }
    }
    return r;
}

__global__ void k_mm_count(i64 nf, const i64* __restrict__ fglob, const i64* __restrict__ rp,
                           const i32* __restrict__ ci, const double* __restrict__ v, const i64* __restrict__ srp,
                           const i32* __restrict__ sci, const char* __restrict__ isc, double* __restrict__ inv1,
                           double* __restrict__ inv2, i64* __restrict__ c1, i64* __restrict__ c2,
                           unsigned long long* __restrict__ bad, unsigned long long* __restrict__ nfb) {
    GRID_STRIDE(fi, nf) {
        const i64 i = fglob[fi];
        const MmRow r = mm_sums(i, rp, ci, v, srp, sci, isc);
        const double den = r.dff + r.gamma;
        if (den == 0.0) {
            atomicMin(bad, static_cast<unsigned long long>(fi));
            c1[fi] = c2[fi] = 0;
            continue;
        }
        const double inv = 1.0 / den;
        inv1[fi] = inv;
        const bool fb = r.beta == 0.0;
        if (fb) atomicAdd(nfb, 1ull);
        inv2[fi] = fb ? 0.0 : 1.0 / r.beta;
        i64 q = r.beta * inv != 0.0;
        i64 s = srp[i];
        const i64 se = srp[i + 1];
        for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
            const i64 j = ci[k];
            while (s < se && sci[s] < j) ++s;
            if (j != i && s < se && sci[s] == j && !isc[j]) q += v[k] * inv != 0.0;
        }
        c1[fi] = q;
        c2[fi] = r.nfc;
    }
}

__global__ void k_mm_fill(i64 nf, const i64* __restrict__ fglob, const i64* __restrict__ floc,
                          const i64* __restrict__ rp, const i32* __restrict__ ci, const double* __restrict__ v,
                          const i64* __restrict__ srp, const i32* __restrict__ sci, const char* __restrict__ isc,
                          const i64* __restrict__ cidx, const double* __restrict__ inv1,
                          const double* __restrict__ inv2, const i64* __restrict__ m1rp, i32* __restrict__ m1ci,
                          double* __restrict__ m1v, const i64* __restrict__ m2rp, i32* __restrict__ m2ci,
                          double* __restrict__ m2v) {
    GRID_STRIDE(fi, nf) {
        const i64 i = fglob[fi];
        const double inv = inv1[fi], ib = inv2[fi];
        double beta = 0.0;
        i64 s = srp[i];
        const i64 se = srp[i + 1];
        for (i64 k = rp[i]; k < rp[i + 1]; ++k) { // beta again, in entry order
            const i64 j = ci[k];
            while (s < se && sci[s] < j) ++s;
            if (j != i && s < se && sci[s] == j && isc[j]) beta += v[k];
        }
        const double dval = beta * inv;
        bool dpending = dval != 0.0;
        i64 o1 = m1rp[fi], o2 = m2rp[fi];
        s = srp[i];
        for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
            const i64 j = ci[k];
            while (s < se && sci[s] < j) ++s;
            if (j == i || !(s < se && sci[s] == j)) continue;
            if (isc[j]) {
                m2ci[o2] = static_cast<i32>(cidx[j]);
                m2v[o2++] = v[k] * ib;
                continue;
            }
            const i64 fj = floc[j];
            if (dpending && fj > fi) { // the diagonal in column order
                m1ci[o1] = static_cast<i32>(fi);
                m1v[o1++] = dval;
                dpending = false;
            }
            const double w = v[k] * inv;
            if (w != 0.0) m1ci[o1] = static_cast<i32>(fj), m1v[o1++] = w;
        }
        if (dpending) m1ci[o1] = static_cast<i32>(fi), m1v[o1] = dval;
    }
}

// P: C rows the identity entry, F rows -W (beta != 0) or their direct weights
template <int PASS>
__global__ void k_mm_assemble(i64 n, const i64* __restrict__ floc, const double* __restrict__ inv2,
                              const i64* __restrict__ wrp, const i32* __restrict__ wci, const double* __restrict__ wv,
                              const i64* __restrict__ rp, const i32* __restrict__ ci, const double* __restrict__ v,
                              const i64* __restrict__ srp, const i32* __restrict__ sci, const char* __restrict__ isc,
                              const i64* __restrict__ cidx, i64* __restrict__ cnt, int* __restrict__ status,
                              unsigned long long* __restrict__ first_bad, const i64* __restrict__ prp,
                              i32* __restrict__ pci, double* __restrict__ pv) {
    GRID_STRIDE(i, n) {
        if (isc[i]) {
            if (PASS == 0)
                cnt[i] = 1;
            else
                pci[prp[i]] = static_cast<i32>(cidx[i]), pv[prp[i]] = 1.0;
            continue;
        }
        const i64 fi = floc[i];
        if (inv2[fi] == 0.0) { // fallback: direct weights
            if (PASS == 0) {
                const int code = direct_row<false>(i, rp, ci, v, srp, sci, isc, cidx, &cnt[i], nullptr, nullptr);
                status[i] = code;
                if (code) atomicMin(first_bad, static_cast<unsigned long long>(i));
            } else {
                direct_row<true>(i, rp, ci, v, srp, sci, isc, cidx, nullptr, pci + prp[i], pv + prp[i]);
            }
            continue;
        }
        if (PASS == 0) {
            cnt[i] = wrp[fi + 1] - wrp[fi];
        } else {
            i64 o = prp[i];
            for (i64 k = wrp[fi]; k < wrp[fi + 1]; ++k) pci[o] = wci[k], pv[o++] = -wv[k];
        }
    }
}

__global__ void k_not(i64 n, const char* __restrict__ isc, char* __restrict__ isf, i64* __restrict__ cnt) {
    GRID_STRIDE(i, n) {
        isf[i] = !isc[i];
        cnt[i] = !isc[i];
    }
}

// stable compaction of idx[0..m) by flags (cub::DeviceSelect keeps the order)
// ws: reusable CUB temporary + count slot (the PMIS rounds call this once per
// round; no allocation per call)
struct SelectWs {
    DBuf<i64> nsel{1};
    DBuf<unsigned char> t;
};
i64 select_flagged(const i64* in, const char* flags, i64* out, i64 m, cudaStream_t st, SelectWs* ws = nullptr) {
    if (m == 0) return 0;
    SelectWs local;
    SelectWs& w = ws ? *ws : local;
    DBuf<i64>& nsel = w.nsel;
    size_t tmp = 0;
    ILUG_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, in, flags, out, nsel.p, m, st));
    if (w.t.n < static_cast<i64>(tmp) + 1) w.t.alloc(static_cast<i64>(tmp) + 1);
    DBuf<unsigned char>& t = w.t;
    ILUG_CUDA(cub::DeviceSelect::Flagged(t.p, tmp, in, flags, out, nsel.p, m, st));
    i64 h = 0;
    ILUG_CUDA(cudaMemcpyAsync(&h, nsel.p, sizeof h, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    return h;
}

__global__ void k_iota(i64 n, i64* __restrict__ a) {
    GRID_STRIDE(i, n) a[i] = i;
}

} // namespace

DevCsr strength_device(const DevCsr& A, double theta, cudaStream_t st) {
    const i64 n = A.nrows;
    DevCsr S;
    S.nrows = n;
    S.ncols = A.ncols;
    DBuf<double> cut(std::max<i64>(n, 1));
    DBuf<i64> cnt(std::max<i64>(n, 1));
    k_strength_count<<<grid_n(n), kB, 0, st>>>(n, A.rp.p, A.ci.p, A.v.p, theta, cut.p, cnt.p);
    ILUG_LAUNCH_CHECK();
    S.rp.alloc(n + 1);
    const i64 nnz = scan_counts(cnt.p, S.rp.p, n, st);
    S.ci.alloc(nnz);
    k_strength_fill<<<grid_n(n), kB, 0, st>>>(n, A.rp.p, A.ci.p, A.v.p, cut.p, S.rp.p, S.ci.p);
    ILUG_LAUNCH_CHECK();
    return S;
}

DevCsr transpose_device(const DevCsr& M, bool values, cudaStream_t st) {
    const i64 n = M.nrows, m = M.ncols, nnz = M.ci.n;
    DevCsr T;
    T.nrows = m;
    T.ncols = n;
    DBuf<unsigned long long> cnt(std::max<i64>(m, 1));
    ILUG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * std::max<i64>(m, 1), st));
    k_col_count<<<grid_n(nnz), kB, 0, st>>>(nnz, M.ci.p, cnt.p);
    ILUG_LAUNCH_CHECK();
    T.rp.alloc(m + 1);
    scan_counts(reinterpret_cast<const i64*>(cnt.p), T.rp.p, m, st);
    DBuf<i32> row(std::max<i64>(nnz, 1));
    k_row_of<<<grid_n(n), kB, 0, st>>>(n, M.rp.p, row.p);
    ILUG_LAUNCH_CHECK();
    ILUG_CUDA(cudaMemcpyAsync(cnt.p, T.rp.p, sizeof(i64) * std::max<i64>(m, 1), cudaMemcpyDeviceToDevice, st));
    T.ci.alloc(nnz);
    if (values) T.v.alloc(nnz);
    k_scatter_t<<<grid_n(nnz), kB, 0, st>>>(nnz, row.p, M.ci.p, values ? M.v.p : nullptr, cnt.p, T.ci.p,
                                            values ? T.v.p : nullptr);
    ILUG_LAUNCH_CHECK();
    k_sort_rows<<<grid_n(m), kB, 0, st>>>(m, T.rp.p, T.ci.p, values ? T.v.p : nullptr);
    ILUG_LAUNCH_CHECK();
    return T;
}

DevSplit pmis_device(const DevCsr& S, const DevCsr& St, std::uint64_t seed, cudaStream_t st) {
    const i64 n = S.nrows;
    DevSplit sp;
    DBuf<double> wt(std::max<i64>(n, 1));
    DBuf<char> state(std::max<i64>(n, 1)), fresh(std::max<i64>(n, 1)), picked(std::max<i64>(n, 1)),
        keep(std::max<i64>(n, 1));
    DBuf<i64> live(std::max<i64>(n, 1)), next(std::max<i64>(n, 1));
    DBuf<unsigned long long> found(1);
    SelectWs sws;
    ILUG_CUDA(cudaMemsetAsync(fresh.p, 0, static_cast<size_t>(std::max<i64>(n, 1)), st));
    k_pmis_init<<<grid_n(n), kB, 0, st>>>(n, St.rp.p, seed, wt.p, state.p, live.p);
    ILUG_LAUNCH_CHECK();
    i64 m = n;
    while (m > 0) {
        ILUG_CUDA(cudaMemsetAsync(found.p, 0, sizeof(unsigned long long), st));
        k_pmis_pick<<<grid_n(m), kB, 0, st>>>(m, live.p, S.rp.p, S.ci.p, St.rp.p, St.ci.p, wt.p, state.p, picked.p,
                                              found.p);
        ILUG_LAUNCH_CHECK();
        unsigned long long f = 0;
        ILUG_CUDA(cudaMemcpyAsync(&f, found.p, sizeof f, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        if (f == 0) { // no local maximum: the smallest free index (live stays ascending)
            ILUG_CUDA(cudaMemsetAsync(picked.p, 0, static_cast<size_t>(m), st));
            const char one = 1;
            ILUG_CUDA(cudaMemcpyAsync(picked.p, &one, 1, cudaMemcpyHostToDevice, st));
        }
        k_pmis_mark<<<grid_n(m), kB, 0, st>>>(m, live.p, picked.p, state.p, fresh.p, 1);
        ILUG_LAUNCH_CHECK();
        k_pmis_fpass<<<grid_n(m), kB, 0, st>>>(m, live.p, S.rp.p, S.ci.p, fresh.p, state.p, keep.p);
        ILUG_LAUNCH_CHECK();
        k_pmis_mark<<<grid_n(m), kB, 0, st>>>(m, live.p, picked.p, state.p, fresh.p, 0);
        ILUG_LAUNCH_CHECK();
        m = select_flagged(live.p, keep.p, next.p, m, st, &sws);
        std::swap(live, next);
    }
    // repair pass (src/amg.cpp:56-84): parallel candidate search, serial ordered promotion
    DBuf<char> cand(std::max<i64>(n, 1));
    k_lacks_c<<<grid_n(n), kB, 0, st>>>(n, S.rp.p, S.ci.p, state.p, cand.p);
    ILUG_LAUNCH_CHECK();
    k_iota<<<grid_n(n), kB, 0, st>>>(n, live.p);
    ILUG_LAUNCH_CHECK();
    const i64 nc = select_flagged(live.p, cand.p, next.p, n, st, &sws);
    if (nc > 0) {
        k_repair<<<1, 32, 0, st>>>(nc, next.p, S.rp.p, S.ci.p, state.p);
        ILUG_LAUNCH_CHECK();
    }
    sp.is_coarse.alloc(std::max<i64>(n, 1));
    sp.coarse_index.alloc(std::max<i64>(n, 1));
    DBuf<i64> flag(std::max<i64>(n, 1)), pre(n + 1);
    k_is_coarse<<<grid_n(n), kB, 0, st>>>(n, state.p, flag.p, sp.is_coarse.p);
    ILUG_LAUNCH_CHECK();
    sp.n_coarse = scan_counts(flag.p, pre.p, n, st);
    k_coarse_index<<<grid_n(n), kB, 0, st>>>(n, sp.is_coarse.p, pre.p, sp.coarse_index.p);
    ILUG_LAUNCH_CHECK();
    sp.n = n;
    return sp;
}

DevCsr interp_direct_device(const DevCsr& A, const DevCsr& S, const DevSplit& sp, cudaStream_t st) {
    const i64 n = A.nrows;
    DevCsr P;
    P.nrows = n;
    P.ncols = sp.n_coarse;
    DBuf<i64> cnt(std::max<i64>(n, 1));
    DBuf<int> status(std::max<i64>(n, 1));
    DBuf<unsigned long long> bad(1);
    const unsigned long long none = ~0ull;
    ILUG_CUDA(cudaMemcpyAsync(bad.p, &none, sizeof none, cudaMemcpyHostToDevice, st));
    k_interp<0><<<grid_n(n), kB, 0, st>>>(n, A.rp.p, A.ci.p, A.v.p, S.rp.p, S.ci.p, sp.is_coarse.p,
                                          sp.coarse_index.p, cnt.p, status.p, bad.p, nullptr, nullptr, nullptr);
    ILUG_LAUNCH_CHECK();
    unsigned long long b = none;
    ILUG_CUDA(cudaMemcpyAsync(&b, bad.p, sizeof b, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    if (b != none) {
        int code = 0;
        ILUG_CUDA(cudaMemcpy(&code, status.p + b, sizeof code, cudaMemcpyDeviceToHost));
        if (code == 1)
            fail_invalid("interp_direct: F-point " + std::to_string(b) +
                         " has no strong C-neighbor (coarsening repair failed)");
        fail_numeric("interp_direct: zero denominator at row " + std::to_string(b));
    }
    P.rp.alloc(n + 1);
    const i64 nnz = scan_counts(cnt.p, P.rp.p, n, st);
    P.ci.alloc(nnz);
    P.v.alloc(nnz);
    k_interp<1><<<grid_n(n), kB, 0, st>>>(n, A.rp.p, A.ci.p, A.v.p, S.rp.p, S.ci.p, sp.is_coarse.p,
                                          sp.coarse_index.p, nullptr, nullptr, nullptr, P.rp.p, P.ci.p, P.v.p);
    ILUG_LAUNCH_CHECK();
    return P;
}

DevCsr interp_mm_ext_device(const DevCsr& A, const DevCsr& S, const DevSplit& sp, i64* fallback_rows,
                            cudaStream_t st) {
    const i64 n = A.nrows, nc = sp.n_coarse;
    const i64 n1 = std::max<i64>(n, 1);
    // F numbering: floc = exclusive scan of the F flags, fglob = the F rows ascending
    DBuf<char> isf(n1);
    DBuf<i64> fcnt(n1), floc(n + 1), idx(n1), fglob(n1);
    k_not<<<grid_n(n), kB, 0, st>>>(n, sp.is_coarse.p, isf.p, fcnt.p);
    ILUG_LAUNCH_CHECK();
    const i64 nf = scan_counts(fcnt.p, floc.p, n, st);
    k_iota<<<grid_n(n), kB, 0, st>>>(n, idx.p);
    ILUG_LAUNCH_CHECK();
    select_flagged(idx.p, isf.p, fglob.p, n, st);
    const i64 nf1 = std::max<i64>(nf, 1);
    DBuf<double> inv1(nf1), inv2(nf1);
    DBuf<i64> c1(nf1), c2(nf1);
    DBuf<unsigned long long> flags(2); // [0] first singular F-row, [1] fallback rows
    const unsigned long long init[2] = {~0ull, 0ull};
    ILUG_CUDA(cudaMemcpyAsync(flags.p, init, sizeof init, cudaMemcpyHostToDevice, st));
    k_mm_count<<<grid_n(nf), kB, 0, st>>>(nf, fglob.p, A.rp.p, A.ci.p, A.v.p, S.rp.p, S.ci.p, sp.is_coarse.p,
                                           inv1.p, inv2.p, c1.p, c2.p, flags.p, flags.p + 1);
    ILUG_LAUNCH_CHECK();
    unsigned long long fl[2] = {0, 0};
    ILUG_CUDA(cudaMemcpyAsync(fl, flags.p, sizeof fl, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    if (fl[0] != ~0ull) {
        i64 row = 0;
        ILUG_CUDA(cudaMemcpy(&row, fglob.p + fl[0], sizeof row, cudaMemcpyDeviceToHost));
        fail_numeric("interp_mm_ext: singular D_FF + D_gamma at F-row " + std::to_string(row));
    }
    if (fallback_rows) *fallback_rows = static_cast<i64>(fl[1]);
    DevCsr M1, M2, W;
    M1.nrows = nf, M1.ncols = nf;
    M2.nrows = nf, M2.ncols = nc;
    M1.rp.alloc(nf + 1);
    M2.rp.alloc(nf + 1);
    M1.ci.alloc(scan_counts(c1.p, M1.rp.p, nf, st));
    M1.v.alloc(M1.ci.n);
    M2.ci.alloc(scan_counts(c2.p, M2.rp.p, nf, st));
    M2.v.alloc(M2.ci.n);
    k_mm_fill<<<grid_n(nf), kB, 0, st>>>(nf, fglob.p, floc.p, A.rp.p, A.ci.p, A.v.p, S.rp.p, S.ci.p, sp.is_coarse.p,
                                          sp.coarse_index.p, inv1.p, inv2.p, M1.rp.p, M1.ci.p, M1.v.p, M2.rp.p,
                                          M2.ci.p, M2.v.p);
    ILUG_LAUNCH_CHECK();
    if (!spgemm_device(nf, nc, M1, M2, W, st)) // a row too wide for the tables: the host product
        W.upload(csr_matmul(M1.download(st), M2.download(st)), st);
    M1 = DevCsr{};
    M2 = DevCsr{};
    DevCsr P;
    P.nrows = n;
    P.ncols = nc;
    DBuf<i64> cnt(n1);
    DBuf<int> status(n1);
    const unsigned long long none = ~0ull;
    ILUG_CUDA(cudaMemcpyAsync(flags.p, &none, sizeof none, cudaMemcpyHostToDevice, st));
    k_mm_assemble<0><<<grid_n(n), kB, 0, st>>>(n, floc.p, inv2.p, W.rp.p, W.ci.p, W.v.p, A.rp.p, A.ci.p, A.v.p,
                                                S.rp.p, S.ci.p, sp.is_coarse.p, sp.coarse_index.p, cnt.p, status.p,
                                                flags.p, nullptr, nullptr, nullptr);
    ILUG_LAUNCH_CHECK();
    unsigned long long b = none;
    ILUG_CUDA(cudaMemcpyAsync(&b, flags.p, sizeof b, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    if (b != none) {
        int code = 0;
        ILUG_CUDA(cudaMemcpy(&code, status.p + b, sizeof code, cudaMemcpyDeviceToHost));
        if (code == 1)
            fail_invalid("interp_direct: F-point " + std::to_string(b) +
                         " has no strong C-neighbor (coarsening repair failed)");
        fail_numeric("interp_direct: zero denominator at row " + std::to_string(b));
    }
    P.rp.alloc(n + 1);
    P.ci.alloc(scan_counts(cnt.p, P.rp.p, n, st));
    P.v.alloc(P.ci.n);
    k_mm_assemble<1><<<grid_n(n), kB, 0, st>>>(n, floc.p, inv2.p, W.rp.p, W.ci.p, W.v.p, A.rp.p, A.ci.p, A.v.p,
                                                S.rp.p, S.ci.p, sp.is_coarse.p, sp.coarse_index.p, nullptr, nullptr,
                                                nullptr, P.rp.p, P.ci.p, P.v.p);
    ILUG_LAUNCH_CHECK();
    return P;
}

bool amg_device_supported(const AmgParams& p) { return p.coarsening == Coarsening::pmis; }

HostHierarchy amg_setup_device(const Csr& A, const AmgParams& prm, const LevelReady& on_level, cudaStream_t st,
                               const DevCsr* Ad, bool keep_device) {
    if (A.nrows != A.ncols) fail_invalid("setup: matrix must be square");
    if (!(prm.theta > 0.0 && prm.theta <= 1.0)) fail_invalid("setup: theta must lie in (0, 1]");
    if (prm.coarse_size < 1) fail_invalid("setup: coarse_size must be >= 1");
    if (prm.max_levels < 1) fail_invalid("setup: max_levels must be >= 1");
    if (prm.cycles_nu < 1) fail_invalid("setup: cycles_nu must be >= 1");
    if (!amg_device_supported(prm)) fail_invalid("device AMG setup: PMIS coarsening only");
    HostHierarchy h;
    h.params = prm;
    h.levels.reserve(static_cast<size_t>(prm.max_levels)); // stable level addresses for on_level
    SetupTimer tm("amg-device");
    auto own = std::make_shared<DevCsr>();
    if (!Ad) own->upload(A, st);
    tm.mark("upload A");
    const DevCsr* curp = Ad ? Ad : own.get(); // level k's operator on the device
    keep_device = keep_device && on_level;
    // Each level's host copy of A (GBs at the fine levels: a host copy at
    // level 0, a download from its own stream below it) overlaps the level's
    // GPU work; joined before anything reads it and before the device copy
    // can change.
    cudaStream_t dl = nullptr;
    ILUG_CUDA(cudaStreamCreateWithFlags(&dl, cudaStreamNonBlocking));
    struct StreamDel {
        cudaStream_t s;
        ~StreamDel() { cudaStreamDestroy(s); }
    } dl_guard{dl};
    std::future<Csr> a0 = std::async(std::launch::async, [&A] { return csr_copy(A); });
    HostLevel* a0_lev = nullptr;
    auto join_a0 = [&] {
        if (a0.valid()) a0_lev->A = a0.get();
    };
    for (;;) {
        h.levels.emplace_back();
        HostLevel& lev = h.levels.back();
        const i64 k = h.num_levels() - 1;
        if (k > 0) { // the device A_k is complete (the previous level synchronised st)
            const DevCsr* src = curp;
            a0 = std::async(std::launch::async, [src, dl] { return src->download(dl); });
        }
        a0_lev = &lev;
        tm.mark("host A", k);
        const i64 nk = curp->nrows;
        if (nk <= prm.coarse_size || k + 1 >= prm.max_levels) break;
        const DevCsr& cur = *curp;
        DevCsr S = strength_device(cur, prm.theta, st);
        DevCsr St = transpose_device(S, false, st);
        tm.mark("strength", k);
        DevSplit sp = pmis_device(S, St, prm.pmis_seed, st);
        tm.mark("pmis", k);
        if (static_cast<double>(sp.n_coarse) > 0.95 * static_cast<double>(nk)) break;
        St = DevCsr{};
        DevCsr P = prm.interpolation == Interpolation::mm_ext
                       ? interp_mm_ext_device(cur, S, sp, &lev.mm_ext_fallback_rows, st)
                       : interp_direct_device(cur, S, sp, st);
        S = DevCsr{};
        DevCsr R = transpose_device(P, true, st);
        tm.mark("interp+transpose", k);
        DevCsr AP, C;
        const bool ok = spgemm_device(cur.nrows, P.ncols, cur, P, AP, st) &&
                        spgemm_device(R.nrows, P.ncols, R, AP, C, st);
        tm.mark("R*(A*P)", k);
        if (!keep_device || !ok) { // the consumer of keep_device builds from the device copies
            lev.P = P.download(st);
            lev.R = R.download(st);
        } else {
            lev.P.nrows = P.nrows, lev.P.ncols = P.ncols;
            lev.R.nrows = R.nrows, lev.R.ncols = R.ncols;
        }
        if (!ok) { // a row too wide for the tables
            join_a0();
            C.upload(csr_matmul(lev.R, csr_matmul(lev.A, lev.P)), st);
        }
        lev.split.n_coarse = sp.n_coarse;
        if (!keep_device) { // (the device-hierarchy consumer never reads the C/F split)
            lev.split.is_coarse.resize(static_cast<size_t>(sp.n));
            lev.split.coarse_index.resize(static_cast<size_t>(sp.n));
        }
        if (sp.n > 0 && !keep_device) {
            sp.is_coarse.download(lev.split.is_coarse.data(), st);
            sp.coarse_index.download(lev.split.coarse_index.data(), st);
        }
        ILUG_CUDA(cudaStreamSynchronize(st));
        tm.mark("download P,R", k);
        if (keep_device) {
            if (curp == own.get()) lev.dA = own;
            lev.dP = std::make_shared<DevCsr>(std::move(P));
            lev.dR = std::make_shared<DevCsr>(std::move(R));
        }
        join_a0();
        if (on_level) on_level(k, lev, false);
        own = std::make_shared<DevCsr>(std::move(C));
        curp = own.get();
    }
    join_a0();
    if (on_level) on_level(h.num_levels() - 1, h.levels.back(), true);
    h.coarse = dense_lu_factor(h.levels.back().A);
    return h;
}

} // namespace ilug
