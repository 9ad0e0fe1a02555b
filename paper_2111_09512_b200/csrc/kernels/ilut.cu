// ILUT(droptol, lfill) on the device, bitwise equal to
// the reference's dual-threshold ILUT (src/ilu.cpp:120-265) and to host/ilu.cpp.
//
// One warp per row, rows taken in ascending order from an atomic ticket by a
// persistent grid, so a row only ever waits on rows claimed before it (no
// deadlock whatever the residency). The working row w lives in the warp's
// shared memory as a column-sorted list (col, value, flags). The reference's
// min-heap of pending lower columns is exactly an ascending scan of that list:
// fill from U row k only adds columns > k, so it lands behind the scan point.
// Per multiplier k (ascending):
//   wait for done[k] (epoch-stamped, acquire), m = w_k / u_kk, drop if
//   |m| < tau, else every lane takes entries of U row k, binary-searches its
//   column in the list (update w_j -= m*u_kj in place) or marks it new; new
//   entries are merged by shifting the tail from the back, chunk by chunk.
// Each w_j receives the serial algorithm's updates in the same order (k
// ascending), with separate multiply/subtract (--fmad=false), so every value
// is bitwise the reference's. Survivor selection follows src/ilu.cpp:190-219:
// U part on |w| >= tau, pattern entries kept, fill ranked by (|w| desc,
// column asc) for lfill slots; L part = kept multipliers with the same fill
// cap. The U row is published (done[i], release) before the L part is
// selected, since only U rows are on the row-to-row chain.
//
// Working rows longer than the shared-memory capacity set an overflow flag;
// every remaining row then publishes immediately and the host relaunches with
// a larger capacity (fewer warps per CTA). A bounded spin turns a scheduling
// bug into an error instead of a hung GPU.
#include "ilu0.hpp"
#include "spgemm.hpp"

#include <cub/device/device_scan.cuh>
#include <cuda/atomic>

#include <cfloat>
#include <climits>
#include <cstdlib>

namespace ilug {

namespace {

constexpr unsigned char kLive = 1, kOrig = 2, kKept = 4, kSel = 8, kDrop = 16;

struct IlutArgs {
    i64 n;
    const i64* rp;
    const i32* ci;
    const double* av;
    const double* tau;   // droptol * |a_i|_2 per row
    i64 lfill;
    double anorm_f;
    int patch;           // 0 error, 1 replace
    double droptol;
    const i64* uoff;     // U slot of row i: [uoff[i], uoff[i+1])
    const i64* loff;
    i32* uci;
    double* uv;
    i32* ulen;
    i32* lci;
    double* lv;
    i32* llen;
    unsigned* done;
    const unsigned* epoch;
    unsigned long long* ticket;
    unsigned long long* first_zero;
    unsigned* err;       // [0] wait timeout, [1] overflow (needed capacity)
    int wrank;           // fill ranking in registers when <= 32 candidates (ILUG_ILUT_WRANK)
    unsigned backoff_ns; // longest poll back-off (ILUG_ILUT_BACKOFF)
    int quota;           // rows a warp takes before its CTA may retire (ILUG_ILUT_QUOTA)
    int chunk;           // consecutive rows per ticket (ILUG_ILUT_CHUNK)
};

// Dependency wait with exponential back-off (32 ns doubling up to max_ns):
// ~95 % of the kernel's executed instructions were polls at a fixed 32 ns,
// issue slots the working warps of the same SM then lack (ncu, C2 128^3).
__device__ __forceinline__ bool wait_flag_backoff(const unsigned* p, unsigned E, unsigned max_ns) {
    if (ld_acquire_flag(p) == E) return true;
    long long spins = 0;
    unsigned ns = max_ns < 32 ? max_ns : 32;
    while (ld_relaxed_flag(p) != E) {
        if (++spins > (1ll << 26)) return false;
        if (ns) __nanosleep(ns);
        ns = ns < max_ns ? ns * 2 : max_ns;
    }
    (void)ld_acquire_flag(p); // synchronises with the producer's release store
    return true;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Value-flag publication of U rows (VF): the row's slot starts filled with
// sentinels (column -1, value = a signalling NaN no arithmetic produces,
// length 0); the producer writes entries, pivot and length with relaxed .gpu
// stores and a consumer validates every word it uses, so the data IS the
// flag — one memory round trip per dependency step instead of a flag poll, an
// acquire and a second fetch.
constexpr unsigned long long kUSentinel = 0x7FF0DEAD5EA1ED01ull;
__device__ __forceinline__ unsigned long long ldr_u64(const double* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ldr_s32(const i32* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void str_f64(double* p, double x) {
    unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    if (b == kUSentinel) b = 0x7FFFFFFFFFFFFFFFull; // never publish the sentinel itself
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(b) : "memory");
}
__device__ __forceinline__ void str_s32(i32* p, int x) {
    asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(x) : "memory");
}
__global__ void k_ilut_vf_fill(i64 ucap, i64 n, i32* __restrict__ uci, double* __restrict__ uv, i32* __restrict__ ulen) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < ucap;
         i += static_cast<i64>(gridDim.x) * blockDim.x) {
        uci[i] = -1;
        reinterpret_cast<unsigned long long*>(uv)[i] = kUSentinel;
        if (i < n) ulen[i] = 0;
    }
}

// A lane group of G lanes (G = 32: the warp; G = 16: each half-warp works
// on its own row): group-relative shuffles, ballots, masks and sync.
template <int G>
struct Grp {
    unsigned mask;
    int lane, shift;
    __device__ __forceinline__ Grp() {
        const int l = static_cast<int>(threadIdx.x & 31);
        lane = l & (G - 1);
        shift = l & ~(G - 1);
        mask = G == 32 ? 0xffffffffu : (((1u << (G & 31)) - 1u) << shift);
    }
    __device__ __forceinline__ unsigned ballot(bool p) const {
        const unsigned b = __ballot_sync(mask, p);
        return G == 32 ? b : (b >> shift) & ((1u << (G & 31)) - 1u);
    }
    template <class T>
    __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(mask, v, src, G); }
    __device__ __forceinline__ bool all(bool p) const { return __all_sync(mask, p); }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
    __device__ __forceinline__ unsigned lt() const { return (1u << lane) - 1u; } // lanes below, group-relative
    __device__ __forceinline__ int sum(int x) const {
        for (int o = G / 2; o; o >>= 1) x += __shfl_xor_sync(mask, x, o, G);
        return x;
    }
};
// the whole warp: every mask a constant, lanemask_lt from the special register
template <>
struct Grp<32> {
    static constexpr unsigned mask = 0xffffffffu;
    int lane;
    __device__ __forceinline__ Grp() : lane(static_cast<int>(threadIdx.x & 31)) {}
    __device__ __forceinline__ unsigned ballot(bool p) const { return __ballot_sync(mask, p); }
    template <class T>
    __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(mask, v, src); }
    __device__ __forceinline__ bool all(bool p) const { return __all_sync(mask, p); }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
    __device__ __forceinline__ unsigned lt() const { return lanemask_lt(); }
    __device__ __forceinline__ int sum(int x) const {
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(mask, x, o);
        return x;
    }
};

// Rank fill candidates in [beg, end) that carry `want` and not kOrig: keep the
// lfill best by (|w| desc, column asc) (the reference's nth_element comparator,
// src/ilu.cpp:206-211). Pattern candidates are always kept. Marks kSel.
template <int G>
__device__ __forceinline__ void select_part(const i32* scol, const double* sval, unsigned char* sflag, int beg,
                                            int end, unsigned char want, bool upper, double tau, i64 lfill,
                                            const Grp<G>& gr, bool wrank) {
    // pass 1: which candidates pass (U part: the threshold), count fill
    int nfill = 0;
    for (int q = beg + gr.lane; q < end; q += G) {
        unsigned char f = sflag[q];
        bool pass = (f & want) && !(upper && fabs(sval[q]) < tau);
        if (pass) {
            f |= kSel;
            if (!(f & kOrig)) ++nfill;
        } else {
            f &= static_cast<unsigned char>(~kSel);
        }
        sflag[q] = f;
    }
    nfill = gr.sum(nfill);
    gr.sync();
    if (nfill <= lfill) return;
    if (wrank && nfill <= G) {
        // pass 2 in registers: the fill candidates compacted into lanes
        // 0..nfill-1 (ballot + nth-set-bit shuffles), each lane ranks its
        // candidate against the others by shuffles — the same comparator, so
        // the same survivors as the shared-memory ranking below. (A two-slot
        // form for up to 64 candidates spilled at the 42-register budget and
        // measured slower: 1.44 vs 1.33 s at C2.)
        double myv = 0.0;
        i32 myc = 0;
        int myq = -1, base = 0;
        for (int q0 = beg; q0 < end; q0 += G) {
            const int q = q0 + gr.lane;
            bool cand = false;
            double v = 0.0;
            i32 c = 0;
            if (q < end) {
                const unsigned char f = sflag[q];
                cand = (f & kSel) && !(f & kOrig);
                v = fabs(sval[q]);
                c = scol[q];
            }
            const unsigned bm = gr.ballot(cand);
            const int cnt = __popc(bm);
            const int k = gr.lane - base; // this lane takes the chunk's k-th candidate
            const int src = (k >= 0 && k < cnt) ? static_cast<int>(__fns(bm, 0, k + 1)) : 0;
            const double sv = gr.shfl(v, src);
            const i32 sc = gr.shfl(c, src);
            if (k >= 0 && k < cnt) myv = sv, myc = sc, myq = q0 + src;
            base += cnt;
        }
        i64 rank = 0;
        for (int r = 0; r < nfill; ++r) {
            const double vr = gr.shfl(myv, r);
            const i32 cr = gr.shfl(myc, r);
            if (r != gr.lane) rank += (vr != myv) ? (vr > myv) : (cr < myc);
        }
        if (myq >= 0 && rank >= lfill) sflag[myq] = static_cast<unsigned char>(sflag[myq] & ~kSel);
        gr.sync();
        return;
    }
    // pass 2: rank each fill candidate against all others; losers get kDrop
    // (the ranking reads only kSel/kOrig, so marking while others rank is safe)
    for (int q = beg + gr.lane; q < end; q += G) {
        const unsigned char f = sflag[q];
        if (!(f & kSel) || (f & kOrig)) continue;
        const double vq = fabs(sval[q]);
        const i32 cq = scol[q];
        i64 rank = 0;
        for (int r = beg; r < end; ++r) {
            const unsigned char g = sflag[r];
            if (!(g & kSel) || (g & kOrig) || r == q) continue;
            const double vr = fabs(sval[r]);
            rank += (vr != vq) ? (vr > vq) : (scol[r] < cq);
        }
        if (rank >= lfill) sflag[q] = f | kDrop;
    }
    gr.sync();
    for (int q = beg + gr.lane; q < end; q += G) {
        const unsigned char f = sflag[q];
        if (f & kDrop) sflag[q] = static_cast<unsigned char>(f & ~(kSel | kDrop));
    }
    gr.sync();
}

// Write the kSel entries of [beg, end) (ascending columns) to out_c/out_v; returns the count.
template <bool VF, int G>
__device__ __forceinline__ int emit(const i32* scol, const double* sval, const unsigned char* sflag, int beg,
                                    int end, i32* out_c, double* out_v, const Grp<G>& gr) {
    int base = 0;
    for (int q0 = beg; q0 < end; q0 += G) {
        const int q = q0 + gr.lane;
        const bool s = q < end && (sflag[q] & kSel);
        const unsigned b = gr.ballot(s);
        if (s) {
            const int o = base + __popc(b & gr.lt());
            if (VF) {
                str_s32(out_c + o, scol[q]);
                str_f64(out_v + o, sval[q]);
            } else {
                out_c[o] = scol[q];
                out_v[o] = sval[q];
            }
        }
        base += __popc(b);
    }
    return base;
}

template <int CAP, int WARPS, bool VF, int G>
__global__ void __launch_bounds__(WARPS * 32, 48 / WARPS) k_ilut(IlutArgs a) {
    extern __shared__ double smem[];
    // NS row slots per CTA: one per lane group (G = 32: per warp)
    constexpr int NS = WARPS * (32 / G);
    const Grp<G> gr;
    const int slot = static_cast<int>(threadIdx.x) / G, lane = gr.lane;
    // [NS*CAP values][NS*CAP columns][NS*G merge positions][NS*CAP flags]
    i32* const col_base = reinterpret_cast<i32*>(smem + static_cast<size_t>(NS) * CAP);
    double* const sval = smem + static_cast<size_t>(slot) * CAP;
    i32* const scol = col_base + static_cast<size_t>(slot) * CAP;
    i32* const snew = col_base + static_cast<size_t>(NS) * CAP + slot * G;
    unsigned char* const sflag = reinterpret_cast<unsigned char*>(col_base + static_cast<size_t>(NS) * CAP +
                                                                  NS * G) + static_cast<size_t>(slot) * CAP;
    const unsigned E = *a.epoch;

    // Rows are claimed in chunks of a.chunk consecutive rows: a line of the
    // grid then advances inside one warp (row i's dependency on row i-1 is its
    // own last row, no cross-SM flag round trip) and the claimed-but-waiting
    // window covers a.chunk times more lines. A started chunk is always
    // finished (its rows are claimed), whatever the quota says.
    i64 next = 0, cend = 0;
    for (int q = a.quota; q > 0 || next < cend; --q) {
        if (next >= cend) {
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(a.ticket, static_cast<unsigned long long>(a.chunk));
            next = static_cast<i64>(gr.shfl(t, 0));
            if (next >= a.n) return;
            cend = next + a.chunk < a.n ? next + a.chunk : a.n;
        }
        const i64 i = next++;
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> fi(a.done[i]);
        const i64 beg = a.rp[i];
        const int alen = static_cast<int>(a.rp[i + 1] - beg);
        unsigned ov = 0;
        if (lane == 0) ov = *reinterpret_cast<volatile unsigned*>(a.err + 1);
        bool bad = gr.shfl(ov, 0) != 0u;
        if (!bad && alen > CAP) {
            if (lane == 0) atomicMax(a.err + 1, static_cast<unsigned>(alen));
            bad = true;
        }
        if (bad) { // capacity exceeded somewhere: publish and let the host relaunch
            gr.sync();
            if (lane == 0) {
                if (VF) { // a valid (meaningless) one-entry row: consumers must not wait
                    const i64 uo = a.uoff[i];
                    str_s32(a.uci + uo, static_cast<i32>(i));
                    str_f64(a.uv + uo, 1.0);
                    str_s32(a.ulen + i, 1);
                } else {
                    fi.store(E, cuda::memory_order_release);
                }
            }
            continue;
        }
        for (int q = lane; q < alen; q += G) {
            scol[q] = a.ci[beg + q];
            sval[q] = a.av[beg + q];
            sflag[q] = kLive | kOrig;
        }
        int len = alen;
        const double tau = a.tau[i];
        gr.sync();

        int p = 0;
        for (; p < len && !bad; ++p) {
            const i32 k = scol[p];
            if (k >= i) break;
            // the slot of U row k is fixed before row k is done: address its
            // first 32 entries ahead, then fetch length, pivot and entries in
            // one round trip once the flag is seen (slot entries past the
            // length are never used)
            const i64 ub = __ldg(a.uoff + k);
            const bool in_slot = lane + 1 < __ldg(a.uoff + k + 1) - ub;
            int ul;
            double ukk, u0;
            i32 j0;
            if (VF) { // length, pivot and the first 32 entries validated word by word
                long long spins = 0;
                for (;;) {
                    ul = ldr_s32(a.ulen + k);
                    const unsigned long long pb = ldr_u64(a.uv + ub);
                    const i32 jj = in_slot ? ldr_s32(a.uci + ub + 1 + lane) : INT_MAX;
                    const unsigned long long vb = in_slot ? ldr_u64(a.uv + ub + 1 + lane) : 0ull;
                    const bool need = lane + 1 < ul;
                    const bool ok = ul > 0 && pb != kUSentinel && (!need || (jj >= 0 && vb != kUSentinel));
                    if (gr.all(ok)) {
                        ukk = __longlong_as_double(static_cast<long long>(pb));
                        j0 = jj;
                        u0 = __longlong_as_double(static_cast<long long>(vb));
                        break;
                    }
                    if (++spins > (1ll << 26)) {
                        if (lane == 0) atomicExch(a.err, 1u);
                        ul = 1, ukk = 1.0, j0 = INT_MAX, u0 = 0.0;
                        break;
                    }
                    __nanosleep(20);
                }
            } else {
                if (!wait_flag_backoff(a.done + k, E, a.backoff_ns)) atomicExch(a.err, 1u);
                ul = a.ulen[k];
                ukk = a.uv[ub];
                j0 = in_slot ? a.uci[ub + 1 + lane] : INT_MAX;
                u0 = in_slot ? a.uv[ub + 1 + lane] : 0.0;
            }
            const double m = sval[p] / ukk;
            gr.sync();
            if (fabs(m) < tau) { // dual-threshold drop of the multiplier
                if (lane == 0) sval[p] = 0.0, sflag[p] = 0;
                gr.sync();
                continue;
            }
            if (lane == 0) sval[p] = m, sflag[p] = kLive | kKept | (sflag[p] & kOrig);
            for (int c = 1; c < ul; c += G) {
                const int kk = c + lane;
                const bool act = kk < ul;
                i32 j = !act ? INT_MAX : (c == 1 ? j0 : a.uci[ub + kk]);
                double u = !act ? 0.0 : (c == 1 ? u0 : a.uv[ub + kk]);
                if (VF && act && c > 1) { // entries past the first 32: validated one by one
                    for (;;) {
                        j = ldr_s32(a.uci + ub + kk);
                        const unsigned long long vb = ldr_u64(a.uv + ub + kk);
                        if (j >= 0 && vb != kUSentinel) {
                            u = __longlong_as_double(static_cast<long long>(vb));
                            break;
                        }
                        __nanosleep(20);
                    }
                }
                int lo = p + 1, hi = len;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (scol[mid] < j) lo = mid + 1;
                    else hi = mid;
                }
                const bool found = act && lo < len && scol[lo] == j;
                const double prod = m * u;
                if (found) sval[lo] = sval[lo] - prod;
                const unsigned nm = gr.ballot(act && !found);
                if (nm == 0u) {
                    gr.sync();
                    continue;
                }
                const int nnew = __popc(nm);
                if (len + nnew > CAP) {
                    if (lane == 0) atomicMax(a.err + 1, static_cast<unsigned>(len + nnew));
                    bad = true;
                    break;
                }
                const int rank = __popc(nm & gr.lt());
                if (act && !found) snew[rank] = lo;
                gr.sync();
                const int minpos = snew[0];
                // shift the tail [minpos, len) up by the number of new entries before
                // each element, from the back (destinations never reach unread slots)
                for (int top = len; top > minpos; top -= G) {
                    const int q = top - 1 - lane;
                    const bool mv = q >= minpos;
                    i32 cc = 0;
                    double vv = 0.0;
                    unsigned char ff = 0;
                    int dst = 0;
                    if (mv) {
                        cc = scol[q], vv = sval[q], ff = sflag[q];
                        int l2 = 0, h2 = nnew;
                        while (l2 < h2) {
                            const int md = (l2 + h2) >> 1;
                            if (snew[md] <= q) l2 = md + 1;
                            else h2 = md;
                        }
                        dst = q + l2;
                    }
                    gr.sync();
                    if (mv) scol[dst] = cc, sval[dst] = vv, sflag[dst] = ff;
                    gr.sync();
                }
                if (act && !found) {
                    const int dst = lo + rank;
                    scol[dst] = j;
                    sval[dst] = 0.0 - prod; // w_j was 0.0: 0.0 - m*u, not -(m*u)
                    sflag[dst] = kLive;
                }
                len += nnew;
                gr.sync();
            }
        }
        if (bad) {
            gr.sync();
            if (lane == 0) {
                if (VF) {
                    const i64 uo = a.uoff[i];
                    str_s32(a.uci + uo, static_cast<i32>(i));
                    str_f64(a.uv + uo, 1.0);
                    str_s32(a.ulen + i, 1);
                } else {
                    fi.store(E, cuda::memory_order_release);
                }
            }
            continue;
        }
        // p: first position with column >= i
        const bool hasd = p < len && scol[p] == static_cast<i32>(i);
        double d = hasd ? sval[p] : 0.0;
        if (d == 0.0) {
            if (a.patch == 0) {
                if (lane == 0) atomicMin(a.first_zero, static_cast<unsigned long long>(i));
                d = 1.0; // placeholder; the factorisation is abandoned
            } else {
                // patched_pivot(0.0, droptol, |a_i|_2, |A|_F): max(droptol*|a_i|_2, 1e-16*|A|_F)
                const double zr = a.tau[i], fl = 1e-16 * a.anorm_f;
                d = zr < fl ? fl : zr;
                if (d == 0.0) d = DBL_MIN;
            }
        }
        const int ub = p + (hasd ? 1 : 0);
        select_part<G>(scol, sval, sflag, ub, len, kLive, true, tau, a.lfill, gr, a.wrank != 0);
        const i64 uo = a.uoff[i];
        const int nu = emit<VF, G>(scol, sval, sflag, ub, len, a.uci + uo + 1, a.uv + uo + 1, gr);
        if (VF) {
            if (lane == 0) {
                str_s32(a.uci + uo, static_cast<i32>(i));
                str_f64(a.uv + uo, d);
                str_s32(a.ulen + i, nu + 1);
            }
        } else {
            if (lane == 0) {
                a.uci[uo] = static_cast<i32>(i);
                a.uv[uo] = d;
                a.ulen[i] = nu + 1;
            }
            gr.sync(); // orders every lane's row writes before lane 0's release (cumulative)
            if (lane == 0) fi.store(E, cuda::memory_order_release);
        }

        select_part<G>(scol, sval, sflag, 0, p, kKept, false, tau, a.lfill, gr, a.wrank != 0);
        const i64 lo = a.loff[i];
        const int nl = emit<false, G>(scol, sval, sflag, 0, p, a.lci + lo, a.lv + lo, gr);
        if (lane == 0) a.llen[i] = nl;
        gr.sync();
    }
}

__global__ void k_ilut_prep(i64 n, const i64* __restrict__ rp, const i32* __restrict__ ci,
                            const double* __restrict__ av, double droptol, i64 lfill, double* __restrict__ tau,
                            i64* __restrict__ ucap, i64* __restrict__ lcap) {
    const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double s = 0.0;
    i64 lo = 0, up = 0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
        s = s + av[k] * av[k]; // row_two_norm: ascending, from 0.0
        lo += ci[k] < i;
        up += ci[k] > i;
    }
    tau[i] = droptol * sqrt(s);
    ucap[i + 1] = 1 + up + lfill;
    lcap[i + 1] = lo + lfill;
    if (i == 0) ucap[0] = lcap[0] = 0;
}

__global__ void k_ilut_bump(unsigned* epoch, unsigned long long* ticket, unsigned* err) {
    *epoch = *epoch + 1u;
    *ticket = 0ull;
    err[0] = err[1] = 0u;
}

__global__ void k_len_to_rp(i64 n, const i32* __restrict__ len, i64* __restrict__ rp1) {
    const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) rp1[i + 1] = len[i];
    if (i == 0) rp1[0] = 0;
}

// warp per row: slot -> compact CSR
__global__ void k_compact(i64 n, const i64* __restrict__ off, const i64* __restrict__ rp, const i32* __restrict__ sc,
                          const double* __restrict__ sv, i32* __restrict__ oc, double* __restrict__ ov) {
    const i64 i = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= n) return;
    const i64 b = rp[i], len = rp[i + 1] - b, o = off[i];
    for (i64 q = lane; q < len; q += 32) {
        oc[b + q] = sc[o + q];
        ov[b + q] = sv[o + q];
    }
}

void inclusive_scan(i64* d, i64 count, cudaStream_t st) {
    size_t tmp = 0;
    ILUG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tmp, d, d, count, st));
    DBuf<char> t(static_cast<i64>(tmp));
    ILUG_CUDA(cub::DeviceScan::InclusiveSum(t.p, tmp, d, d, count, st));
    ILUG_CUDA(cudaStreamSynchronize(st)); // t is freed on return
}

// ILUG_ILUT_VF=1: value-flag publication of U rows (A/B; bitwise the same).
// Off: C2 factor kernel 1.71-1.73 s vs 1.64-1.67 s with the done flags in an
// interleaved A/B (profiles/r02_ilut_vf_ab.txt) — the kernel is bound by its
// per-row work across the SMs (2.1 / 2.9 / 5.8 s on 96 / 64 / 32 SMs), not by
// the flag round trip of the dependency chain.
// ILUG_ILUT_BACKOFF=<ns>: longest dependency-poll back-off (A/B)
unsigned ilut_backoff_ns() {
    const char* e = std::getenv("ILUG_ILUT_BACKOFF");
    return e ? static_cast<unsigned>(std::max(0, std::atoi(e))) : 32u;
}

// ILUG_ILUT_WRANK=0: the fill ranking always in shared memory (A/B)
bool ilut_wrank() {
    const char* e = std::getenv("ILUG_ILUT_WRANK");
    return !(e && e[0] == '0');
}

// ILUG_ILUT_CHUNK=<rows>: consecutive rows a warp claims per ticket
int ilut_chunk() {
    const char* e = std::getenv("ILUG_ILUT_CHUNK");
    const int c = e ? std::atoi(e) : 1;
    return c > 0 ? c : 1;
}

// ILUG_ILUT_QUOTA=<rows>: rows per warp before its CTA retires (0: persistent)
int ilut_quota() {
    const char* e = std::getenv("ILUG_ILUT_QUOTA");
    const int q = e ? std::atoi(e) : 256;
    return q > 0 ? q : INT_MAX;
}

// ILUG_ILUT_HALF=1: two rows per warp, one per 16-lane half (twice the rows
// in flight; working rows up to 160 entries before the capacity relaunch)
bool ilut_half() {
    const char* e = std::getenv("ILUG_ILUT_HALF");
    return e && e[0] == '1';
}

bool ilut_value_flags() {
    const char* e = std::getenv("ILUG_ILUT_VF");
    return e && e[0] == '1';
}

template <int CAP, int WARPS, int G = 32>
void launch_ilut(const IlutArgs& a, i64 ucap, cudaStream_t st) {
    constexpr int NS = WARPS * (32 / G); // rows in flight per CTA
    constexpr size_t smem = static_cast<size_t>(NS) * CAP * (sizeof(double) + sizeof(i32) + 1) +
                            static_cast<size_t>(NS) * G * sizeof(i32);
    const bool vf = ilut_value_flags();
    if (vf) {
        k_ilut_vf_fill<<<static_cast<unsigned>(std::min<i64>((ucap + 255) / 256, 148 * 64)), 256, 0, st>>>(
            ucap, a.n, a.uci, a.uv, a.ulen);
        ILUG_LAUNCH_CHECK();
    }
    auto* fn = vf ? k_ilut<CAP, WARPS, true, G> : k_ilut<CAP, WARPS, false, G>;
    ILUG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    int per_sm = 0;
    ILUG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, WARPS * 32, smem));
    if (per_sm < 1) fail_invalid("ilut (device): kernel does not fit an SM");
    // ILUG_ILUT_SMS (A/B): SMs the persistent grid may occupy (the rest stay free
    // for the AMG setup kernels that run concurrently inside run_solve)
    i64 sms = device_sm_count();
    if (const char* e = std::getenv("ILUG_ILUT_SMS"))
        if (std::atoi(e) > 0) sms = std::min<i64>(sms, std::atoi(e));
    // Each warp retires after a.quota rows, so the grid is the resident set
    // plus enough CTAs to cover every row: CTAs of the concurrent AMG setup (on
    // higher-priority streams) take the slots retiring CTAs free instead of
    // waiting for the whole factorisation. Safe: a warp claims its ticket when
    // it starts, so it only waits on rows claimed by running or finished warps.
    const i64 resident = std::min<i64>(static_cast<i64>(per_sm) * sms, (a.n + NS - 1) / NS);
    const i64 cover = (a.n + static_cast<i64>(NS) * a.quota - 1) / (static_cast<i64>(NS) * a.quota);
    const i64 grid = std::min<i64>(std::max(resident, cover + resident), INT_MAX);
    fn<<<static_cast<unsigned>(std::max<i64>(grid, 1)), WARPS * 32, smem, st>>>(a);
    ILUG_LAUNCH_CHECK();
}

} // namespace

bool ilut_on_device() {
    const char* e = std::getenv("ILUG_ILUT_DEVICE");
    return !(e && e[0] == '0');
}

DevFactors ilut_resident(const Csr& A, const IluParams& p, cudaStream_t st, bool keep_A, const DevCsr* Ad) {
    if (A.nrows != A.ncols) fail_invalid("ilut: matrix must be square");
    if (!(p.droptol >= 0.0) || !std::isfinite(p.droptol)) fail_invalid("ilut: droptol must be finite and >= 0");
    if (p.lfill < 0) fail_invalid("ilut: lfill must be >= 0");
    const i64 n = A.nrows;
    DevFactors f;
    f.n = n;
    f.diag_first = true;
    f.Lrp_h.assign(static_cast<size_t>(n) + 1, 0);
    f.Urp_h.assign(static_cast<size_t>(n) + 1, 0);
    if (n == 0) {
        f.Lrp.upload(f.Lrp_h.data(), 1, st);
        f.Urp.upload(f.Urp_h.data(), 1, st);
        ILUG_CUDA(cudaStreamSynchronize(st));
        return f;
    }
    SetupTimer tm("ilut-device");
    double anorm_f = 0.0; // |A|_F: computed only if a zero pivot is patched (see ilu0_eliminate)
    const i64 nnz = A.nnz();
    DBuf<i64> rp, uoff(n + 1), loff(n + 1);
    DBuf<i32> ci;
    DBuf<double> av, tau(n);
    if (!Ad) {
        rp.upload(A.rp.data(), n + 1, st);
        ci.upload(A.ci.data(), nnz, st);
        av.upload(A.v.data(), nnz, st);
    }
    const i64* const rpp = Ad ? Ad->rp.p : rp.p;
    const i32* const cip = Ad ? Ad->ci.p : ci.p;
    const double* const avp = Ad ? Ad->v.p : av.p;
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    k_ilut_prep<<<g, 256, 0, st>>>(n, rpp, cip, avp, p.droptol, p.lfill, tau.p, uoff.p, loff.p);
    ILUG_LAUNCH_CHECK();
    inclusive_scan(uoff.p, n + 1, st);
    inclusive_scan(loff.p, n + 1, st);
    i64 ucap = 0, lcap = 0;
    ILUG_CUDA(cudaMemcpyAsync(&ucap, uoff.p + n, sizeof ucap, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaMemcpyAsync(&lcap, loff.p + n, sizeof lcap, cudaMemcpyDeviceToHost, st));
    ILUG_CUDA(cudaStreamSynchronize(st));
    tm.mark("upload + slots");
    DBuf<i32> uci(ucap), lci(lcap), ulen(n), llen(n);
    DBuf<double> uv(ucap), lv(lcap);
    DBuf<unsigned> sync(n + 3); // done flags, epoch, err[2]
    DBuf<unsigned long long> ctl(2); // ticket, first zero
    ILUG_CUDA(cudaMemsetAsync(sync.p, 0, static_cast<size_t>(n + 3) * sizeof(unsigned), st));
    IlutArgs a{n,       rpp,    cip,    avp,    tau.p,   p.lfill, anorm_f, 0,
               p.droptol, uoff.p, loff.p, uci.p, uv.p, ulen.p, lci.p, lv.p, llen.p, sync.p, sync.p + n,
               ctl.p,   ctl.p + 1, sync.p + n + 1, ilut_wrank() ? 1 : 0, ilut_backoff_ns(), ilut_quota(), ilut_chunk()};
    unsigned err[2] = {0, 0};
    for (int pass = 0; pass < 2; ++pass) {
        for (int cap_level = 0;; ++cap_level) {
            const unsigned long long init[2] = {0ull, ~0ull};
            ILUG_CUDA(cudaMemcpyAsync(ctl.p, init, sizeof init, cudaMemcpyHostToDevice, st));
            k_ilut_bump<<<1, 1, 0, st>>>(sync.p + n, ctl.p, sync.p + n + 1);
            ILUG_LAUNCH_CHECK();
            if (cap_level == 0 && ilut_half())
                launch_ilut<160, 8, 16>(a, ucap, st);
            else if (cap_level == 0)
                launch_ilut<256, 8>(a, ucap, st);
            else if (cap_level == 1)
                launch_ilut<1024, 4>(a, ucap, st);
            else
                launch_ilut<6144, 2>(a, ucap, st);
            // wait in cudaStreamSynchronize, not inside the pageable copy: a
            // thread blocked in that copy stalls other threads' cudaMalloc
            // (the concurrent AMG setup) until the kernel ends
            ILUG_CUDA(cudaStreamSynchronize(st));
            ILUG_CUDA(cudaMemcpyAsync(err, sync.p + n + 1, sizeof err, cudaMemcpyDeviceToHost, st));
            ILUG_CUDA(cudaStreamSynchronize(st));
            if (err[0]) fail_numeric("ilut (device): dependency wait timed out (scheduling error)");
            if (err[1] == 0) break;
            if (cap_level == 2 || err[1] > 6144)
                fail_invalid("ilut (device): a working row needs " + std::to_string(err[1]) +
                             " entries (> 6144); set ILUG_ILUT_DEVICE=0 to factor on the host");
        }
        tm.mark("factor kernel");
        unsigned long long fz = 0;
        ILUG_CUDA(cudaMemcpyAsync(&fz, ctl.p + 1, sizeof fz, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        if (fz == ~0ull || pass == 1) break;
        if (p.pivot_patch == PivotPatch::error)
            fail_numeric("zero pivot at step " + std::to_string(fz) +
                         " (no pivoting; rerun with pivot_patch=replace to substitute)");
        anorm_f = frobenius_norm(A); // patched pivots: rerun with the reference's |A|_F
        a.anorm_f = anorm_f;
        a.patch = 1;
    }
    // compact the slots into CSR (stays on the device; row starts to the host)
    if (keep_A && !Ad) {
        f.Arp = std::move(rp), f.Aci = std::move(ci), f.Av = std::move(av);
    } else {
        rp.release(), ci.release(), av.release();
    }
    for (int part = 0; part < 2; ++part) {
        const DBuf<i32>& len = part == 0 ? llen : ulen;
        DBuf<i64>& mrp = part == 0 ? f.Lrp : f.Urp;
        mrp.alloc(n + 1);
        k_len_to_rp<<<g, 256, 0, st>>>(n, len.p, mrp.p);
        ILUG_LAUNCH_CHECK();
        inclusive_scan(mrp.p, n + 1, st);
        RawVec<i64>& hrp = part == 0 ? f.Lrp_h : f.Urp_h;
        mrp.download(hrp.data(), st);
        ILUG_CUDA(cudaStreamSynchronize(st));
        const i64 nz = hrp[n];
        DBuf<i32>& mc = part == 0 ? f.Lci : f.Uci;
        DBuf<double>& mv = part == 0 ? f.Lv : f.Uv;
        mc.alloc(nz);
        mv.alloc(nz);
        if (nz > 0) {
            const unsigned gw = static_cast<unsigned>((n * 32 + 255) / 256);
            k_compact<<<gw, 256, 0, st>>>(n, part == 0 ? loff.p : uoff.p, mrp.p, part == 0 ? lci.p : uci.p,
                                          part == 0 ? lv.p : uv.p, mc.p, mv.p);
            ILUG_LAUNCH_CHECK();
        }
    }
    ILUG_CUDA(cudaStreamSynchronize(st)); // slot arrays die at scope exit
    tm.mark("compact");
    return f;
}

} // namespace ilug
