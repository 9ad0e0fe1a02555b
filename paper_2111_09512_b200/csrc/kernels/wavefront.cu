// K2/K3 temporally blocked: m-1 Richardson (or Jacobi) sweeps of a strictly
// triangular factor in ONE launch, so the factor streams from HBM about once
// per triangular phase instead of once per sweep (the rest hits L2).
//
// Why it is legal: x_{k+1}[i] = rhs[i] - sum_j T_ij x_k[j] reads x_k only at
// the columns of row i. Rows are cut into 128-row tiles (SELL positions),
// numbered in processing order (ascending for L, descending for U: a banded
// triangular factor then only reads tiles at or before its own position, plus
// a few ahead inside a SELL-C-sigma sorting window). Work items (position,
// sweep) are handed out from an atomic ticket in wavefront order: sweep k+1
// trails sweep k by `lag` positions.
//   * dependencies: item (p, k+1) needs positions need[2p]..need[2p+1] of
//     sweep k done: epoch-stamped per-position flags, checked by the whole CTA
//     with relaxed loads and one acquire fence per thread (which also drops
//     the SM's L1, so the gathers can use coherent L1-cached loads);
//   * progress: every input of an item has a smaller ticket (lag >= fwd), so
//     it was claimed by a running CTA before, which only waits on smaller
//     tickets -> no deadlock whatever the residency;
//   * no stalls: lag * nsweeps ~ 1.5 x the CTAs in flight, so an item's
//     inputs are normally finished when it is claimed;
//   * L2 reuse: between two sweeps of one tile only ~lag * nsweeps items run,
//     and the grid is sized so their operator bytes fit the L2 budget.
// Each row is one thread summing its columns in ascending order exactly as
// k_rowdot does, so the result is bitwise that of the separate sweeps. A
// bounded spin turns a scheduling bug into an error flag, never a hung GPU.
#include "wavefront.hpp"

#include <algorithm>
#include <cstdlib>

namespace ilug {

namespace {

// Sync words after the per-(sweep, position) done flags.
struct SyncWords {
    unsigned* flags; ///< [kWaveMaxSweeps][ntiles], epoch-stamped "position done"
    unsigned* epoch;
    unsigned* ticket;
    unsigned* err;
    unsigned* waits; ///< items that found their inputs unfinished (diagnostic)
};
constexpr i64 kSyncExtra = 4;

SyncWords sync_words(const WavePlan& W) {
    unsigned* base = W.sync.p + W.ntiles * kWaveMaxSweeps;
    return {W.sync.p, base, base + 1, base + 2, base + 3};
}

__global__ void k_wave_bump(SyncWords s) {
    *s.epoch = *s.epoch + 1u;
    *s.ticket = 0u;
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned* p, unsigned v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool UPPER, bool MID_DIV, WaveLast LAST>
__global__ void __launch_bounds__(kWaveTile)
k_wave(SellView M, i64 nrows, i64 ntiles, int ns, i64 lag, const i32* __restrict__ need, SyncWords sw,
       const double* __restrict__ x1, const double* __restrict__ rhs, const double* __restrict__ mdiv, double* tmp,
       const double* __restrict__ div, double* out, double* out2, bool hints) {
    __shared__ unsigned s_item;
    const unsigned E = *sw.epoch;
    const i64 total = (ntiles + (ns - 1) * lag) * static_cast<i64>(ns);
    const unsigned long long keep = l2_policy_last(), drop = l2_policy_first();
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(sw.ticket, 1u);
        __syncthreads();
        const i64 it = s_item;
        if (it >= total) return;
        const int j = static_cast<int>(it % ns);
        const i64 pos = it / ns - j * lag;
        if (pos < 0 || pos >= ntiles) {
            __syncthreads(); // everyone has read s_item before thread 0 rewrites it
            continue;
        }
        if (j > 0) {
            // inputs: positions lo..hi of sweep j-1, one epoch-stamped flag each,
            // checked by all threads in parallel (relaxed loads)
            const unsigned* fl = sw.flags + static_cast<i64>(j - 1) * ntiles;
            const i64 lo = need[2 * pos], hi = need[2 * pos + 1];
            bool waited = false;
            for (i64 q = lo + threadIdx.x; q <= hi; q += kWaveTile) {
                long long spins = 0;
                while (ld_relaxed(fl + q) != E) {
                    waited = true;
                    if (++spins > (1ll << 22)) { // ~seconds: scheduling bug, do not hang the GPU
                        atomicExch(sw.err, 1u);
                        break;
                    }
                    __nanosleep(32);
                }
            }
            if (waited) atomicAdd(sw.waits, 1u);
            __threadfence(); // acquire (also drops this SM's L1 lines: the gathers below see the new iterate)
        }
        __syncthreads();
        const i64 t = UPPER ? ntiles - 1 - pos : pos;
        const double* xin = j == 0 ? x1 : tmp + (j - 1) * nrows; // not __restrict__
        const bool last = j == ns - 1;
        const unsigned long long pol = last ? drop : keep;
        const i64 p = t * kWaveTile + threadIdx.x;
        const i64 row = p < M.nrows_pad ? (M.perm ? M.perm[p] : p) : -1;
        if (row >= 0 && row < nrows) {
            const int len = M.rowlen[p];
            const double* vp = M.vals + M.slice_ptr[p >> 5] + (p & 31);
            const int* cp = M.cols + M.slice_ptr[p >> 5] + (p & 31);
            double s = 0.0;
            int q = 0;
            for (; q + 4 <= len; q += 4) {
                double a[4], xv[4];
                int c[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    a[u] = hints ? ld_stream(vp + (q + u) * kSlice, pol) : ld_stream(vp + (q + u) * kSlice);
                    c[u] = hints ? ld_stream(cp + (q + u) * kSlice, pol) : ld_stream(cp + (q + u) * kSlice);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) xv[u] = xin[c[u]]; // coherent load (not .nc): written in this launch
#pragma unroll
                for (int u = 0; u < 4; ++u) s = s + a[u] * xv[u];
            }
            for (; q < len; ++q) s = s + ld_stream(vp + q * kSlice) * xin[ld_stream(cp + q * kSlice)];
            const double v = rhs[row] - s;
            if (!last) {
                tmp[j * nrows + row] = MID_DIV ? v / mdiv[row] : v;
            } else if (LAST == WaveLast::plain) {
                out[row] = v;
            } else if (LAST == WaveLast::div) {
                out[row] = v / div[row];
            } else if (LAST == WaveLast::acc) {
                out[row] = out[row] + v;
            } else if (LAST == WaveLast::acc_div) {
                out[row] = out[row] + v / div[row];
            } else { // both
                out[row] = v;
                out2[row] = v / div[row];
            }
        }
        __syncthreads(); // the tile's writes precede thread 0's release; s_item consumed
        if (!last && threadIdx.x == 0) {
            __threadfence(); // release: the CTA's writes (ordered by the barrier) before the flag
            st_relaxed(sw.flags + static_cast<i64>(j) * ntiles + pos, E);
        }
    }
}

template <bool UPPER, bool MID>
void launch(WaveLast last, dim3 g, cudaStream_t st, const SellView& mv, i64 nrows, i64 ntiles, int ns, i64 lag,
            const i32* need, const SyncWords& sw, const double* x1, const double* rhs, const double* mdiv,
            double* tmp, const double* div, double* out, double* out2, bool hints) {
#define ILUG_WAVE(L)                                                                                         \
    k_wave<UPPER, MID, L><<<g, kWaveTile, 0, st>>>(mv, nrows, ntiles, ns, lag, need, sw, x1, rhs, mdiv, tmp, \
                                                    div, out, out2, hints)
    switch (last) {
    case WaveLast::plain: ILUG_WAVE(WaveLast::plain); break;
    case WaveLast::div: ILUG_WAVE(WaveLast::div); break;
    case WaveLast::acc: ILUG_WAVE(WaveLast::acc); break;
    case WaveLast::acc_div: ILUG_WAVE(WaveLast::acc_div); break;
    case WaveLast::both: ILUG_WAVE(WaveLast::both); break;
    }
#undef ILUG_WAVE
    ILUG_LAUNCH_CHECK();
}

i64 env_i64(const char* name, i64 dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atoll(e) : dflt;
}

bool forced() {
    const char* e = std::getenv("ILUG_WAVEFRONT");
    return e && e[0] == '1';
}

// L2 bytes the operator slices of the items between two sweeps of a tile may
// occupy (B200: 126 MB L2; leave room for the iterates and other traffic).
double l2_budget() { return static_cast<double>(env_i64("ILUG_WAVE_L2_MB", 64)) * 1e6; }

// Items in flight between two sweeps of one tile, relative to the grid.
constexpr double kWindow = 1.5;

// Grid and lag of one launch.
void schedule(const WavePlan& W, int ns, i64& ctas, i64& lag) {
    const i64 sms = device_sm_count();
    const i64 per_sm = env_i64("ILUG_WAVE_CTAS_PER_SM", 0);
    if (per_sm > 0) {
        ctas = sms * std::min<i64>(per_sm, W.resident);
    } else {
        const i64 fit = static_cast<i64>(l2_budget() / std::max(W.tile_bytes, 1.0) / kWindow);
        ctas = std::clamp<i64>(fit, sms, sms * W.resident);
    }
    lag = std::max<i64>({1, W.fwd, static_cast<i64>(kWindow * static_cast<double>(ctas) / ns + 0.999)});
}

} // namespace

// Opt-in (ILUG_WAVEFRONT=1). Measured on B200 at C2 (pressure27 256^3 ILUT,
// tools/probe_wave.py, profiles/r01_wavefront_probe.txt): U m=5 4.3-5.2 ms fused
// vs 2.6-3.5 ms as separate sweeps. The LTS (L2 slice) throughput cap is only
// ~1.8x HBM, every L2 hit still crosses it, and the per-item acquire fences
// drop the SM's L1 (the x gathers' stencil reuse), so the fused kernel loses.
bool wave_enabled(i64 n) {
    if (n <= 0) return false;
    const char* e = std::getenv("ILUG_WAVEFRONT");
    return e && e[0] == '1';
}

void wave_build(WavePlan& W, const Csr& T, const Sell& S, bool upper, cudaStream_t st) {
    W = WavePlan{};
    const i64 n = T.nrows;
    if (n == 0 || S.nrows_pad == 0) return;
    const i64 ntiles = (S.nrows_pad + kWaveTile - 1) / kWaveTile;
    std::vector<i32> perm;
    if (S.perm.n > 0) {
        perm.resize(static_cast<size_t>(S.perm.n));
        S.perm.download(perm.data(), st);
        ILUG_CUDA(cudaStreamSynchronize(st));
    }
    // processing position of every original row
    std::vector<i32> pos_of(static_cast<size_t>(n));
    for (i64 p = 0; p < S.nrows_pad; ++p) {
        const i64 r = perm.empty() ? p : perm[p];
        if (r >= 0 && r < n) {
            const i64 t = p / kWaveTile;
            pos_of[r] = static_cast<i32>(upper ? ntiles - 1 - t : t);
        }
    }
    std::vector<i32> need(static_cast<size_t>(2 * ntiles));
    std::vector<i64> fwd(static_cast<size_t>(ntiles), 0), span(static_cast<size_t>(ntiles), 0);
    parallel_ranges(ntiles, [&](i64 b, i64 e, int) {
        for (i64 pos = b; pos < e; ++pos) {
            const i64 t = upper ? ntiles - 1 - pos : pos;
            i64 lo = ntiles, hi = -1;
            for (i64 p = t * kWaveTile; p < std::min(S.nrows_pad, (t + 1) * kWaveTile); ++p) {
                const i64 i = perm.empty() ? p : perm[p];
                if (i < 0 || i >= n) continue;
                for (i64 k = T.rp[i]; k < T.rp[i + 1]; ++k) {
                    const i64 c = T.ci[k];
                    if (upper ? c > i : c < i) {
                        lo = std::min<i64>(lo, pos_of[c]);
                        hi = std::max<i64>(hi, pos_of[c]);
                    }
                }
            }
            if (hi < 0) lo = 0; // reads nothing: empty range
            need[2 * pos] = static_cast<i32>(lo);
            need[2 * pos + 1] = static_cast<i32>(hi);
            fwd[pos] = std::max<i64>(0, hi - pos);
            span[pos] = std::max<i64>(0, hi - lo + 1);
        }
    }, 256);
    const i64 maxfwd = *std::max_element(fwd.begin(), fwd.end());
    i64 tot_span = 0;
    for (const i64 v : span) tot_span += v;
    // per tile-sweep: operator (values + columns incl. padding), rowlen, perm, and
    // the row's x gather (~ once per row via L2), rhs read and result write
    const double vec_bytes = 2.0 + (perm.empty() ? 0.0 : 4.0) + 3.0 * 8.0;
    const double tile_bytes = (12.0 * static_cast<double>(S.padded) + vec_bytes * static_cast<double>(S.nrows_pad)) /
                              static_cast<double>(ntiles);
    int resident = 0;
    ILUG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k_wave<true, false, WaveLast::plain>,
                                                            kWaveTile, 0));
    const bool fits = l2_budget() / tile_bytes / kWindow >= 4.0 * device_sm_count(); // >= 4 CTAs per SM
    const bool narrow = tot_span <= 2048 * ntiles; // flag checks stay cheap
    if (!forced() && !(fits && narrow && resident >= 4 && maxfwd <= ntiles / 8)) return;
    W.ntiles = ntiles;
    W.upper = upper;
    W.fwd = maxfwd;
    W.tile_bytes = tile_bytes;
    W.resident = std::max(resident, 1);
    W.need.upload(need.data(), 2 * ntiles, st);
    W.sync.alloc(ntiles * kWaveMaxSweeps + kSyncExtra);
    ILUG_CUDA(cudaMemsetAsync(W.sync.p, 0, static_cast<size_t>(W.sync.n) * sizeof(unsigned), st));
    ILUG_CUDA(cudaStreamSynchronize(st));
}

bool wave_stalled(const WavePlan& W, long long* waits) {
    if (waits) *waits = 0;
    if (!W.ready()) return false;
    const SyncWords sw = sync_words(W);
    unsigned h[2] = {0, 0};
    ILUG_CUDA(cudaDeviceSynchronize());
    ILUG_CUDA(cudaMemcpy(&h[0], sw.err, sizeof(unsigned), cudaMemcpyDeviceToHost));
    ILUG_CUDA(cudaMemcpy(&h[1], sw.waits, sizeof(unsigned), cudaMemcpyDeviceToHost));
    ILUG_CUDA(cudaMemset(sw.err, 0, sizeof(unsigned)));
    ILUG_CUDA(cudaMemset(sw.waits, 0, sizeof(unsigned)));
    if (waits) *waits = h[1];
    return h[0] != 0;
}

void wave_sweeps(const Sell& T, const WavePlan& W, int ns, const double* x1, const double* rhs,
                 const double* mid_div, double* tmp, WaveLast last, const double* div, double* out,
                 double* out2, cudaStream_t st) {
    if (ns < 1 || ns > kWaveMaxSweeps) fail_invalid("wavefront: sweep count out of range");
    if (!W.ready() || T.nrows_pad == 0) fail_invalid("wavefront: plan not built");
    const SyncWords sw = sync_words(W);
    k_wave_bump<<<1, 1, 0, st>>>(sw);
    ILUG_LAUNCH_CHECK();
    i64 ctas = 0, lag = 0;
    schedule(W, ns, ctas, lag);
    const i64 items = (W.ntiles + (ns - 1) * lag) * static_cast<i64>(ns);
    const dim3 g(static_cast<unsigned>(std::min<i64>(items, ctas)));
    const bool hints = env_i64("ILUG_WAVE_HINTS", 0) != 0;
    const SellView mv = view(T);
    if (W.upper) {
        if (mid_div)
            launch<true, true>(last, g, st, mv, T.nrows, W.ntiles, ns, lag, W.need.p, sw, x1, rhs, mid_div, tmp, div,
                               out, out2, hints);
        else
            launch<true, false>(last, g, st, mv, T.nrows, W.ntiles, ns, lag, W.need.p, sw, x1, rhs, mid_div, tmp,
                                div, out, out2, hints);
    } else {
        if (mid_div)
            launch<false, true>(last, g, st, mv, T.nrows, W.ntiles, ns, lag, W.need.p, sw, x1, rhs, mid_div, tmp,
                                div, out, out2, hints);
        else
            launch<false, false>(last, g, st, mv, T.nrows, W.ntiles, ns, lag, W.need.p, sw, x1, rhs, mid_div, tmp,
                                 div, out, out2, hints);
    }
}

} // namespace ilug
