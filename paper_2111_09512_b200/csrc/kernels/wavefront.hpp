// Temporally blocked Richardson/Jacobi sweeps (kernels/wavefront.cu).
#pragma once

#include "ops.hpp"

namespace ilug {

constexpr int kWaveTile = 128;     // rows per work item = threads per CTA (one row per thread)
constexpr int kWaveMaxSweeps = 9;  // up to 8 intermediate iterates

/// Dependency plan of a strictly triangular SELL operator for the wavefront
/// kernel. Tile = kWaveTile consecutive SELL positions (after the SELL-C-sigma
/// row sort); tiles are processed in order for a lower operator and in reverse
/// order for an upper one ("position" = index in that order). The rows at
/// position p read previous-sweep iterates only at positions need[2p]..need[2p+1]
/// (empty range: no input). fwd = max(need[2p+1] - p, 0): dependencies ahead of
/// the reader (only inside a sorting window for banded factors).
struct WavePlan {
    i64 ntiles = 0;
    bool upper = true;
    i64 fwd = 0;
    double tile_bytes = 0; ///< HBM bytes one tile-sweep streams (operator + vectors), for the L2 budget
    int resident = 0;      ///< CTAs of the kernel resident per SM
    DBuf<i32> need;        ///< 2 * ntiles: [lo, hi] input positions
    DBuf<unsigned> sync;   ///< done flags, frontiers, epoch, ticket, error, wait counter
    bool ready() const { return ntiles > 0; }
};

/// Build the plan of the SELL operator S packed from the host pattern T (strict
/// part selection identical: upper = columns > row, lower = columns < row).
/// Leaves the plan empty (not ready) when the fused kernel cannot keep a
/// sweep's operator in L2 between sweeps or the dependency ranges are too wide,
/// unless ILUG_WAVEFRONT=1 forces it.
void wave_build(WavePlan& W, const Csr& T, const Sell& S, bool upper, cudaStream_t st);

/// Whether the fused path is considered for an operator of n rows: opt-in with
/// ILUG_WAVEFRONT=1 (measured slower than separate sweeps on B200, see .cu).
bool wave_enabled(i64 n);

/// How the last of the fused sweeps writes its result (s = row sum with the
/// last input iterate): plain out = rhs - s; div out = (rhs - s) / d;
/// acc out += rhs - s; acc_div out += (rhs - s) / d; both out = rhs - s and
/// out2 = (rhs - s) / d. Intermediate sweeps write rhs - s, or (rhs - s) / d
/// when `mid_div` is set (Jacobi form).
enum class WaveLast { plain, div, acc, acc_div, both };

/// nsweeps consecutive sweeps x_{k+1} = rhs - T x_k (or D^-1 (rhs - T x_k))
/// starting from x_1 = x1, in ONE launch: items (tile, sweep) are handed out
/// in wavefront order, each waits only for the tiles its rows read in the
/// previous sweep, and a tile's operator slices are reused from L2 by the
/// following sweeps. tmp: (nsweeps-1) * n doubles, the intermediate iterates
/// back to back. Bitwise equal to nsweeps separate sweeps.
void wave_sweeps(const Sell& T, const WavePlan& W, int nsweeps, const double* x1, const double* rhs,
                 const double* mid_div, double* tmp, WaveLast last, const double* div, double* out,
                 double* out2, cudaStream_t st);

/// Whether any launch on this plan hit the bounded-spin guard since the last
/// call (then its result is wrong; a scheduling bug); `waits` = work items that
/// found their inputs unfinished when claimed (schedule diagnostic).
/// Synchronizes; resets both counters.
bool wave_stalled(const WavePlan& W, long long* waits = nullptr);

} // namespace ilug
