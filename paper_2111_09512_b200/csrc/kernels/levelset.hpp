// K5 level-scheduled solves (see levelset.cu).
#pragma once

#include "ops.hpp"

namespace ilug {

class LevelPlan {
public:
    enum class Kind { lower_unit, upper, gauss_seidel };

    /// Analyse T's dependency DAG (strict lower part for lower_unit and
    /// gauss_seidel, strict upper part for upper) and upload a level-ordered
    /// SELL copy of T (all stored entries; the kernel skips the diagonal).
    /// dev_vals (optional): device copy of T's values to use instead of T.v
    /// (e.g. the K1-scaled U that only exists on the device).
    void build(const Csr& T, Kind kind, cudaStream_t st, const double* dev_vals = nullptr);

    /// New values for the same pattern (device CSR of T): the level-ordered copy
    /// is refilled in place (numeric refactorisation).
    void refill(const i64* rp, const i32* ci, const double* v, cudaStream_t st);

    /// lower_unit / upper: x = T^-1 b. gauss_seidel: x = one forward GS sweep
    /// from xold (x and xold must differ).
    void solve(const double* b, double* x, const double* xold, cudaStream_t st) const;

    int levels() const { return nlev_; }
    int grid() const { return single_cta_ ? cluster_ : grid_; }
    bool cluster_schedule() const { return single_cta_; }
    const Sell& matrix() const { return M_; }

private:
    Kind kind_ = Kind::lower_unit;
    Sell M_;
    DBuf<i64> level_ptr_;
    DBuf<unsigned> flags_; // sync-free schedule: row flags + epoch + ticket
    bool single_cta_ = true;
    int nlev_ = 0;
    int grid_ = 1;
    int cluster_ = 1;       // CTAs of the level-synchronous cluster schedule
    bool old_cta_ = false;  // ILUG_LEVELSET=cta1: the one-CTA register-pipelined kernel
    int block_ = 512;       // threads per CTA of the warp-per-row cluster kernel
    int slots_ = 1;         // rows per warp prefetched and processed together
    bool value_flags_ = true; // sync-free schedule polls x itself (sentinel-filled) instead of flags
    int vf_form_ = 0;
    bool sx_ = false;         // one-CTA warp kernel with the solution in shared memory         // value-flag kernel form: 1 thread per row (8-entry chunks), 8 / 83 lanes per row
    i64 max_level_rows_ = 0;
    int dsm_cs_ = 0, dsm_shift_ = 0, dsm_smem_ = 0, dsm_max_row_ = 0; // ILUG_LEVELSET_DSM=1 cluster form
};

/// Sync `st`, then raise ERR_NUMERIC if a sync-free level-set kernel hit its
/// dependency-wait bound since the last check (and clear the flag).
void levelset_check_error(cudaStream_t st);

} // namespace ilug
