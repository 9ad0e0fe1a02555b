// cuSPARSE SpSV as an alternative direct triangular solve (ILUG_DIRECT=cusparse):
// the library comparison point for the level-scheduled K5 kernels, used by the
// bench's direct-solve time-to-solution variant. Not bitwise (cuSPARSE's
// summation order is its own); iteration counts are what the comparison needs.
#pragma once

#include "../kernels/dev.cuh"

#include <memory>

namespace ilug {

class CusparseTri {
public:
    CusparseTri();
    ~CusparseTri();
    CusparseTri(const CusparseTri&) = delete;
    CusparseTri& operator=(const CusparseTri&) = delete;
    /// Device CSR (int64 row starts, int32 columns, values) copied; lower: unit
    /// diagonal implicit (strict storage); upper: diagonal stored.
    void build(i64 n, const i64* rp, const i32* ci, const double* v, i64 nnz, bool lower, cudaStream_t st);
    void solve(const double* b, double* x, cudaStream_t st) const;
    bool ready() const { return ready_; }

private:
    struct Impl;
    std::unique_ptr<Impl> p_;
    bool ready_ = false;
};

/// ILUG_DIRECT=cusparse
bool direct_uses_cusparse();

} // namespace ilug
