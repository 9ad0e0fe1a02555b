// Host CSR container and the setup-phase sparse kernels (transpose, SpGEMM).
//
// Same invariants as the reference's SparseMatrix (include/iluamg/sparse.hpp:14-51):
// non-decreasing row starts from 0, strictly increasing columns per row, fp64
// values, ascending-column accumulation. Storage differs: 64-bit row starts but
// 32-bit column indices (every matrix this path handles has ncols < 2^31), which
// is also the device layout, so uploads are a straight copy.
#pragma once

#include "common.hpp"

#include <tuple>

namespace ilug {

/// Allocator whose value-construction is default-initialisation: resize() of
/// the big CSR arrays does not zero-fill them on one thread; the parallel
/// loops that fill them touch the pages first (first-touch is the dominant
/// cost of assembling multi-GB operators on the host).
template <class T>
struct NoInitAlloc : std::allocator<T> {
    using std::allocator<T>::allocator;
    template <class U>
    struct rebind {
        using other = NoInitAlloc<U>;
    };
    template <class U, class... Args>
    void construct(U* p, Args&&... args) {
        if constexpr (sizeof...(Args) == 0)
            ::new (static_cast<void*>(p)) U;
        else
            ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
    }
};
template <class T>
using RawVec = std::vector<T, NoInitAlloc<T>>;

struct Csr {
    i64 nrows = 0;
    i64 ncols = 0;
    RawVec<i64> rp{0};
    RawVec<i32> ci;
    RawVec<double> v;

    i64 nnz() const { return static_cast<i64>(v.size()); }
    i64 row_len(i64 i) const { return rp[i + 1] - rp[i]; }
};

struct Triplet {
    i64 i, j;
    double v;
};

/// Sort by (row, col), sum duplicates, drop exact zeros unless keep_zeros
/// (SparseMatrix::from_triplets, src/sparse.cpp:49-86; its std::sort order for
/// repeated entries). Parallel above 2^20 triplets.
Csr csr_from_triplets(i64 nrows, i64 ncols, std::vector<Triplet> t, bool keep_zeros = false);

/// Validating adopt (SparseMatrix::from_csr, src/sparse.cpp:88-118).
Csr csr_from_arrays(i64 nrows, i64 ncols, const i64* rp, const i64* ci, const double* v);
void csr_validate(const Csr& A, const char* what);

/// Parallel deep copy (first touch spread over the worker pool).
Csr csr_copy(const Csr& A);
Csr csr_identity(i64 n);

/// y = A x, one row per task, ascending columns from 0.0 (src/sparse.cpp:162-174).
void csr_spmv(const Csr& A, const double* x, double* y);

/// Structural transpose; rows of A^T list their columns in ascending order
/// (src/sparse.cpp:233-257). Parallel two-pass bucket fill.
Csr csr_transpose(const Csr& A);

/// Exact product C = A B with the reference's accumulation order: for every row,
/// contributions a_ik b_kj arrive in (k ascending in A's row, j ascending in B's
/// row) order into a dense accumulator; exact-zero results are dropped
/// (src/sparse.cpp:176-231). Rows are independent, so it runs row-parallel.
Csr csr_matmul(const Csr& A, const Csr& B);

/// (strict lower, diagonal, strict upper) partition of a square A (src/sparse.cpp:302-325).
std::tuple<Csr, Csr, Csr> csr_split_triangular(const Csr& A);

/// Diagonal (0.0 where absent) (src/sparse.cpp:287-300).
Vec csr_diag(const Csr& A);

double frobenius_norm(const Csr& A);

} // namespace ilug
