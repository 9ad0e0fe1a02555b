// Host-callable launchers for every device kernel (K1-K8 of SURVEY.md §2).
// All take a stream and never synchronise; errors surface as ilug::Error
// through ILUG_CUDA (mapped to status 2/3 at the C ABI).
#pragma once

#include "dev.cuh"
#include "../host/csr.hpp"

namespace ilug {

// ---- SELL construction (setup) -------------------------------------------------
enum class Part { all, strict_lower, strict_upper };

/// Upload a host CSR and pack the selected part into SELL-32 on the device.
void sell_from_host(Sell& out, const Csr& A, Part part, cudaStream_t s);
/// The same SELL (all entries) from a device CSR (nrows x ncols, nnz entries).
void sell_from_device(Sell& out, i64 nrows, i64 ncols, i64 nnz, const i64* rp, const i32* ci, const double* v,
                      cudaStream_t s, Part part = Part::all);
/// SELL-C-sigma sorting window in rows (ILUG_SELL_SIGMA, default 1024; <=1 = unsorted).
i64 sell_sigma();

/// Pack part of an already-uploaded CSR (device rp/ci/v; `pattern` is the host
/// copy of its structure, used for the layout) into SELL-32. When
/// `perm_host` is non-empty the SELL rows follow it (level-ordered copies);
/// entries equal to -1 are padding rows.
void sell_from_device_csr(Sell& out, const Csr& pattern, const i64* rp, const i32* ci,
                          const double* v, Part part, const std::vector<i32>& perm_host,
                          cudaStream_t s, bool encode = true);
/// Dictionary-code the columns (Sell::codes) when the matrix has <= 255
/// distinct offsets c - row; otherwise leaves it uncoded. The builders call it.
void sell_encode(Sell& M, cudaStream_t s);
bool sell_d8_enabled();

/// Same from device CSR arrays when only the row starts are on the host: the
/// selected part of row r has rp_host[r+1] - rp_host[r] - skip entries (skip =
/// 1 for the strict upper part of a factor whose rows start with the diagonal).
void sell_from_device_rows(Sell& out, i64 nrows, i64 ncols, const RawVec<i64>& rp_host, i64 skip, const i64* rp,
                           const i32* ci, const double* v, Part part, cudaStream_t s);

/// Rewrite the entries of an existing SELL from a device CSR with the pattern
/// it was built from (numeric refactorisation: layout and permutation reused).
void sell_refill(Sell& M, const i64* rp, const i32* ci, const double* v, Part part, cudaStream_t s);

/// Unpack a SELL back to host CSR (tests / parity downloads).
Csr sell_to_host(const Sell& M);

// ---- thread-per-row products (K2, K3, K6) ---------------------------------------
// s_i = sum_t M[i,t] x[col]  (ascending, from 0.0); then per row i:
void spmv(const Sell& M, const double* x, double* y, cudaStream_t st);                 // y = s
void spmv_add(const Sell& M, const double* x, double* acc, cudaStream_t st);           // acc += s
/// Makes a stream wait for an exchange in flight (device/dist.cu
/// HaloExchange::end). Given to a split product, the rows that read only local
/// columns are launched BEFORE the wait and the halo rows after it, so the
/// local rows overlap the exchange (Sell::split_slices); without it (or on an
/// unsplit SELL) the wait comes first and one launch covers every row.
struct HaloWait {
    void (*fn)(const void* ctx, cudaStream_t st) = nullptr;
    const void* ctx = nullptr;
    void operator()(cudaStream_t st) const {
        if (fn) fn(ctx, st);
    }
};
/// SELL of a rank's rows, local-only rows first (Sell::split_slices); columns
/// >= nloc index the halo.
void sell_from_host_split(Sell& out, const Csr& A, i64 nloc, cudaStream_t s);
/// Distributed rows: columns < nloc read x, columns >= nloc read halo[c - nloc].
void residual_split(const Sell& M, const double* x, const double* halo, i64 nloc, const double* b, double* r,
                    cudaStream_t st, const HaloWait* w = nullptr);
void spmv_split(const Sell& M, const double* x, const double* halo, i64 nloc, double* y, cudaStream_t st,
                const HaloWait* w = nullptr);
/// Split forms of the fused smoother epilogues (distributed rows: columns >= nloc read the halo)
void spmv_add_split(const Sell& M, const double* x, const double* halo, i64 nloc, double* acc, cudaStream_t st,
                    const HaloWait* w = nullptr);
void residual_scale_step_split(const Sell& M, const double* x, const double* halo, i64 nloc, const double* rhs,
                               const double* scale, double* out, cudaStream_t st, const HaloWait* w = nullptr);
void residual_scale_init_split(const Sell& M, const double* x, const double* halo, i64 nloc, const double* rhs,
                               const double* scale, double* term, double* acc, cudaStream_t st,
                               const HaloWait* w = nullptr);
void residual(const Sell& M, const double* x, const double* b, double* r, cudaStream_t st); // r = b - s
/// out = (rhs - s) / div
void sweep_div(const Sell& M, const double* x, const double* rhs, const double* div, double* out,
               cudaStream_t st);
/// out = rhs - s and out2 = out / div
void sweep_both(const Sell& M, const double* x, const double* rhs, const double* div, double* out,
                double* out2, cudaStream_t st);
/// acc += rhs - s (div == nullptr) or acc += (rhs - s) / div
void sweep_acc(const Sell& M, const double* x, const double* rhs, const double* div, double* acc,
               cudaStream_t st);
/// Jacobi-like step out of place: out = x + scale * (rhs - s)  (out != x)
void residual_scale_step(const Sell& M, const double* x, const double* rhs, const double* scale,
                         double* out, cudaStream_t st);
/// poly_gs: term = scale * (rhs - s); acc = term
void residual_scale_init(const Sell& M, const double* x, const double* rhs, const double* scale,
                         double* term, double* acc, cudaStream_t st);
/// poly_gs: term = -scale * s; acc += term
void neg_scale_acc(const Sell& M, const double* x, const double* scale, double* term, double* acc,
                   cudaStream_t st);

// ---- K1 factor scaling on the device CSR of U -----------------------------------
/// Row scaling (src/ilu.cpp:271-295) in place: d = diag(U); diag -> 1.0; off *= 1.0/d.
/// Row/column scaling (src/ilu.cpp:297-333). kind: 1 row, 2 row_col.
/// Returns -1 or the first row with a zero diagonal (numeric error).
i64 scale_upper(i64 n, const i64* rp, const i32* ci, double* v, int kind, double* rs, double* cs,
                double* scratch_dr, double* scratch_dc, cudaStream_t st);
/// d = diag(U) (0 where absent); returns first zero-diagonal row or -1.
i64 extract_diag(i64 n, const i64* rp, const i32* ci, const double* v, double* d, cudaStream_t st);

// ---- elementwise / BLAS-1 (K8 building blocks) -------------------------------------
void vec_copy(double* dst, const double* src, i64 n, cudaStream_t st);
void vec_zero(double* dst, i64 n, cudaStream_t st);
void vec_div(double* out, const double* a, const double* d, i64 n, cudaStream_t st);   // out = a / d
void vec_acc(double* x, const double* z, i64 n, cudaStream_t st);                      // x += z
void vec_acc_div(double* x, const double* z, const double* d, i64 n, cudaStream_t st); // x += z / d
void vec_scale_div(double* out, const double* w, double h, i64 n, cudaStream_t st);    // out = w / h
/// out = w / *h with h in device memory; no-op when *h == 0
void vec_scale_div_dev(double* out, const double* w, const double* h, i64 n, cudaStream_t st);
void vec_add_into(double* out, const double* a, const double* b, i64 n, cudaStream_t st); // out = a + b
void vec_sub_into(double* out, const double* a, const double* b, i64 n, cudaStream_t st); // out = a - b

/// Deterministic reductions: fixed grid, per-block partial sums, ordered final pass.
/// Results are written to device memory (out[0..]); `ws` is caller-owned device
/// workspace of reduce_ws_doubles(n, k) doubles (one in-flight reduction per ws;
/// k = the widest multi-output call it serves, any k >= 1).
i64 reduce_ws_doubles(i64 n, i64 k = 64);
void dot_dev(const double* a, const double* b, i64 n, double* out, double* ws, cudaStream_t st);
void nrm2sq_dev(const double* a, i64 n, double* out, double* ws, cudaStream_t st);
/// out = sum_i (w_i - h v_i)^2 with the scalar h read from device memory
void nrm2sq_diff_dev(const double* w, const double* v, const double* h, i64 n, double* out, double* ws,
                     cudaStream_t st);

/// CGS2 passes over the Krylov basis V (k vectors, leading dimension ld):
/// h[0..k) = V^T w
void multi_dot(const double* V, i64 ld, int k, const double* w, i64 n, double* h, double* ws,
               cudaStream_t st);
/// w -= V h_in; then h_out[0..k) = V^T w (fused: one read of V and w)
void multi_axpy_dot(const double* V, i64 ld, int k, const double* h_in, double* w, i64 n,
                    double* h_out, double* ws, cudaStream_t st);
/// w -= V h_in; then out[0] = ||w||^2 (fused)
void multi_axpy_nrm(const double* V, i64 ld, int k, const double* h_in, double* w, i64 n,
                    double* out, double* ws, cudaStream_t st);
/// y = base + sum_i c_i V_i (base may be null = 0.0), accumulated per element in
/// ascending i exactly like the reference's x_k / vy loops (src/krylov.cpp:200-211).
void multi_combine(const double* V, i64 ld, int k, const double* c, const double* base, double* y,
                   i64 n, cudaStream_t st);

// ---- K7 coarse dense solve -----------------------------------------------------------
void dense_lu_solve_dev(i64 n, const double* lu, const i64* piv, const double* b, double* x,
                        cudaStream_t st);

} // namespace ilug
