// ILU(0) factorisation on the device (kernels/ilu0.cu).
#pragma once

#include "../host/ilu.hpp"
#include "ops.hpp"

#include <cstdint>
#include <memory>

namespace ilug {

struct DevCsr; // spgemm.hpp

/// Incomplete factors resident on the device, CSR: L strict (unit diagonal
/// implicit), U upper. `diag_first`: every U row starts with its diagonal
/// (true for every factorisation here), so the strict-upper part of row r has
/// Urp_h[r+1] - Urp_h[r] - 1 entries and the SELL layout needs only the row
/// starts on the host (Lrp_h / Urp_h), not the columns or values.
struct DevFactors {
    i64 n = 0;
    DBuf<i64> Lrp, Urp;
    DBuf<i32> Lci, Uci;
    DBuf<double> Lv, Uv;
    RawVec<i64> Lrp_h, Urp_h;
    bool diag_first = false;
    /// The factorised matrix's device CSR, kept when requested (keep_A) so the
    /// level-0 operator is built from it instead of a second upload.
    DBuf<i64> Arp;
    DBuf<i32> Aci;
    DBuf<double> Av;

    /// Download to host CSR (parity tests, the direct-solve level plans).
    HostFactors to_host(cudaStream_t st) const;
    static DevFactors upload(const HostFactors& f, cudaStream_t st);
};

/// Device-resident ILU(0) / ILUT (no host round trip of the factors).
/// Ad: A already on the device (shared with the concurrent AMG setup; read
/// only, the caller keeps it, keep_A is then ignored), else A is uploaded.
DevFactors ilu0_resident(const Csr& A, PivotPatch patch, cudaStream_t st, bool keep_A = false,
                         const DevCsr* Ad = nullptr);
DevFactors ilut_resident(const Csr& A, const IluParams& p, cudaStream_t st, bool keep_A = false,
                         const DevCsr* Ad = nullptr);
/// factorize() that leaves the factors on the device (host factorisations,
/// when forced with ILUG_ILU0_DEVICE=0 / ILUG_ILUT_DEVICE=0, are uploaded).
DevFactors factorize_resident(const Csr& A, const IluParams& p, cudaStream_t st, bool keep_A = false,
                              const DevCsr* Ad = nullptr);

/// Hash of a CSR's column pattern (pattern checks for refactorisation).
std::uint64_t csr_pattern_hash(const Csr& A);

/// Symbolic part of ILU(0) kept on the device for numeric refactorisations
/// of matrices with the same pattern (the time-stepping case of the paper's
/// finest level): row starts, columns, diagonal positions, the L/U
/// split pattern. factor() uploads only the new values, eliminates, and
/// splits; the result is bitwise the fresh ilu0_resident of the new matrix.
struct Ilu0Symbolic {
    i64 n = 0, nnz = 0;
    DBuf<i64> rp, dpos, Lrp, Urp;
    DBuf<i32> ci, order; // order: rows by wavefront level (the elimination's schedule)
    RawVec<i64> rp_h, Lrp_h, Urp_h;
    std::uint64_t ci_hash = 0;

    static std::unique_ptr<Ilu0Symbolic> analyse(const Csr& A, cudaStream_t st);
    /// Same errors as ilu0 (zero pivot); invalid if A's pattern differs.
    DevFactors factor(const Csr& A, PivotPatch patch, cudaStream_t st) const;
};

/// ILU(0) of A on the device, bitwise equal to host ilu0 (and the reference):
/// same zero-pivot policy and error messages. Returns host factors (the device
/// object builders take their patterns from the host copies).
HostFactors ilu0_device(const Csr& A, PivotPatch patch, cudaStream_t st);

/// ILUG_ILU0_DEVICE=0 keeps ILU(0) on the host (A/B, tests).
bool ilu0_on_device();

/// ILUT(droptol, lfill) of A on the device (kernels/ilut.cu), bitwise equal to
/// host ilut (and the reference, src/ilu.cpp:120-265): warp per row, rows
/// scheduled by dependency flags. Same errors as the host path.
HostFactors ilut_device(const Csr& A, const IluParams& p, cudaStream_t st);

/// ILUG_ILUT_DEVICE=0 keeps ILUT on the host (A/B, tests).
bool ilut_on_device();

/// The factorisation the device objects use: ILU(0) and ILUT on the device
/// (host versions behind ILUG_ILU0_DEVICE=0 / ILUG_ILUT_DEVICE=0).
HostFactors factorize(const Csr& A, const IluParams& p, cudaStream_t st);

} // namespace ilug
