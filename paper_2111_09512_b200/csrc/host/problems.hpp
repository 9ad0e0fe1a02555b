// Seeded problem generators (host, parallel, direct-to-CSR).
//
// The 2D family reproduces the reference generators value-for-value
// (src/problems.cpp:9-41) so the reference's own golden iteration counts
// (tests/acceptance.cpp:154-183, :380-410) apply unchanged. The 3D family is new:
// the reference has no 3D generator, and every BASELINE
// config needs one; their definitions are in DESIGN.md §3.
#pragma once

#include "csr.hpp"

#include <string>

namespace ilug {

Csr poisson1d(i64 n);
Csr anisotropic2d(i64 nx, i64 ny, double eps);
inline Csr poisson2d(i64 nx, i64 ny) { return anisotropic2d(nx, ny, 1.0); }

/// 7-point Dirichlet Laplacian, diagonal 6, off-diagonals -1, x fastest (C1/C4).
Csr poisson3d(i64 nx, i64 ny, i64 nz);

/// Constant 27-point stencil, diagonal 26, off-diagonals -1 (BASELINE §2 probes).
Csr stencil27(i64 nx, i64 ny, i64 nz);

/// Variable-coefficient 27-point pressure matrix (C2): kappa_i = 10^(4u-2),
/// u = hash_unit(seed, i); off-diagonal -w_d * hm(kappa_i, kappa_j) with w_d = 1,
/// 1/2, 1/4 for face/edge/corner neighbours and hm the harmonic mean; the
/// diagonal sums |off| over all 26 slots, out-of-grid slots using kappa_j = kappa_i.
Csr pressure27(i64 nx, i64 ny, i64 nz, std::uint64_t seed);

/// Low-Mach cut-cell 7-point matrix (C3): sphere of radius 0.3*nx centred in the
/// box, rho = 1000 inside / 1 outside; in the band |r - R| < 0.75 the cell
/// coefficient is 10^(16u), u = hash_unit(seed, i), else 1. Face coefficient
/// (kappa_i + kappa_j)/2 * 2/(rho_i + rho_j); diagonal = sum of the six faces,
/// out-of-grid faces mirroring cell i.
Csr cutcell(i64 nx, i64 ny, i64 nz, std::uint64_t seed);

/// "poisson1d(n)", "poisson2d(nx,ny)", "anisotropic2d(nx,ny,eps)" (reference
/// specs) plus "poisson3d(nx,ny,nz)", "stencil27(nx,ny,nz)",
/// "pressure27(nx,ny,nz[,seed])", "cutcell(nx,ny,nz[,seed])".
Csr generate_problem(const std::string& spec);
bool is_generator_spec(const std::string& s);

/// splitmix64 jitter in [0,1), identical to include/iluamg/rng.hpp:16-27.
double hash_unit(std::uint64_t seed, std::uint64_t index);

/// mt19937_64 + uniform_real_distribution(-1, 1) through the same libstdc++ as
/// the reference (include/iluamg/rng.hpp:29-35), so seeded vectors match bitwise.
Vec random_uniform(i64 n, std::uint64_t seed);

/// Matrix Market coordinate real general/symmetric reader and writer (%.17g),
/// src/matrix_market.cpp semantics: symmetric storage expanded, duplicates summed.
Csr mm_read(const std::string& path);
void mm_write(const Csr& A, const std::string& path);

} // namespace ilug
