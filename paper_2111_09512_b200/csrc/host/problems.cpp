#include "problems.hpp"
#include "dist.hpp"

#include <atomic>
#include <charconv>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <cctype>
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <memory>
#include <random>
#include <sstream>

namespace ilug {

namespace {

std::uint64_t splitmix(std::uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Build a CSR from a per-row emitter: pass 1 counts, pass 2 fills, both
// row-parallel. emit(i, cols, vals) must produce strictly increasing columns.
// Rows [r0, r1) of a generated matrix (global column ids); the full matrix is
// r0 = 0, r1 = n. Pass 1 counts, pass 2 fills, both row-parallel.
template <typename Emit>
Csr build_range(i64 r0, i64 r1, i64 ncols, Emit emit) {
    const i64 n = r1 - r0;
    Csr A;
    A.nrows = n;
    A.ncols = ncols;
    A.rp.assign(static_cast<size_t>(n) + 1, 0);
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        i32 c[64];
        double v[64];
        for (i64 i = b; i < e; ++i) A.rp[i + 1] = emit(r0 + i, c, v);
    });
    for (i64 i = 0; i < n; ++i) A.rp[i + 1] += A.rp[i];
    A.ci.resize(static_cast<size_t>(A.rp[n]));
    A.v.resize(static_cast<size_t>(A.rp[n]));
    parallel_ranges(n, [&](i64 b, i64 e, int) {
        i32 c[64];
        double v[64];
        for (i64 i = b; i < e; ++i) {
            const int m = emit(r0 + i, c, v);
            std::copy(c, c + m, A.ci.begin() + A.rp[i]);
            std::copy(v, v + m, A.v.begin() + A.rp[i]);
        }
    });
    return A;
}

template <typename Emit>
Csr build_rows(i64 n, i64 ncols, int, Emit emit) {
    return build_range(0, n, ncols, emit);
}

// Active row range of a 3D generator call (whole matrix unless a range is given).
struct Range {
    i64 r0 = 0, r1 = -1;
    i64 lo(i64) const { return r0; }
    i64 hi(i64 n) const { return r1 < 0 ? n : r1; }
};

void check_grid(i64 nx, i64 ny, i64 nz, const char* what) {
    if (nx < 1 || ny < 1 || nz < 1) fail_invalid(std::string(what) + ": grid dimensions must be >= 1");
    if (nx * ny * nz > 0x7fffffffLL) fail_invalid(std::string(what) + ": more than 2^31-1 rows");
}

} // namespace

double hash_unit(std::uint64_t seed, std::uint64_t index) {
    return static_cast<double>(splitmix(seed ^ splitmix(index)) >> 11) * 0x1.0p-53;
}

Vec random_uniform(i64 n, std::uint64_t seed) {
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    Vec v(static_cast<size_t>(n));
    for (double& x : v) x = dist(gen);
    return v;
}

Csr poisson1d(i64 n) {
    if (n < 1) fail_invalid("poisson1d: n must be >= 1");
    return build_rows(n, n, 3, [n](i64 i, i32* c, double* v) {
        int m = 0;
        if (i > 0) c[m] = static_cast<i32>(i - 1), v[m++] = -1.0;
        c[m] = static_cast<i32>(i), v[m++] = 2.0;
        if (i + 1 < n) c[m] = static_cast<i32>(i + 1), v[m++] = -1.0;
        return m;
    });
}

Csr anisotropic2d(i64 nx, i64 ny, double eps) {
    if (nx < 1 || ny < 1) fail_invalid("anisotropic2d: grid dimensions must be >= 1");
    if (!(eps > 0.0)) fail_invalid("anisotropic2d: eps must be > 0");
    const double diag = 2.0 * eps + 2.0;
    return build_rows(nx * ny, nx * ny, 5, [=](i64 i, i32* c, double* v) {
        const i64 ix = i % nx, iy = i / nx;
        int m = 0;
        if (iy > 0) c[m] = static_cast<i32>(i - nx), v[m++] = -1.0;
        if (ix > 0) c[m] = static_cast<i32>(i - 1), v[m++] = -eps;
        c[m] = static_cast<i32>(i), v[m++] = diag;
        if (ix + 1 < nx) c[m] = static_cast<i32>(i + 1), v[m++] = -eps;
        if (iy + 1 < ny) c[m] = static_cast<i32>(i + nx), v[m++] = -1.0;
        return m;
    });
}

namespace {

Csr poisson3d_range(i64 nx, i64 ny, i64 nz, Range rg) {
    check_grid(nx, ny, nz, "poisson3d");
    const i64 pl = nx * ny, n = pl * nz;
    return build_range(rg.lo(n), rg.hi(n), n, [=](i64 i, i32* c, double* v) {
        const i64 ix = i % nx, iy = (i / nx) % ny, iz = i / pl;
        int m = 0;
        auto put = [&](i64 j, double x) { c[m] = static_cast<i32>(j), v[m++] = x; };
        if (iz > 0) put(i - pl, -1.0);
        if (iy > 0) put(i - nx, -1.0);
        if (ix > 0) put(i - 1, -1.0);
        put(i, 6.0);
        if (ix + 1 < nx) put(i + 1, -1.0);
        if (iy + 1 < ny) put(i + nx, -1.0);
        if (iz + 1 < nz) put(i + pl, -1.0);
        return m;
    });
}

template <typename Coef>
Csr box27(i64 nx, i64 ny, i64 nz, Coef coef, Range rg) {
    const i64 pl = nx * ny, n = pl * nz;
    return build_range(rg.lo(n), rg.hi(n), n, [=](i64 i, i32* c, double* v) {
        const i64 ix = i % nx, iy = (i / nx) % ny, iz = i / pl;
        int m = 0, dpos = -1;
        double diag = 0.0;
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    if (dx == 0 && dy == 0 && dz == 0) {
                        dpos = m;
                        c[m] = static_cast<i32>(i), v[m++] = 0.0;
                        continue;
                    }
                    const int dist = (dx != 0) + (dy != 0) + (dz != 0);
                    const bool inside = ix + dx >= 0 && ix + dx < nx && iy + dy >= 0 &&
                                        iy + dy < ny && iz + dz >= 0 && iz + dz < nz;
                    const i64 j = inside ? i + dz * pl + dy * nx + dx : -1;
                    const double a = coef(i, j, dist); // off-diagonal magnitude
                    diag += a;
                    if (inside) c[m] = static_cast<i32>(j), v[m++] = -a;
                }
        v[dpos] = diag;
        return m;
    });
}

Csr stencil27_range(i64 nx, i64 ny, i64 nz, Range rg) {
    check_grid(nx, ny, nz, "stencil27");
    return box27(nx, ny, nz, [](i64, i64, int) { return 1.0; }, rg);
}

Csr pressure27_range(i64 nx, i64 ny, i64 nz, std::uint64_t seed, Range rg) {
    check_grid(nx, ny, nz, "pressure27");
    const i64 n = nx * ny * nz, pl = nx * ny;
    // kappa of the active rows and their stencil neighbours (one plane + one row + 1 each side)
    const i64 k0 = std::max<i64>(0, rg.lo(n) - pl - nx - 1), k1 = std::min(n, rg.hi(n) + pl + nx + 1);
    auto kap = std::make_shared<std::vector<double>>(static_cast<size_t>(k1 - k0));
    parallel_ranges(k1 - k0, [&](i64 b, i64 e, int) {
        for (i64 i = b; i < e; ++i)
            (*kap)[i] = std::pow(10.0, 4.0 * hash_unit(seed, static_cast<std::uint64_t>(k0 + i)) - 2.0);
    });
    const double* kappa = kap->data() - k0;
    return box27(nx, ny, nz, [=](i64 i, i64 j, int dist) {
        const double w = dist == 1 ? 1.0 : (dist == 2 ? 0.5 : 0.25);
        const double ki = kappa[i];
        if (j < 0) return w * ki; // out-of-grid slot: hm(ki, ki) = ki
        const double kj = kappa[j];
        return w * (2.0 * ki * kj / (ki + kj));
    }, rg);
}

Csr cutcell_range(i64 nx, i64 ny, i64 nz, std::uint64_t seed, Range rg) {
    check_grid(nx, ny, nz, "cutcell");
    const i64 pl = nx * ny, n = pl * nz;
    const double R = 0.3 * static_cast<double>(nx);
    const double cx = 0.5 * nx, cy = 0.5 * ny, cz = 0.5 * nz;
    auto cell = [=](i64 i, double& kappa, double& rho) {
        const double x = static_cast<double>(i % nx) + 0.5 - cx;
        const double y = static_cast<double>((i / nx) % ny) + 0.5 - cy;
        const double z = static_cast<double>(i / pl) + 0.5 - cz;
        const double r = std::sqrt(x * x + y * y + z * z);
        rho = r < R ? 1000.0 : 1.0;
        kappa = std::abs(r - R) < 0.75
                    ? std::pow(10.0, 16.0 * hash_unit(seed, static_cast<std::uint64_t>(i)))
                    : 1.0;
    };
    return build_range(rg.lo(n), rg.hi(n), n, [=](i64 i, i32* c, double* v) {
        const i64 ix = i % nx, iy = (i / nx) % ny, iz = i / pl;
        double ki, ri;
        cell(i, ki, ri);
        auto face = [&](bool inside, i64 j) {
            if (!inside) return ki / ri; // mirrored cell: (ki+ki)/2 * 2/(ri+ri)
            double kj, rj;
            cell(j, kj, rj);
            return (ki + kj) / 2.0 * (2.0 / (ri + rj));
        };
        const bool in[6] = {iz > 0, iy > 0, ix > 0, ix + 1 < nx, iy + 1 < ny, iz + 1 < nz};
        const i64 nb[6] = {i - pl, i - nx, i - 1, i + 1, i + nx, i + pl};
        double f[6], diag = 0.0;
        for (int s = 0; s < 6; ++s) {
            f[s] = face(in[s], nb[s]);
            diag += f[s];
        }
        int m = 0;
        for (int s = 0; s < 3; ++s)
            if (in[s]) c[m] = static_cast<i32>(nb[s]), v[m++] = -f[s];
        c[m] = static_cast<i32>(i), v[m++] = diag;
        for (int s = 3; s < 6; ++s)
            if (in[s]) c[m] = static_cast<i32>(nb[s]), v[m++] = -f[s];
        return m;
    });
}

} // namespace

Csr poisson3d(i64 nx, i64 ny, i64 nz) { return poisson3d_range(nx, ny, nz, {}); }
Csr stencil27(i64 nx, i64 ny, i64 nz) { return stencil27_range(nx, ny, nz, {}); }
Csr pressure27(i64 nx, i64 ny, i64 nz, std::uint64_t seed) { return pressure27_range(nx, ny, nz, seed, {}); }
Csr cutcell(i64 nx, i64 ny, i64 nz, std::uint64_t seed) { return cutcell_range(nx, ny, nz, seed, {}); }

Csr generate_rows(const std::string& spec, i64 row0, i64 row1) {
    const auto open = spec.find('('), close = spec.rfind(')');
    if (open == std::string::npos || close == std::string::npos || close < open)
        fail_invalid("generate_rows: malformed spec '" + spec + "'");
    const std::string kind = spec.substr(0, open);
    std::string args = spec.substr(open + 1, close - open - 1);
    for (char& ch : args)
        if (ch == ',') ch = ' ';
    std::istringstream in(args);
    i64 nx = 0, ny = 0, nz = 0;
    if (!(in >> nx >> ny >> nz)) fail_invalid("generate_rows: " + kind + " expects (nx,ny,nz[,seed])");
    std::uint64_t seed = 2111;
    {
        unsigned long long s;
        if (in >> s) seed = s;
    }
    if (row0 < 0 || row1 < row0 || row1 > nx * ny * nz) fail_invalid("generate_rows: row range out of bounds");
    const Range rg{row0, row1};
    if (kind == "poisson3d") return poisson3d_range(nx, ny, nz, rg);
    if (kind == "stencil27") return stencil27_range(nx, ny, nz, rg);
    if (kind == "pressure27") return pressure27_range(nx, ny, nz, seed, rg);
    if (kind == "cutcell") return cutcell_range(nx, ny, nz, seed, rg);
    fail_invalid("generate_rows: only 3D generators support row ranges, got '" + kind + "'");
}

namespace {
const char* kSpecs[] = {"poisson1d(",  "poisson2d(", "anisotropic2d(", "poisson3d(",
                        "stencil27(",  "pressure27(", "cutcell("};
}

bool is_generator_spec(const std::string& s) {
    for (const char* p : kSpecs)
        if (s.rfind(p, 0) == 0) return true;
    return false;
}

Csr generate_problem(const std::string& spec) {
    const auto open = spec.find('('), close = spec.rfind(')');
    if (open == std::string::npos || close == std::string::npos || close < open)
        fail_invalid("generate_problem: malformed spec '" + spec + "'");
    const std::string kind = spec.substr(0, open);
    std::string args = spec.substr(open + 1, close - open - 1);
    for (char& ch : args)
        if (ch == ',') ch = ' ';
    std::istringstream in(args);
    auto need = [&](bool ok, const char* sig) {
        if (!ok) fail_invalid("generate_problem: " + kind + " expects " + sig);
    };
    if (kind == "poisson1d") {
        i64 n = 0;
        need(static_cast<bool>(in >> n), "(n)");
        return poisson1d(n);
    }
    if (kind == "poisson2d" || kind == "anisotropic2d") {
        i64 nx = 0, ny = 0;
        double eps = 1.0;
        if (kind == "poisson2d")
            need(static_cast<bool>(in >> nx >> ny), "(nx,ny)");
        else
            need(static_cast<bool>(in >> nx >> ny >> eps), "(nx,ny,eps)");
        return anisotropic2d(nx, ny, eps);
    }
    i64 nx = 0, ny = 0, nz = 0;
    need(static_cast<bool>(in >> nx >> ny >> nz), "(nx,ny,nz[,seed])");
    std::uint64_t seed = 2111;
    {
        unsigned long long s;
        if (in >> s) seed = s;
    }
    if (kind == "poisson3d") return poisson3d(nx, ny, nz);
    if (kind == "stencil27") return stencil27(nx, ny, nz);
    if (kind == "pressure27") return pressure27(nx, ny, nz, seed);
    if (kind == "cutcell") return cutcell(nx, ny, nz, seed);
    fail_invalid("generate_problem: unknown generator '" + kind + "'");
}

namespace {

bool mm_space(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// Parallel parse of the entry section data[0, size): tokens are maximal
// non-whitespace runs (the reference reads entries with operator>>, so line
// breaks carry no meaning). Fills i/j (1-based) and v for the first nnz
// entries. Returns false on anything the plain from_chars path does not parse
// exactly like operator>> would (a sign '+', inf/nan, out-of-range numbers,
// trailing garbage in a token, fewer than 3*nnz tokens): the caller then
// re-reads the file with the reference-order stream parser.
bool mm_parse_entries(const char* data, size_t size, i64 nnz, std::vector<i64>& I, std::vector<i64>& J,
                      std::vector<double>& V) {
    const i64 need = 3 * nnz;
    const int T = std::max(1, host_threads() * 4);
    std::vector<size_t> cut(static_cast<size_t>(T) + 1, size);
    cut[0] = 0;
    for (int c = 1; c < T; ++c) {
        size_t p = size * static_cast<size_t>(c) / static_cast<size_t>(T);
        while (p < size && !mm_space(data[p])) ++p; // chunk edges on whitespace
        cut[c] = std::max(p, cut[c - 1]);
    }
    std::vector<i64> ntok(static_cast<size_t>(T) + 1, 0);
    parallel_ranges(T, [&](i64 b, i64 e, int) {
        for (i64 c = b; c < e; ++c) {
            i64 n = 0;
            bool in = false;
            for (size_t p = cut[c]; p < cut[c + 1]; ++p) {
                const bool sp = mm_space(data[p]);
                n += !sp && !in;
                in = !sp;
            }
            ntok[c + 1] = n;
        }
    }, 1);
    for (int c = 0; c < T; ++c) ntok[c + 1] += ntok[c];
    if (ntok[T] < need) return false;
    I.resize(static_cast<size_t>(nnz));
    J.resize(static_cast<size_t>(nnz));
    V.resize(static_cast<size_t>(nnz));
    std::atomic<bool> ok{true};
    parallel_ranges(T, [&](i64 b, i64 e, int) {
        for (i64 c = b; c < e && ok.load(std::memory_order_relaxed); ++c) {
            i64 g = ntok[c];
            size_t p = cut[c];
            const size_t end = cut[c + 1];
            while (p < end && g < need) {
                while (p < end && mm_space(data[p])) ++p;
                if (p >= end) break;
                size_t q = p;
                while (q < end && !mm_space(data[q])) ++q;
                const char* a = data + p;
                const char* z = data + q;
                const i64 ent = g / 3;
                // a digit or '.' first, after at most one '-': no '+', inf or nan
                const char* d0 = *a == '-' && a + 1 < z ? a + 1 : a;
                if (*d0 != '.' && !(*d0 >= '0' && *d0 <= '9')) {
                    ok = false;
                    return;
                }
                if (g % 3 < 2) {
                    i64 x = 0;
                    const auto r = std::from_chars(a, z, x);
                    if (r.ec != std::errc() || r.ptr != z) {
                        ok = false;
                        return;
                    }
                    (g % 3 == 0 ? I : J)[static_cast<size_t>(ent)] = x;
                } else {
                    double x = 0.0;
                    const auto r = std::from_chars(a, z, x, std::chars_format::general);
                    // subnormal results: the stream parser's range handling decides
                    if (r.ec != std::errc() || r.ptr != z || (x != 0.0 && std::abs(x) < DBL_MIN)) {
                        ok = false;
                        return;
                    }
                    V[static_cast<size_t>(ent)] = x;
                }
                ++g;
                p = q;
            }
        }
    }, 1);
    return ok.load();
}

} // namespace

// src/matrix_market.cpp semantics (header/size checks, entry errors by entry
// number, symmetric storage expanded, then from_triplets: duplicates summed in
// input order, exact zeros dropped). The entry section is parsed in parallel
// from a memory map; files the fast parser declines are read with the
// reference-order stream parser (mm_read_stream), so results and errors are
// the reference's either way.
Csr mm_read_stream(std::istream& in, const std::string& path, i64 nr, i64 nc, i64 nnz, bool symmetric) {
    std::vector<Triplet> t;
    t.reserve(static_cast<size_t>(symmetric ? 2 * nnz : nnz));
    for (i64 k = 0; k < nnz; ++k) {
        i64 i = 0, j = 0;
        double v = 0.0;
        if (!(in >> i >> j >> v)) fail_io("mm_read: '" + path + "' truncated at entry " + std::to_string(k + 1));
        if (i < 1 || i > nr || j < 1 || j > nc)
            fail_io("mm_read: '" + path + "' index out of range at entry " + std::to_string(k + 1));
        t.push_back({i - 1, j - 1, v});
        if (symmetric && i != j) t.push_back({j - 1, i - 1, v});
    }
    return csr_from_triplets(nr, nc, std::move(t));
}

Csr mm_read(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail_io("mm_read: cannot open '" + path + "'");
    std::string line;
    if (!std::getline(in, line)) fail_io("mm_read: '" + path + "' is empty");
    std::istringstream hdr(line);
    std::string banner, object, format, field, sym;
    hdr >> banner >> object >> format >> field >> sym;
    auto low = [](std::string s) {
        for (char& ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
        return s;
    };
    if (banner != "%%MatrixMarket" || low(object) != "matrix")
        fail_io("mm_read: '" + path + "' has a malformed Matrix Market header");
    format = low(format), field = low(field), sym = low(sym);
    if (format != "coordinate") fail_io("mm_read: only coordinate format is supported (got '" + format + "')");
    if (field == "complex" || field == "pattern")
        fail_io("mm_read: field type '" + field + "' is not supported; real matrices only");
    if (field != "real" && field != "integer") fail_io("mm_read: unsupported field type '" + field + "'");
    if (sym != "general" && sym != "symmetric")
        fail_io("mm_read: unsupported symmetry '" + sym + "'; general and symmetric only");
    const bool symmetric = sym == "symmetric";
    while (std::getline(in, line))
        if (!line.empty() && line[0] != '%') break;
    std::istringstream sz(line);
    i64 nr = 0, nc = 0, nnz = 0;
    if (!(sz >> nr >> nc >> nnz) || nr < 0 || nc < 0 || nnz < 0)
        fail_io("mm_read: '" + path + "' has a malformed size line");
    const std::streamoff body = in.tellg();

    // fast path: map the file, parse the entry section in parallel
    if (body >= 0 && nnz > 0) {
        const int fd = ::open(path.c_str(), O_RDONLY);
        struct stat st {};
        if (fd >= 0 && ::fstat(fd, &st) == 0 && st.st_size > body) {
            const size_t fsize = static_cast<size_t>(st.st_size);
            void* m = ::mmap(nullptr, fsize, PROT_READ, MAP_PRIVATE, fd, 0);
            ::close(fd);
            if (m != MAP_FAILED) {
                std::vector<i64> I, J;
                std::vector<double> V;
                const bool ok = mm_parse_entries(static_cast<const char*>(m) + body, fsize - static_cast<size_t>(body),
                                                 nnz, I, J, V);
                ::munmap(m, fsize);
                if (ok) {
                    // first out-of-range entry in order, as the stream parser reports it
                    std::atomic<i64> bad{nnz};
                    parallel_ranges(nnz, [&](i64 b, i64 e, int) {
                        for (i64 k = b; k < e; ++k)
                            if (I[k] < 1 || I[k] > nr || J[k] < 1 || J[k] > nc) {
                                i64 cur = bad.load();
                                while (k < cur && !bad.compare_exchange_weak(cur, k)) {
                                }
                                return;
                            }
                    });
                    if (bad.load() < nnz)
                        fail_io("mm_read: '" + path + "' index out of range at entry " +
                                std::to_string(bad.load() + 1));
                    // triplets in input order (a symmetric off-diagonal entry is followed by its mirror)
                    std::vector<i64> off(static_cast<size_t>(nnz) + 1, 0);
                    if (symmetric) {
                        parallel_ranges(nnz, [&](i64 b, i64 e, int) {
                            for (i64 k = b; k < e; ++k) off[k + 1] = I[k] != J[k];
                        });
                        for (i64 k = 0; k < nnz; ++k) off[k + 1] += off[k];
                    }
                    std::vector<Triplet> t(static_cast<size_t>(nnz + off[nnz]));
                    parallel_ranges(nnz, [&](i64 b, i64 e, int) {
                        for (i64 k = b; k < e; ++k) {
                            const i64 o = k + off[k];
                            t[o] = {I[k] - 1, J[k] - 1, V[k]};
                            if (symmetric && I[k] != J[k]) t[o + 1] = {J[k] - 1, I[k] - 1, V[k]};
                        }
                    });
                    return csr_from_triplets(nr, nc, std::move(t));
                }
            }
        } else if (fd >= 0) {
            ::close(fd);
        }
        in.clear();
        in.seekg(body);
    }
    return mm_read_stream(in, path, nr, nc, nnz, symmetric);
}

// Same text as src/matrix_market.cpp mm_write ("%.17g" values, 1-based
// indices, one entry per line); rows are formatted in parallel blocks and
// written in order.
void mm_write(const Csr& A, const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "w");
    if (!f) fail_io("mm_write: cannot open '" + path + "' for writing");
    std::fprintf(f, "%%%%MatrixMarket matrix coordinate real general\n%lld %lld %lld\n",
                 static_cast<long long>(A.nrows), static_cast<long long>(A.ncols),
                 static_cast<long long>(A.nnz()));
    constexpr i64 kRows = 1 << 16; // rows per formatted block
    const i64 nblk = (A.nrows + kRows - 1) / kRows;
    bool ok = true;
    for (i64 b0 = 0; b0 < nblk && ok; b0 += 64) { // 64 blocks in flight at a time
        const i64 b1 = std::min(nblk, b0 + 64);
        std::vector<std::string> text(static_cast<size_t>(b1 - b0));
        parallel_ranges(b1 - b0, [&](i64 lo, i64 hi, int) {
            char buf[96];
            for (i64 bb = lo; bb < hi; ++bb) {
                std::string& out = text[static_cast<size_t>(bb)];
                const i64 r0 = (b0 + bb) * kRows, r1 = std::min(A.nrows, r0 + kRows);
                out.reserve(static_cast<size_t>(A.rp[r1] - A.rp[r0]) * 36);
                for (i64 i = r0; i < r1; ++i)
                    for (i64 k = A.rp[i]; k < A.rp[i + 1]; ++k) {
                        const int m = std::snprintf(buf, sizeof buf, "%lld %d %.17g\n", static_cast<long long>(i + 1),
                                                    A.ci[k] + 1, A.v[k]);
                        out.append(buf, static_cast<size_t>(m));
                    }
            }
        }, 1);
        for (const std::string& t : text)
            if (std::fwrite(t.data(), 1, t.size(), f) != t.size()) ok = false;
    }
    if (std::fclose(f) != 0 || !ok) fail_io("mm_write: write to '" + path + "' failed");
}

} // namespace ilug
