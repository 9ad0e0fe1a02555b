// K9: the ILUT Schur-complement smoother (reference: schur_smooth,
// src/schur.cpp:158-219), device side. Every vector step is a kernel; the
// three scalars of the one-iteration interface GMRES (beta, h11, h21^2) and
// the step length alpha stay in device memory, so one application is a fixed
// launch sequence with no host round trip (capturable in the V-cycle graph).
#include "dist.hpp"

#include <cstring>

namespace ilug {

namespace {

constexpr int kB = 256;

inline unsigned grid_of(i64 n) {
    return static_cast<unsigned>(std::max<i64>(1, std::min<i64>((n + kB - 1) / kB, 148 * 64)));
}

// fg[perm[i]] = r[i]: interior values first, then interface (src/schur.cpp:166-172)
__global__ void k_split(i64 n, const i32* __restrict__ perm, const double* __restrict__ r,
                        double* __restrict__ fg) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        fg[perm[i]] = r[i];
}

// x[i] += upd[perm[i]] (interior += x_I, interface += y; src/schur.cpp:214-217)
__global__ void k_merge(i64 n, const i32* __restrict__ perm, const double* __restrict__ upd,
                        double* __restrict__ x) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        x[i] = x[i] + upd[perm[i]];
}

// v1 = gt / beta with beta = sqrt(beta2) (only meaningful when beta > 0; for
// beta == 0, gt == 0 and v1 = 0 keeps every later product zero).
__global__ void k_normalize(i64 n, const double* __restrict__ gt, const double* __restrict__ sc,
                            double* __restrict__ v1) {
    const double beta = sqrt(sc[0]);
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        v1[i] = beta > 0.0 ? gt[i] / beta : 0.0;
}

// alpha = beta h11 / (h11^2 + h21^2) if the denominator is positive, else 0
// (src/schur.cpp:197-204); y = alpha v1.
__global__ void k_step(i64 n, const double* __restrict__ sc, const double* __restrict__ v1,
                       double* __restrict__ y) {
    const double beta = sqrt(sc[0]), h11 = sc[1], h21sq = sc[2];
    const double denom = h11 * h11 + h21sq;
    const bool go = beta > 0.0 && denom > 0.0;
    const double alpha = go ? beta * h11 / denom : 0.0;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        y[i] = go ? alpha * v1[i] : 0.0;
}

} // namespace

void DeviceSchur::build(const Csr& A, const SmootherConfig& cfg, cudaStream_t st) {
    SchurSetup s = schur_partition(A, cfg.schur_blocks);
    n_ = A.nrows;
    ni_ = static_cast<i64>(s.interior_idx.size());
    nf_ = nf_global_ = static_cast<i64>(s.interface_idx.size());
    tr_ = nullptr;
    sell_from_host(C_, s.C, Part::all, st);
    std::vector<i32> perm(s.perm.begin(), s.perm.end());
    finish_build(s.B, s.E, s.F, perm, cfg, st, &s);
}

namespace {
void put_ids(std::vector<char>& b, const std::vector<i64>& v) {
    const char* c = reinterpret_cast<const char*>(v.data());
    b.insert(b.end(), c, c + v.size() * sizeof(i64));
}
std::vector<i64> get_ids(const std::vector<char>& b) {
    std::vector<i64> v(b.size() / sizeof(i64));
    if (!v.empty()) std::memcpy(v.data(), b.data(), v.size() * sizeof(i64));
    return v;
}
} // namespace

void DeviceSchur::build_dist(const HaloPlan& A, const Transport& t, const SmootherConfig& cfg, cudaStream_t st) {
    // partition (src/schur.cpp:19-105) with block b = rank b's rows: a row is
    // interface iff it couples across a cut — it reads another rank's column
    // (an off-block entry) or another rank reads it (it is in a send list)
    if (cfg.schur_blocks != A.nranks)
        fail_invalid("distributed schur_ilut: schur.blocks (" + std::to_string(cfg.schur_blocks) +
                     ") must equal the rank count (" + std::to_string(A.nranks) + ")");
    const i64 n = A.nloc;
    std::vector<char> iface(static_cast<size_t>(n), 0);
    for (i64 i = 0; i < n; ++i)
        if (A.A_off.rp[i + 1] > A.A_off.rp[i]) iface[i] = 1;
    for (i32 r : A.send_local) iface[r] = 1;
    std::vector<i32> perm(static_cast<size_t>(n));
    std::vector<i64> my_iface; // ascending global ids
    i64 ni = 0;
    for (i64 i = 0; i < n; ++i)
        if (!iface[i]) perm[i] = static_cast<i32>(ni++);
    for (i64 i = 0, k = 0; i < n; ++i)
        if (iface[i]) {
            perm[i] = static_cast<i32>(ni + k++);
            my_iface.push_back(A.row0 + i);
        }
    const i64 nf = static_cast<i64>(my_iface.size());
    // every rank's interface rows: global interface numbering = rank order, ascending ids
    std::vector<char> msg;
    put_ids(msg, my_iface);
    const auto all = t.allgather(msg);
    std::vector<std::vector<i64>> ids(all.size());
    RowPartition part;
    part.p = A.nranks;
    part.starts.push_back(0);
    for (size_t q = 0; q < all.size(); ++q) {
        ids[q] = get_ids(all[q]);
        part.starts.push_back(part.starts.back() + static_cast<i64>(ids[q].size()));
    }
    part.n = part.starts.back();
    auto owner_of_row = [&](i64 g) { // the row partition of A (contiguous blocks)
        for (i64 q = 0; q < A.nranks; ++q)
            if (!ids[q].empty() && g <= ids[q].back() && g >= ids[q].front()) return q;
        return i64{-1};
    };
    auto iface_pos = [&](i64 g) -> i64 {
        const i64 q = owner_of_row(g);
        if (q >= 0) {
            const auto it = std::lower_bound(ids[q].begin(), ids[q].end(), g);
            if (it != ids[q].end() && *it == g) return part.starts[q] + (it - ids[q].begin());
        }
        fail_invalid("distributed schur_ilut: an off-block column is not an interface row of its owner");
    };
    // B (interior x interior), E (interior x interface), F (interface x interior): block-local,
    // C (interface x interface) rows with global interface ids; entries in global column order
    Csr B, E, F, Crows;
    B.nrows = B.ncols = ni;
    E.nrows = ni, E.ncols = nf;
    F.nrows = nf, F.ncols = ni;
    Crows.nrows = nf, Crows.ncols = part.n;
    B.rp.assign(1, 0), E.rp.assign(1, 0), F.rp.assign(1, 0), Crows.rp.assign(1, 0);
    for (i64 i = 0; i < n; ++i) {
        const bool ri = !iface[i];
        for (i64 k = A.A_ext.rp[i]; k < A.A_ext.rp[i + 1]; ++k) {
            const i32 c = A.A_ext.ci[k];
            const double v = A.A_ext.v[k];
            if (c < n) {
                const i64 pc = perm[c];
                const bool ci = pc < ni;
                Csr& M = ri ? (ci ? B : E) : (ci ? F : Crows);
                M.ci.push_back(static_cast<i32>(ri || ci ? (ci ? pc : pc - ni) : part.starts[A.rank] + (pc - ni)));
                M.v.push_back(v);
            } else { // another rank's row: an interface column of C (interior rows have none)
                if (ri) fail_invalid("distributed schur_ilut: interior row with an off-block entry");
                Crows.ci.push_back(static_cast<i32>(iface_pos(A.halo_global[c - n])));
                Crows.v.push_back(v);
            }
        }
        if (ri) {
            B.rp.push_back(static_cast<i64>(B.ci.size()));
            E.rp.push_back(static_cast<i64>(E.ci.size()));
        } else {
            F.rp.push_back(static_cast<i64>(F.ci.size()));
            Crows.rp.push_back(static_cast<i64>(Crows.ci.size()));
        }
    }
    HaloPlan Cp = halo_plan(std::move(Crows), part, A.rank);
    plan_exchange(Cp, t);
    n_ = n;
    ni_ = ni;
    nf_ = nf;
    nf_global_ = part.n;
    tr_ = &t;
    Chx_.setup(Cp, t, st);
    sell_from_host(C_, Cp.A_ext, Part::all, st);
    finish_build(B, E, F, perm, cfg, st, nullptr);
}

void DeviceSchur::finish_build(const Csr& B, const Csr& E, const Csr& F, const std::vector<i32>& perm,
                               const SmootherConfig& cfg, cudaStream_t st, SchurSetup* host) {
    ts_ = cfg.trisolve;
    const bool rich = ts_.mode == TriSolveMode::richardson;
    if (rich && cfg.scaling == ScalingKind::none)
        fail_invalid("factorize_blocks: Richardson block solves require row or row/col scaling");
    // The interior matrix B is block diagonal, so factoring it whole on the
    // device gives every block's factors row for row (fill and thresholds stay
    // inside a block). Zero pivots are the exception — the reference patches /
    // reports them per block (block-local step, per-block |B_b|_F) — so any
    // failure of the device factorisation falls back to the per-block host
    // path, which reproduces the reference's result or error exactly.
    bool built = false;
    const bool dev = cfg.ilu_params.variant == IluVariant::ilu0 ? ilu0_on_device() : ilut_on_device();
    if (dev && ni_ > 0) {
        IluParams strict = cfg.ilu_params;
        strict.pivot_patch = PivotPatch::error;
        try {
            DevFactors df = factorize_resident(B, strict, st);
            blocks_.build(std::move(df), cfg.scaling, UpperIteration::scaled, !rich, st);
            built = true;
        } catch (const Error&) {
            built = false;
        }
    }
    if (!built && ni_ > 0) {
        if (host) {
            schur_factorize(*host, cfg.ilu_params, cfg.scaling, cfg.trisolve);
            blocks_ = DeviceIlu();
            blocks_.build(host->factors, cfg.scaling, UpperIteration::scaled, !rich, st);
        } else { // distributed: this rank's B is one block of the reference's factorize_blocks
            blocks_ = DeviceIlu();
            blocks_.build(ilu_factorize(B, cfg.ilu_params), cfg.scaling, UpperIteration::scaled, !rich, st);
        }
    }
    sell_from_host(E_, E, Part::all, st);
    sell_from_host(F_, F, Part::all, st);
    perm_.upload(perm.data(), n_, st);
    // ws: r(n) fg(n) t(ni) gt(nf) v1(nf) w(nf) tE(ni) tB(ni) upd(n) y(ni), then the L/U sweep scratch
    const i64 sweep_ws = blocks_.sweep_ws(std::max(ts_.m_lower, ts_.m_upper)) + std::max<i64>(ni_, 1);
    ws_.alloc(3 * n_ + 4 * ni_ + 3 * nf_ + ni_ + std::max<i64>(sweep_ws, 3 * ni_) + 8);
    red_.alloc(reduce_ws_doubles(std::max(n_, i64{1})));
    scal_.alloc(8);
    ILUG_CUDA(cudaStreamSynchronize(st));
}

void DeviceSchur::block_solve(const double* f, double* out, cudaStream_t st) const {
    if (ni_ == 0) return; // every row of the block is an interface row (thin blocks)
    // block_solve (src/schur.cpp:137-156) over the block-diagonal interior factor
    double* y = ws_.p + 3 * n_ + 4 * ni_ + 3 * nf_;
    double* scr = y + ni_;
    if (ts_.mode == TriSolveMode::direct) {
        blocks_.solve_lower(f, y, st);
        blocks_.solve_upper(y, out, scr, st);
    } else {
        blocks_.sweep_lower(f, y, ts_.m_lower, scr, st);
        blocks_.sweep_upper(y, out, ts_.m_upper, scr, st);
    }
}

void DeviceSchur::apply(const DeviceMatrix& A, const double* b, double* x, cudaStream_t st) const {
    double* r = ws_.p;
    double* fg = r + n_;         // [f | g]
    double* upd = fg + n_;       // [x_I | y]
    double* t = upd + n_;        // ni
    double* tE = t + ni_;        // ni
    double* tB = tE + ni_;       // ni
    double* fi = tB + ni_;       // ni
    double* gt = fi + ni_;       // nf
    double* v1 = gt + nf_;       // nf
    double* w = v1 + nf_;        // nf
    double* f = fg;
    double* g = fg + ni_;
    double* xI = upd;
    double* y = upd + ni_;
    double* sc = scal_.p;        // beta^2, h11, h21^2

    A.residual(x, b, r, st); // halo-exchanged when A holds a rank's rows
    k_split<<<grid_of(n_), kB, 0, st>>>(n_, perm_.p, r, fg);
    ILUG_LAUNCH_CHECK();
    if (nf_global_ > 0) { // collective when distributed: every rank takes the branch
        block_solve(f, t, st);
        residual(F_, t, g, gt, st);                   // gt = g - F B^-1 f
        nrm2sq_dev(gt, nf_, sc, red_.p, st);          // beta^2
        transport_allreduce(tr_, sc, 1, st);
        k_normalize<<<grid_of(nf_), kB, 0, st>>>(nf_, gt, sc, v1);
        ILUG_LAUNCH_CHECK();
        spmv(E_, v1, tE, st);                         // E v1
        block_solve(tE, tB, st);                      // B^-1 E v1
        if (tr_) {                                    // w = C v1 (C couples the ranks' interfaces)
            Chx_.exchange(v1, st);
            spmv_split(C_, v1, Chx_.halo.p, Chx_.nloc, w, st);
        } else {
            spmv(C_, v1, w, st);
        }
        residual(F_, tB, w, w, st);                   // w = w - F B^-1 E v1 (row-local: in-place safe)
        dot_dev(v1, w, nf_, sc + 1, red_.p, st);      // h11
        transport_allreduce(tr_, sc + 1, 1, st);
        nrm2sq_diff_dev(w, v1, sc + 1, nf_, sc + 2, red_.p, st); // h21^2
        transport_allreduce(tr_, sc + 2, 1, st);
        k_step<<<grid_of(nf_), kB, 0, st>>>(nf_, sc, v1, y);
        ILUG_LAUNCH_CHECK();
        residual(E_, y, f, fi, st);                   // f - E y
    } else {
        vec_copy(fi, f, ni_, st);
    }
    block_solve(fi, xI, st);
    k_merge<<<grid_of(n_), kB, 0, st>>>(n_, perm_.p, upd, x);
    ILUG_LAUNCH_CHECK();
}

} // namespace ilug
