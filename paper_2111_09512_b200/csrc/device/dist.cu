// Multi-GPU plumbing and the row-block distributed solve phase (dist.hpp).
//
// Halo messages are small (one grid plane per neighbour for a z-slab
// partition), so an exchange is latency-bound; it is issued on the compute
// stream right before the product that consumes it. Sums are stream-ordered
// NCCL all-reduces (GMRES reductions, the coarsest right-hand side).
#include "dist.hpp"

#include <nccl.h> // types only: the library is bound at run time (below)

#include <dlfcn.h>

#include <cstdlib>

namespace ilug {

namespace {

// NCCL is resolved lazily with dlopen on first multi-GPU use, never linked:
// (1) an already-loaded libnccl.so.2 (torch's, in a torch process) is reused;
// (2) else ILUG_NCCL_LIB (set by paper_2111_09512_b200.dist to torch's bundled
// copy) or the system libnccl.so.2. Linking the system 2.27 at build time would
// shadow torch's 2.28 by SONAME and break `import torch` afterwards.
struct NcclApi {
    decltype(&ncclGetUniqueId) GetUniqueId;
    decltype(&ncclCommInitRank) CommInitRank;
    decltype(&ncclCommDestroy) CommDestroy;
    decltype(&ncclAllReduce) AllReduce;
    decltype(&ncclAllGather) AllGather;
    decltype(&ncclSend) Send;
    decltype(&ncclRecv) Recv;
    decltype(&ncclGroupStart) GroupStart;
    decltype(&ncclGroupEnd) GroupEnd;
    decltype(&ncclGetErrorString) GetErrorString;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* env = std::getenv("ILUG_NCCL_LIB");
            h = dlopen(env && *env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        }
        if (!h) fail_invalid(std::string("NCCL library not found (set ILUG_NCCL_LIB): ") + dlerror());
        NcclApi a{};
        auto bind = [&](auto& fp, const char* name) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, name));
            if (!fp) fail_invalid(std::string("NCCL symbol missing: ") + name);
        };
        bind(a.GetUniqueId, "ncclGetUniqueId");
        bind(a.CommInitRank, "ncclCommInitRank");
        bind(a.CommDestroy, "ncclCommDestroy");
        bind(a.AllReduce, "ncclAllReduce");
        bind(a.AllGather, "ncclAllGather");
        bind(a.Send, "ncclSend");
        bind(a.Recv, "ncclRecv");
        bind(a.GroupStart, "ncclGroupStart");
        bind(a.GroupEnd, "ncclGroupEnd");
        bind(a.GetErrorString, "ncclGetErrorString");
        return a;
    }();
    return api;
}

[[noreturn]] void nccl_fail(ncclResult_t r, const char* what) {
    fail_numeric(std::string("NCCL error ") + nccl().GetErrorString(r) + " in " + what);
}
#define ILUG_NCCL(call)                                   \
    do {                                                  \
        ncclResult_t r__ = (call);                        \
        if (r__ != ncclSuccess) nccl_fail(r__, #call);    \
    } while (0)

__global__ void k_pack(i64 n, const i32* __restrict__ idx, const double* __restrict__ x, double* __restrict__ out) {
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<i64>(gridDim.x) * blockDim.x)
        out[i] = x[idx[i]];
}

// ---------------------------------------------------------------- NCCL transport
class NcclTransport final : public Transport {
public:
    NcclTransport(int p, int r, const char id[128]) {
        nranks = p;
        rank = r;
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        ILUG_NCCL(nccl().CommInitRank(&comm_, nranks, uid, rank));
    }
    ~NcclTransport() override {
        if (comm_) nccl().CommDestroy(comm_);
    }
    void allreduce_sum(double* buf, i64 count, cudaStream_t st) const override {
        ILUG_NCCL(nccl().AllReduce(buf, buf, static_cast<size_t>(count), ncclDouble, ncclSum, comm_, st));
    }
    void exchange(const HaloExchange& hx, cudaStream_t st) const override {
        if (hx.send_ranks.empty() && hx.recv_ranks.empty()) return;
        ILUG_NCCL(nccl().GroupStart());
        for (size_t k = 0; k < hx.send_ranks.size(); ++k)
            ILUG_NCCL(nccl().Send(hx.sendbuf.p + hx.send_offsets[k],
                                  static_cast<size_t>(hx.send_offsets[k + 1] - hx.send_offsets[k]), ncclDouble,
                                  static_cast<int>(hx.send_ranks[k]), comm_, st));
        for (size_t k = 0; k < hx.recv_ranks.size(); ++k)
            ILUG_NCCL(nccl().Recv(hx.halo.p + hx.recv_offsets[k],
                                  static_cast<size_t>(hx.recv_offsets[k + 1] - hx.recv_offsets[k]), ncclDouble,
                                  static_cast<int>(hx.recv_ranks[k]), comm_, st));
        ILUG_NCCL(nccl().GroupEnd());
    }
    std::vector<std::vector<char>> allgather(const std::vector<char>& mine) const override {
        // lengths, then the payloads padded to the longest (setup only)
        DBuf<i64> lens(nranks);
        const i64 my = static_cast<i64>(mine.size());
        ILUG_CUDA(cudaMemcpy(lens.p + rank, &my, sizeof my, cudaMemcpyHostToDevice));
        ILUG_NCCL(nccl().AllGather(lens.p + rank, lens.p, 1, ncclInt64, comm_, nullptr));
        std::vector<i64> hl(static_cast<size_t>(nranks));
        ILUG_CUDA(cudaMemcpy(hl.data(), lens.p, sizeof(i64) * nranks, cudaMemcpyDeviceToHost));
        const i64 w = std::max<i64>(1, *std::max_element(hl.begin(), hl.end()));
        DBuf<char> all(w * nranks);
        if (my > 0) ILUG_CUDA(cudaMemcpy(all.p + rank * w, mine.data(), static_cast<size_t>(my), cudaMemcpyHostToDevice));
        ILUG_NCCL(nccl().AllGather(all.p + rank * w, all.p, static_cast<size_t>(w), ncclChar, comm_, nullptr));
        std::vector<char> h(static_cast<size_t>(w * nranks));
        ILUG_CUDA(cudaMemcpy(h.data(), all.p, h.size(), cudaMemcpyDeviceToHost));
        std::vector<std::vector<char>> out(static_cast<size_t>(nranks));
        for (int q = 0; q < nranks; ++q) out[q].assign(h.begin() + q * w, h.begin() + q * w + hl[q]);
        return out;
    }

private:
    ncclComm_t comm_ = nullptr;
};

// ------------------------------------------------- in-process (threads) transport
class LocalTransport final : public Transport {
public:
    LocalTransport(std::shared_ptr<LocalGroup> g, int r) : g_(std::move(g)) {
        nranks = g_->size();
        rank = r;
        if (r < 0 || r >= nranks) fail_invalid("local transport: rank out of range");
    }
    void allreduce_sum(double* buf, i64 count, cudaStream_t st) const override {
        // every rank sums the same staged copies in rank order: identical results
        auto& mine = g_->stage[static_cast<size_t>(rank)];
        mine.resize(static_cast<size_t>(count));
        ILUG_CUDA(cudaMemcpyAsync(mine.data(), buf, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
        g_->barrier();
        std::vector<double> sum(static_cast<size_t>(count), 0.0);
        for (int q = 0; q < nranks; ++q) {
            const auto& v = g_->stage[static_cast<size_t>(q)];
            if (static_cast<i64>(v.size()) != count) fail_invalid("local allreduce: ranks disagree on the count");
            for (i64 i = 0; i < count; ++i) sum[i] = q == 0 ? v[i] : sum[i] + v[i];
        }
        g_->barrier(); // every rank has read the stages
        ILUG_CUDA(cudaMemcpyAsync(buf, sum.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
        ILUG_CUDA(cudaStreamSynchronize(st));
    }
    void exchange(const HaloExchange& hx, cudaStream_t st) const override {
        ILUG_CUDA(cudaStreamSynchronize(st)); // the pack kernel has written sendbuf
        g_->slot[static_cast<size_t>(rank)] = &hx;
        g_->barrier();
        for (size_t k = 0; k < hx.recv_ranks.size(); ++k) {
            const auto* src = static_cast<const HaloExchange*>(g_->slot[static_cast<size_t>(hx.recv_ranks[k])]);
            const i64 cnt = hx.recv_offsets[k + 1] - hx.recv_offsets[k];
            size_t s = 0;
            while (s < src->send_ranks.size() && src->send_ranks[s] != rank) ++s;
            if (s == src->send_ranks.size() || src->send_offsets[s + 1] - src->send_offsets[s] != cnt)
                fail_invalid("local exchange: halo plans of the ranks do not match");
            ILUG_CUDA(cudaMemcpyAsync(hx.halo.p + hx.recv_offsets[k], src->sendbuf.p + src->send_offsets[s],
                                      sizeof(double) * cnt, cudaMemcpyDefault, st));
        }
        ILUG_CUDA(cudaStreamSynchronize(st));
        g_->barrier(); // nobody repacks its send buffer before every peer has copied it
    }
    std::vector<std::vector<char>> allgather(const std::vector<char>& mine) const override {
        g_->slot[static_cast<size_t>(rank)] = &mine;
        g_->barrier();
        std::vector<std::vector<char>> out;
        for (int q = 0; q < nranks; ++q) out.push_back(*static_cast<const std::vector<char>*>(g_->slot[q]));
        g_->barrier();
        return out;
    }

private:
    std::shared_ptr<LocalGroup> g_;
};

void put_i64(std::vector<char>& b, i64 v) {
    const char* c = reinterpret_cast<const char*>(&v);
    b.insert(b.end(), c, c + sizeof v);
}
i64 get_i64(const std::vector<char>& b, size_t& pos) {
    if (pos + sizeof(i64) > b.size()) fail_invalid("plan exchange: truncated message");
    i64 v;
    std::memcpy(&v, b.data() + pos, sizeof v);
    pos += sizeof v;
    return v;
}

} // namespace

// ---------------------------------------------------------------- public pieces
void dist_unique_id(char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    ILUG_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(out, &id, 128);
}

std::unique_ptr<Transport> make_nccl_transport(int nranks, int rank, const char id[128]) {
    return std::make_unique<NcclTransport>(nranks, rank, id);
}

LocalGroup::LocalGroup(int nranks) : slot(static_cast<size_t>(nranks)), stage(static_cast<size_t>(nranks)), p_(nranks) {
    if (nranks < 1) fail_invalid("local group: nranks must be >= 1");
}

void LocalGroup::barrier() {
    std::unique_lock<std::mutex> l(m_);
    if (aborted_) fail_invalid("local rank group aborted: another rank failed");
    const unsigned long long g = gen_;
    if (++arrived_ == p_) {
        arrived_ = 0;
        ++gen_;
        cv_.notify_all();
        return;
    }
    cv_.wait(l, [&] { return gen_ != g || aborted_; });
    if (gen_ == g) fail_invalid("local rank group aborted: another rank failed");
}

void LocalGroup::abort() {
    std::lock_guard<std::mutex> l(m_);
    aborted_ = true;
    cv_.notify_all();
}

std::unique_ptr<Transport> make_local_transport(std::shared_ptr<LocalGroup> g, int rank) {
    return std::make_unique<LocalTransport>(std::move(g), rank);
}

HaloExchange::~HaloExchange() {
    if (cst_) cudaStreamSynchronize(cst_), cudaStreamDestroy(cst_);
    if (packed_) cudaEventDestroy(packed_);
    if (done_) cudaEventDestroy(done_);
}

void HaloExchange::begin(const double* x, cudaStream_t st) const {
    if (pending_) end(st); // a begin without its end: keep the buffers ordered
    const i64 ns = send_idx.n;
    if (ns > 0) {
        const unsigned g = static_cast<unsigned>(std::min<i64>((ns + 255) / 256, 4096));
        k_pack<<<g, 256, 0, st>>>(ns, send_idx.p, x, sendbuf.p);
        ILUG_LAUNCH_CHECK();
    }
    if (!(tr && tr->nranks > 1)) return;
    // the transfer on the exchange's stream, after the pack; the previous
    // exchange's readers of halo (and writers of sendbuf) are ordered before
    // this pack on the caller's stream, so the buffers are free
    ILUG_CUDA(cudaEventRecord(packed_, st));
    ILUG_CUDA(cudaStreamWaitEvent(cst_, packed_, 0));
    tr->exchange(*this, cst_);
    ILUG_CUDA(cudaEventRecord(done_, cst_));
    pending_ = true;
}

void HaloExchange::end(cudaStream_t st) const {
    if (!pending_) return;
    ILUG_CUDA(cudaStreamWaitEvent(st, done_, 0));
    pending_ = false;
}

void plan_exchange(HaloPlan& plan, const Transport& t) {
    if (t.nranks != plan.nranks || t.rank != plan.rank) fail_invalid("plan exchange: plan and transport ranks differ");
    // message: for every destination q: count, then the global ids wanted from q
    std::vector<char> mine;
    for (i64 q = 0; q < plan.nranks; ++q) {
        const std::vector<i64> ids = q == plan.rank ? std::vector<i64>{} : halo_requests(plan, q);
        put_i64(mine, static_cast<i64>(ids.size()));
        for (i64 g : ids) put_i64(mine, g);
    }
    const auto all = t.allgather(mine);
    plan.send_ranks.clear();
    plan.send_offsets.clear();
    plan.send_local.clear();
    for (i64 q = 0; q < plan.nranks; ++q) {
        if (q == plan.rank) continue;
        size_t pos = 0;
        std::vector<i64> wanted;
        for (i64 d = 0; d < plan.nranks; ++d) {
            const i64 cnt = get_i64(all[q], pos);
            for (i64 i = 0; i < cnt; ++i) {
                const i64 g = get_i64(all[q], pos);
                if (d == plan.rank) wanted.push_back(g);
            }
        }
        if (!wanted.empty()) halo_set_sends(plan, q, wanted);
    }
}

void HaloExchange::setup(const HaloPlan& plan, const Transport& t, cudaStream_t st) {
    tr = &t;
    nloc = plan.nloc;
    nhalo = plan.nhalo;
    recv_ranks = plan.recv_ranks;
    recv_offsets = plan.recv_offsets;
    send_ranks = plan.send_ranks;
    send_offsets = plan.send_offsets;
    send_idx.upload(plan.send_local.data(), static_cast<i64>(plan.send_local.size()), st);
    sendbuf.alloc(static_cast<i64>(plan.send_local.size()));
    halo.alloc(std::max<i64>(plan.nhalo, 1));
    if (t.nranks > 1 && !cst_) {
        ILUG_CUDA(cudaStreamCreateWithFlags(&cst_, cudaStreamNonBlocking));
        ILUG_CUDA(cudaEventCreateWithFlags(&packed_, cudaEventDisableTiming));
        ILUG_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
    }
}

void transport_allreduce(const Transport* t, double* buf, i64 count, cudaStream_t st) {
    if (t && t->nranks > 1) t->allreduce_sum(buf, count, st);
}

void DistOperator::build(const HaloPlan& plan, const Transport& t, cudaStream_t st) {
    hx.setup(plan, t, st);
    sell_from_host_split(M.A, plan.A_ext, plan.nloc, st); // local-only rows first: they overlap the exchange
    M.n = plan.A_ext.nrows;
    M.halo = &hx;
}

// ---------------------------------------------------------------- smoother
void DistSmoother::build(const HaloPlan& plan, const DistComm& comm, const SmootherConfig& cfg, cudaStream_t st) {
    if (plan.nranks > 1 && plan.send_offsets.size() != plan.send_ranks.size() + (plan.send_ranks.empty() ? 0 : 1))
        fail_invalid("distributed smoother: halo sends not set");
    op_.build(plan, *comm.t, st);
    s_.build(plan.diag(), op_.M, cfg, st, nullptr, &plan); // rank-local factors / level plans
    ILUG_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------- hierarchy
void DistHierarchy::build(const HostHierarchy& h, const DistComm& comm, cudaStream_t st) {
    comm_ = &comm;
    const Transport& t = *comm.t;
    const int L = static_cast<int>(h.num_levels());
    if (L < 1) fail_invalid("distributed AMG: empty hierarchy");
    nlev_ = L;
    nu_ = h.params.cycles_nu;
    levels_.clear();
    SetupTimer tm("dist");
    std::vector<DistLevelPlan> plans = dist_level_plans(h, comm.nranks, comm.rank);
    tm.mark("level plans");
    for (int k = 0; k + 1 < L; ++k) {
        DistLevelPlan& d = plans[k];
        Lev& lv = levels_.emplace_back();
        lv.n = d.A.nloc;
        lv.row0 = d.A.row0;
        lv.last = d.last;
        plan_exchange(d.A, t);
        lv.A.build(d.A, t, st);
        if (!d.last) {
            plan_exchange(d.R, t);
            lv.R.build(d.R, t, st);
            plan_exchange(d.P, t);
            lv.P.build(d.P, t, st);
        } else {
            sell_from_host(lv.R_full, d.R_full, Part::all, st);
            sell_from_host(lv.P_rows, d.P_rows, Part::all, st);
            gather_.alloc(std::max<i64>(d.n, 1));
        }
        tm.mark("operators", k);
        lv.smoother.build(d.A.diag(), lv.A.M, h.params.plan.for_level(k), st, nullptr, &d.A);
        tm.mark("smoother", k);
        lv.b.alloc(std::max<i64>(lv.n, 1));
        lv.x.alloc(std::max<i64>(lv.n, 1));
        lv.r.alloc(std::max<i64>(lv.n, 1));
    }
    const Csr& Ac = h.levels[L - 1].A;
    coarse_n_ = Ac.nrows;
    lu_.upload(h.coarse.lu.data(), static_cast<i64>(h.coarse.lu.size()), st);
    piv_.upload(h.coarse.piv.data(), static_cast<i64>(h.coarse.piv.size()), st);
    cb_.alloc(std::max<i64>(coarse_n_, 1));
    cx_.alloc(std::max<i64>(coarse_n_, 1));
    if (L == 1) { // the only level is the replicated coarse solve; GMRES still needs this rank's rows
        const RowPartition part = row_partition(coarse_n_, comm.nranks);
        HaloPlan plan = halo_plan(csr_row_block(Ac, part.starts[comm.rank], part.starts[comm.rank + 1]), part,
                                  comm.rank);
        plan_exchange(plan, t);
        coarse_A_.build(plan, t, st);
        row0_ = plan.row0;
    } else {
        row0_ = levels_[0].row0;
    }
    ILUG_CUDA(cudaStreamSynchronize(st));
}

void DistHierarchy::cycle(int k, bool x_zero, cudaStream_t st) {
    Lev& lv = levels_[k];
    lv.smoother.smooth(lv.b.p, lv.x.p, x_zero, st);
    lv.A.M.residual(lv.x.p, lv.b.p, lv.r.p, st);
    if (!lv.last) {
        Lev& nx = levels_[k + 1];
        lv.R.M.spmv(lv.r.p, nx.b.p, st); // halo of the fine residual
        vec_zero(nx.x.p, nx.n, st);
        for (i64 i = 0; i < nu_; ++i) cycle(k + 1, i == 0, st);
        lv.P.hx.begin(nx.x.p, st); // halo of the coarse correction; local rows overlap it
        const HaloWait w = lv.P.hx.waiter();
        spmv_add_split(lv.P.M.A, nx.x.p, lv.P.hx.halo.p, lv.P.hx.nloc, lv.x.p, st, &w);
    } else {
        // coarsest: all-gather this level's residual (zero-padded sum: exact),
        // form the whole coarse right-hand side, solve it on every rank
        const i64 N = gather_.n;
        vec_zero(gather_.p, N, st);
        vec_copy(gather_.p + lv.row0, lv.r.p, lv.n, st);
        comm_->allreduce_sum(gather_.p, N, st);
        spmv(lv.R_full, gather_.p, cb_.p, st);
        dense_lu_solve_dev(coarse_n_, lu_.p, piv_.p, cb_.p, cx_.p, st); // nu solves of one rhs: one
        spmv_add(lv.P_rows, cx_.p, lv.x.p, st);
    }
    lv.smoother.smooth(lv.b.p, lv.x.p, false, st);
}

void DistHierarchy::vcycle(const double* r, double* z, cudaStream_t st) {
    if (levels_.empty()) {
        const i64 n = coarse_A_.M.n;
        vec_zero(cb_.p, coarse_n_, st);
        vec_copy(cb_.p + row0_, r, n, st);
        comm_->allreduce_sum(cb_.p, coarse_n_, st);
        dense_lu_solve_dev(coarse_n_, lu_.p, piv_.p, cb_.p, cx_.p, st);
        vec_copy(z, cx_.p + row0_, n, st);
        return;
    }
    Lev& l0 = levels_[0];
    vec_copy(l0.b.p, r, l0.n, st);
    vec_zero(l0.x.p, l0.n, st);
    cycle(0, true, st);
    vec_copy(z, l0.x.p, l0.n, st);
}

// ---------------------------------------------------------------- GMRES
void DistSolver::build(const HostHierarchy& h, const DistComm& comm, cudaStream_t st) {
    comm_ = &comm;
    H_.build(h, comm, st);
}

KrylovReport DistSolver::solve(const double* b, double* x, const KrylovParams& p, cudaStream_t st) {
    KrylovParams q = p;
    q.estimate_anorm = false; // |A|_2 needs a global transpose: not formed across ranks
    auto M = [this](const double* r, double* z, cudaStream_t s) { H_.vcycle(r, z, s); };
    return device_gmres(H_.A0(), nullptr, M, b, x, q, st, comm_, &work_);
}

} // namespace ilug
