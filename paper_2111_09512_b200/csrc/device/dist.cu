// Multi-GPU plumbing (one process per GPU): NCCL communicator from a
// caller-broadcast unique id, and the halo exchange of a row-block
// distributed operator — pack the rows other ranks need, then one grouped
// ncclSend/ncclRecv per neighbour (NVLink/NVSwitch underneath). Halo messages
// are small (one grid plane per neighbour for a z-slab partition), so the
// exchange is latency-bound; it is issued on the compute stream right before
// the residual kernel that consumes it.
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

} // namespace

void dist_unique_id(char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    ILUG_NCCL(nccl().GetUniqueId(&id));
    std::memcpy(out, &id, 128);
}

DistComm::DistComm(int nranks_, int rank_, const char id[128]) : nranks(nranks_), rank(rank_) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclComm_t c;
    ILUG_NCCL(nccl().CommInitRank(&c, nranks, uid, rank));
    comm = c;
}

DistComm::~DistComm() {
    if (comm) nccl().CommDestroy(static_cast<ncclComm_t>(comm));
}

void DistComm::allreduce_sum(double* buf, i64 count, cudaStream_t st) const {
    if (nranks == 1) return;
    ILUG_NCCL(nccl().AllReduce(buf, buf, static_cast<size_t>(count), ncclDouble, ncclSum,
                            static_cast<ncclComm_t>(comm), st));
}

void HaloExchange::exchange(const double* x, cudaStream_t st) const {
    const i64 ns = send_idx.n;
    if (ns > 0) {
        const unsigned g = static_cast<unsigned>(std::min<i64>((ns + 255) / 256, 4096));
        k_pack<<<g, 256, 0, st>>>(ns, send_idx.p, x, sendbuf.p);
        ILUG_LAUNCH_CHECK();
    }
    if (send_ranks.empty() && recv_ranks.empty()) return;
    auto c = static_cast<ncclComm_t>(comm);
    ILUG_NCCL(nccl().GroupStart());
    for (size_t k = 0; k < send_ranks.size(); ++k)
        ILUG_NCCL(nccl().Send(sendbuf.p + send_offsets[k], static_cast<size_t>(send_offsets[k + 1] - send_offsets[k]),
                           ncclDouble, static_cast<int>(send_ranks[k]), c, st));
    for (size_t k = 0; k < recv_ranks.size(); ++k)
        ILUG_NCCL(nccl().Recv(halo.p + recv_offsets[k], static_cast<size_t>(recv_offsets[k + 1] - recv_offsets[k]),
                           ncclDouble, static_cast<int>(recv_ranks[k]), c, st));
    ILUG_NCCL(nccl().GroupEnd());
}

namespace {
void setup_halo(HaloExchange& hx, DeviceMatrix& A, const HaloPlan& plan, const DistComm& comm, cudaStream_t st) {
    hx.comm = comm.comm;
    hx.nloc = plan.nloc;
    hx.nhalo = plan.nhalo;
    hx.recv_ranks = plan.recv_ranks;
    hx.recv_offsets = plan.recv_offsets;
    hx.send_ranks = plan.send_ranks;
    hx.send_offsets = plan.send_offsets;
    hx.send_idx.upload(plan.send_local.data(), static_cast<i64>(plan.send_local.size()), st);
    hx.sendbuf.alloc(static_cast<i64>(plan.send_local.size()));
    hx.halo.alloc(std::max<i64>(plan.nhalo, 1));
    A.build(plan.A_ext, st);
    A.n = plan.nloc;
    A.halo = &hx;
}
} // namespace

void DistSolver::build(const HaloPlan& plan, const DistComm& comm, const AmgParams& ap, bool use_graph,
                       cudaStream_t st) {
    comm_ = &comm;
    setup_halo(hx_, A_, plan, comm, st);
    A_diag_ = plan.A_diag;
    hh_ = amg_setup(A_diag_, ap);
    H_.set_use_graph(use_graph);
    H_.build(hh_, st);
    ILUG_CUDA(cudaStreamSynchronize(st));
}

KrylovReport DistSolver::solve(const double* b, double* x, const KrylovParams& p, cudaStream_t st) {
    KrylovParams q = p;
    // |A|_2 needs a global transpose (skipped across ranks); with the relres
    // criterion and no per-iteration iterates nothing in the solve reads it
    // (the single-process driver moves it out of the timed region likewise)
    if (comm_->nranks > 1 || (!q.form_iterates && !q.nrbe_criterion)) q.estimate_anorm = false;
    return device_gmres(A_, A_diag_, H_, b, x, q, st, comm_);
}

void DistSmoother::build(const HaloPlan& plan, const DistComm& comm, const SmootherConfig& cfg, cudaStream_t st) {
    if (cfg.kind != SmootherKind::ilu) fail_invalid("distributed smoother: smoother.kind must be ilu");
    if (plan.nranks > 1 && plan.send_offsets.size() != plan.send_ranks.size() + (plan.send_ranks.empty() ? 0 : 1))
        fail_invalid("distributed smoother: halo sends not set");
    hx_.comm = comm.comm;
    hx_.nloc = plan.nloc;
    hx_.nhalo = plan.nhalo;
    hx_.recv_ranks = plan.recv_ranks;
    hx_.recv_offsets = plan.recv_offsets;
    hx_.send_ranks = plan.send_ranks;
    hx_.send_offsets = plan.send_offsets;
    hx_.send_idx.upload(plan.send_local.data(), static_cast<i64>(plan.send_local.size()), st);
    hx_.sendbuf.alloc(static_cast<i64>(plan.send_local.size()));
    hx_.halo.alloc(std::max<i64>(plan.nhalo, 1));
    A_.build(plan.A_ext, st);
    A_.n = plan.nloc;
    A_.halo = &hx_;
    // block-Jacobi: the ILU factors of this rank's diagonal block
    s_.build(plan.A_diag, A_, cfg, st);
    ILUG_CUDA(cudaStreamSynchronize(st));
}

} // namespace ilug
