#include "spsv_cusparse.hpp"

#include <cusparse.h>
#include <dlfcn.h>

#include <cstdlib>
#include <mutex>
#include <string>

namespace ilug {

namespace {

// cuSPARSE is bound lazily with dlopen (only ILUG_DIRECT=cusparse uses it), so
// libilug.so has no load-time dependency on it and never pins a second copy
// next to torch's. Prefers an already-loaded libcusparse.so.12.
struct Api {
#define ILUG_CS_FN(name) decltype(&::name) name = nullptr;
    ILUG_CS_FN(cusparseCreate)
    ILUG_CS_FN(cusparseDestroy)
    ILUG_CS_FN(cusparseSetStream)
    ILUG_CS_FN(cusparseCreateCsr)
    ILUG_CS_FN(cusparseDestroySpMat)
    ILUG_CS_FN(cusparseSpMatSetAttribute)
    ILUG_CS_FN(cusparseCreateDnVec)
    ILUG_CS_FN(cusparseDestroyDnVec)
    ILUG_CS_FN(cusparseDnVecSetValues)
    ILUG_CS_FN(cusparseSpSV_createDescr)
    ILUG_CS_FN(cusparseSpSV_destroyDescr)
    ILUG_CS_FN(cusparseSpSV_bufferSize)
    ILUG_CS_FN(cusparseSpSV_analysis)
    ILUG_CS_FN(cusparseSpSV_solve)
#undef ILUG_CS_FN
};

const Api& api() {
    static Api a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libcusparse.so.12", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libcusparse.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libcusparse.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
#define ILUG_CS_BIND(name) a.name = reinterpret_cast<decltype(a.name)>(dlsym(h, #name));
        ILUG_CS_BIND(cusparseCreate)
        ILUG_CS_BIND(cusparseDestroy)
        ILUG_CS_BIND(cusparseSetStream)
        ILUG_CS_BIND(cusparseCreateCsr)
        ILUG_CS_BIND(cusparseDestroySpMat)
        ILUG_CS_BIND(cusparseSpMatSetAttribute)
        ILUG_CS_BIND(cusparseCreateDnVec)
        ILUG_CS_BIND(cusparseDestroyDnVec)
        ILUG_CS_BIND(cusparseDnVecSetValues)
        ILUG_CS_BIND(cusparseSpSV_createDescr)
        ILUG_CS_BIND(cusparseSpSV_destroyDescr)
        ILUG_CS_BIND(cusparseSpSV_bufferSize)
        ILUG_CS_BIND(cusparseSpSV_analysis)
        ILUG_CS_BIND(cusparseSpSV_solve)
#undef ILUG_CS_BIND
    });
    if (!a.cusparseSpSV_solve) fail_invalid("ILUG_DIRECT=cusparse: libcusparse.so.12 could not be loaded");
    return a;
}

void ck(cusparseStatus_t s, const char* what) {
    if (s != CUSPARSE_STATUS_SUCCESS) fail_numeric(std::string("cusparse: ") + what + " failed (" +
                                                   std::to_string(static_cast<int>(s)) + ")");
}

__global__ void k_rp32(i64 n, const i64* __restrict__ rp, i32* __restrict__ out) {
    const i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i <= n) out[i] = static_cast<i32>(rp[i]);
}

} // namespace

struct CusparseTri::Impl {
    cusparseHandle_t h = nullptr;
    cusparseSpMatDescr_t mat = nullptr;
    cusparseDnVecDescr_t vb = nullptr, vx = nullptr;
    cusparseSpSVDescr_t sv = nullptr;
    DBuf<i32> rp, ci;
    DBuf<double> v, scratch_b, scratch_x;
    DBuf<char> buf;
    i64 n = 0;
    ~Impl() {
        if (sv) api().cusparseSpSV_destroyDescr(sv);
        if (vb) api().cusparseDestroyDnVec(vb);
        if (vx) api().cusparseDestroyDnVec(vx);
        if (mat) api().cusparseDestroySpMat(mat);
        if (h) api().cusparseDestroy(h);
    }
};

CusparseTri::CusparseTri() : p_(new Impl) {}
CusparseTri::~CusparseTri() = default;

bool direct_uses_cusparse() {
    const char* e = std::getenv("ILUG_DIRECT");
    return e && std::string(e) == "cusparse";
}

void CusparseTri::build(i64 n, const i64* rp, const i32* ci, const double* v, i64 nnz, bool lower,
                        cudaStream_t st) {
    Impl& m = *p_;
    m.n = n;
    if (nnz >= (i64{1} << 31)) fail_invalid("cusparse direct: more than 2^31-1 entries");
    ck(api().cusparseCreate(&m.h), "create");
    ck(api().cusparseSetStream(m.h, st), "set stream");
    m.rp.alloc(n + 1);
    m.ci.alloc(std::max<i64>(nnz, 1));
    m.v.alloc(std::max<i64>(nnz, 1));
    k_rp32<<<static_cast<unsigned>((n + 256) / 256), 256, 0, st>>>(n, rp, m.rp.p);
    ILUG_LAUNCH_CHECK();
    if (nnz > 0) {
        ILUG_CUDA(cudaMemcpyAsync(m.ci.p, ci, static_cast<size_t>(nnz) * 4, cudaMemcpyDeviceToDevice, st));
        ILUG_CUDA(cudaMemcpyAsync(m.v.p, v, static_cast<size_t>(nnz) * 8, cudaMemcpyDeviceToDevice, st));
    }
    ck(api().cusparseCreateCsr(&m.mat, n, n, nnz, m.rp.p, m.ci.p, m.v.p, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                         CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F),
       "create csr");
    cusparseFillMode_t fm = lower ? CUSPARSE_FILL_MODE_LOWER : CUSPARSE_FILL_MODE_UPPER;
    cusparseDiagType_t dt = lower ? CUSPARSE_DIAG_TYPE_UNIT : CUSPARSE_DIAG_TYPE_NON_UNIT;
    ck(api().cusparseSpMatSetAttribute(m.mat, CUSPARSE_SPMAT_FILL_MODE, &fm, sizeof fm), "fill mode");
    ck(api().cusparseSpMatSetAttribute(m.mat, CUSPARSE_SPMAT_DIAG_TYPE, &dt, sizeof dt), "diag type");
    m.scratch_b.alloc(std::max<i64>(n, 1));
    m.scratch_x.alloc(std::max<i64>(n, 1));
    ck(api().cusparseCreateDnVec(&m.vb, n, m.scratch_b.p, CUDA_R_64F), "vec b");
    ck(api().cusparseCreateDnVec(&m.vx, n, m.scratch_x.p, CUDA_R_64F), "vec x");
    ck(api().cusparseSpSV_createDescr(&m.sv), "spsv descr");
    const double one = 1.0;
    size_t ws = 0;
    ck(api().cusparseSpSV_bufferSize(m.h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, m.mat, m.vb, m.vx, CUDA_R_64F,
                               CUSPARSE_SPSV_ALG_DEFAULT, m.sv, &ws),
       "buffer size");
    m.buf.alloc(static_cast<i64>(std::max<size_t>(ws, 1)));
    ck(api().cusparseSpSV_analysis(m.h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, m.mat, m.vb, m.vx, CUDA_R_64F,
                             CUSPARSE_SPSV_ALG_DEFAULT, m.sv, m.buf.p),
       "analysis");
    ILUG_CUDA(cudaStreamSynchronize(st));
    ready_ = true;
}

void CusparseTri::solve(const double* b, double* x, cudaStream_t st) const {
    Impl& m = *p_;
    if (m.n == 0) return;
    ck(api().cusparseSetStream(m.h, st), "set stream");
    ck(api().cusparseDnVecSetValues(m.vb, const_cast<double*>(b)), "set b");
    ck(api().cusparseDnVecSetValues(m.vx, x), "set x");
    const double one = 1.0;
    ck(api().cusparseSpSV_solve(m.h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, m.mat, m.vb, m.vx, CUDA_R_64F,
                          CUSPARSE_SPSV_ALG_DEFAULT, m.sv),
       "solve");
}

} // namespace ilug
