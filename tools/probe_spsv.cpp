// Sanity check of the direct (level-scheduled) comparison point against
// cuSPARSE SpSV on the same ILUT factors (not a test, not the bench):
//
//   g++ -O2 -std=c++17 tools/probe_spsv.cpp -Iinclude -I/usr/local/cuda/include \
//       -Lpaper_2111_09512_b200 -lilug -L/usr/local/cuda/lib64 -lcusparse -lcudart \
//       -Wl,-rpath,$PWD/paper_2111_09512_b200 -o /tmp/probe_spsv && /tmp/probe_spsv [SPEC]
//
// Times one lower (unit) and one upper triangular solve of the C2 ILUT(1e-3,5)
// factors with ilug_solve_lower/upper (K5) and with cusparseSpSV_solve.
#include "ilug.h"

#include <cuda_runtime.h>
#include <cusparse.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        if ((x) != 0) {                                                             \
            std::fprintf(stderr, "%s failed (%d): %s\n", #x, (int)(x), iluamg_last_error()); \
            std::exit(1);                                                           \
        }                                                                           \
    } while (0)

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main(int argc, char** argv) {
    const char* spec = argc > 1 ? argv[1] : "pressure27(256,256,256)";
    iluamg_matrix* A = nullptr;
    CK(iluamg_matrix_generate(spec, &A));
    iluamg_config* cfg = nullptr;
    CK(iluamg_config_create(&cfg));
    CK(iluamg_config_set(cfg, "ilu.variant", "ilut"));
    CK(iluamg_config_set(cfg, "ilu.droptol", "1e-3"));
    CK(iluamg_config_set(cfg, "ilu.lfill", "5"));
    iluamg_matrix *L = nullptr, *U = nullptr;
    CK(ilug_ilu_factorize_device(A, cfg, &L, &U));
    const long long n = iluamg_matrix_rows(A);

    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double *b = nullptr, *x = nullptr;
    cudaMalloc(&b, n * sizeof(double));
    cudaMalloc(&x, n * sizeof(double));
    std::vector<double> hb(n);
    for (long long i = 0; i < n; ++i) hb[i] = 1.0 + (i % 7) * 0.125;
    cudaMemcpy(b, hb.data(), n * sizeof(double), cudaMemcpyHostToDevice);
    const int reps = 5;

    // ---- ours (K5, unscaled U: upper_iteration = jacobi keeps D, direct plans)
    ilug_factors* f = nullptr;
    CK(ilug_factors_create(A, cfg, 0, 1, 1, &f));
    for (int w = 0; w < 2; ++w) {
        CK(ilug_solve_lower(f, b, x, nullptr));
        CK(ilug_solve_upper(f, b, x, nullptr));
    }
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) CK(ilug_solve_lower(f, b, x, nullptr));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    const float our_l = time_ms(e0, e1) / reps;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) CK(ilug_solve_upper(f, b, x, nullptr));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    const float our_u = time_ms(e0, e1) / reps;

    // ---- K5 schedule variants (env knobs read per launch): "SUB=4,SLEEP=32,WARPS=8" ...
    // each checked bitwise against the default schedule's solution
    {
        std::vector<double> ref_l(n), ref_u(n), got(n);
        CK(ilug_solve_lower(f, b, x, nullptr));
        cudaMemcpy(ref_l.data(), x, n * sizeof(double), cudaMemcpyDeviceToHost);
        CK(ilug_solve_upper(f, b, x, nullptr));
        cudaMemcpy(ref_u.data(), x, n * sizeof(double), cudaMemcpyDeviceToHost);
        for (int a = 2; a < argc; ++a) {
            std::string cfgs = argv[a];
            unsetenv("ILUG_VF_SUB"), unsetenv("ILUG_VF_SLEEP"), unsetenv("ILUG_VF_WARPS");
            size_t pos = 0;
            while (pos < cfgs.size()) {
                size_t comma = cfgs.find(',', pos);
                if (comma == std::string::npos) comma = cfgs.size();
                const std::string kv = cfgs.substr(pos, comma - pos);
                const size_t eq = kv.find('=');
                setenv(("ILUG_VF_" + kv.substr(0, eq)).c_str(), kv.substr(eq + 1).c_str(), 1);
                pos = comma + 1;
            }
            float t[2];
            bool same[2];
            for (int part = 0; part < 2; ++part) {
                auto solve = [&] { CK(part == 0 ? ilug_solve_lower(f, b, x, nullptr) : ilug_solve_upper(f, b, x, nullptr)); };
                solve();
                cudaMemcpy(got.data(), x, n * sizeof(double), cudaMemcpyDeviceToHost);
                same[part] = std::memcmp(got.data(), part == 0 ? ref_l.data() : ref_u.data(), n * sizeof(double)) == 0;
                cudaDeviceSynchronize();
                cudaEventRecord(e0);
                for (int r = 0; r < reps; ++r) solve();
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                t[part] = time_ms(e0, e1) / reps;
            }
            std::printf("{\"variant\": \"%s\", \"lower_ms\": %.3f, \"upper_ms\": %.3f, \"bitwise\": [%s, %s]}\n",
                        cfgs.c_str(), t[0], t[1], same[0] ? "true" : "false", same[1] ? "true" : "false");
            std::fflush(stdout);
        }
        unsetenv("ILUG_VF_SUB"), unsetenv("ILUG_VF_SLEEP"), unsetenv("ILUG_VF_WARPS");
    }

    // ---- cuSPARSE SpSV on the same factors
    cusparseHandle_t h;
    cusparseCreate(&h);
    float cs_ms[2] = {0, 0}, cs_an[2] = {0, 0};
    for (int part = 0; part < 2; ++part) {
        iluamg_matrix* M = part == 0 ? L : U;
        const long long nnz = iluamg_matrix_nnz(M);
        std::vector<long long> rp(n + 1), ci(nnz);
        std::vector<double> v(nnz);
        CK(ilug_matrix_copy_csr(M, rp.data(), ci.data(), v.data()));
        std::vector<int> rp32(n + 1), ci32(nnz);
        for (long long i = 0; i <= n; ++i) rp32[i] = (int)rp[i];
        for (long long k = 0; k < nnz; ++k) ci32[k] = (int)ci[k];
        int *drp, *dci;
        double* dv;
        cudaMalloc(&drp, (n + 1) * sizeof(int));
        cudaMalloc(&dci, nnz * sizeof(int));
        cudaMalloc(&dv, nnz * sizeof(double));
        cudaMemcpy(drp, rp32.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice);
        cudaMemcpy(dci, ci32.data(), nnz * sizeof(int), cudaMemcpyHostToDevice);
        cudaMemcpy(dv, v.data(), nnz * sizeof(double), cudaMemcpyHostToDevice);
        cusparseSpMatDescr_t mat;
        cusparseCreateCsr(&mat, n, n, nnz, drp, dci, dv, CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                          CUSPARSE_INDEX_BASE_ZERO, CUDA_R_64F);
        cusparseFillMode_t fm = part == 0 ? CUSPARSE_FILL_MODE_LOWER : CUSPARSE_FILL_MODE_UPPER;
        cusparseDiagType_t dt = part == 0 ? CUSPARSE_DIAG_TYPE_UNIT : CUSPARSE_DIAG_TYPE_NON_UNIT;
        cusparseSpMatSetAttribute(mat, CUSPARSE_SPMAT_FILL_MODE, &fm, sizeof fm);
        cusparseSpMatSetAttribute(mat, CUSPARSE_SPMAT_DIAG_TYPE, &dt, sizeof dt);
        cusparseDnVecDescr_t vb, vx;
        cusparseCreateDnVec(&vb, n, b, CUDA_R_64F);
        cusparseCreateDnVec(&vx, n, x, CUDA_R_64F);
        cusparseSpSVDescr_t sv;
        cusparseSpSV_createDescr(&sv);
        const double one = 1.0;
        size_t ws = 0;
        cusparseSpSV_bufferSize(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, mat, vb, vx, CUDA_R_64F,
                                CUSPARSE_SPSV_ALG_DEFAULT, sv, &ws);
        void* buf = nullptr;
        cudaMalloc(&buf, ws ? ws : 1);
        cudaEventRecord(e0);
        cusparseSpSV_analysis(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, mat, vb, vx, CUDA_R_64F,
                              CUSPARSE_SPSV_ALG_DEFAULT, sv, buf);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cs_an[part] = time_ms(e0, e1);
        for (int w = 0; w < 2; ++w)
            cusparseSpSV_solve(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, mat, vb, vx, CUDA_R_64F,
                               CUSPARSE_SPSV_ALG_DEFAULT, sv);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < reps; ++r)
            cusparseSpSV_solve(h, CUSPARSE_OPERATION_NON_TRANSPOSE, &one, mat, vb, vx, CUDA_R_64F,
                               CUSPARSE_SPSV_ALG_DEFAULT, sv);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cs_ms[part] = time_ms(e0, e1) / reps;
        cusparseSpSV_destroyDescr(sv);
        cusparseDestroyDnVec(vb);
        cusparseDestroyDnVec(vx);
        cusparseDestroySpMat(mat);
        cudaFree(buf), cudaFree(drp), cudaFree(dci), cudaFree(dv);
    }
    long long nl = 0, nu = 0, pad = 0, nn = 0;
    int lvl_l = 0, lvl_u = 0;
    CK(ilug_factors_stats(f, &nn, &nl, &nu, &pad, &lvl_l, &lvl_u));
    std::printf("{\"spec\": \"%s\", \"n\": %lld, \"levels_L\": %d, \"levels_U\": %d, "
                "\"ours_lower_ms\": %.3f, \"ours_upper_ms\": %.3f, \"cusparse_lower_ms\": %.3f, "
                "\"cusparse_upper_ms\": %.3f, \"cusparse_analysis_ms\": [%.1f, %.1f]}\n",
                spec, n, lvl_l, lvl_u, our_l, our_u, cs_ms[0], cs_ms[1], cs_an[0], cs_an[1]);
    return 0;
}
