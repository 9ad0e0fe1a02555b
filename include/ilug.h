/*
 * ilug: the device-handle C ABI of the hot path — the plug points inside the
 * reference's solve phase, each taking DEVICE pointers and a cudaStream_t
 * (passed as void*). Handles own device memory and are read-only after
 * creation except where noted; every call returns an ILUAMG_* status with
 * the message in ilug_last_error() (same thread-local slot as
 * iluamg_last_error()). Nothing here synchronises the stream unless stated.
 *
 * Reference interfaces replaced (file:line in /root/reference/proj):
 *   ilug_factors_*      IluFactors + ilu_factorize/row_scale/row_col_scale
 *                       (include/iluamg/ilu.hpp:33-62, src/ilu.cpp:271-333)      [K1]
 *   ilug_sweep_upper    richardson_upper_scaled (include/iluamg/trisolve.hpp:46,
 *                       src/trisolve.cpp:132-147) + the unscaled Jacobi form       [K2]
 *   ilug_sweep_lower    richardson_lower (trisolve.hpp:39, src/trisolve.cpp:94-104) [K3]
 *   ilug_smooth         smooth / ilu_smooth_sweep (include/iluamg/smoother.hpp:45-49,
 *                       src/smoother.cpp:143-187)                                  [K4]
 *   ilug_solve_lower/upper  solve_lower_direct / solve_upper_scaled_direct
 *                       (trisolve.hpp:25-52), level-scheduled                        [K5]
 *   ilug_spmv/residual  spmv_into / residual (include/iluamg/sparse.hpp:63-84)       [K6]
 *   ilug_vcycle         vcycle (include/iluamg/amg.hpp:105, src/amg.cpp:394-418)
 *                       incl. the coarse DenseLu::solve (src/dense.cpp:40-55)       [K6,K7]
 *   ilug_gmres          krylov_solve/gmres_impl (include/iluamg/krylov.hpp:64-80),
 *                       CGS2 orthogonalisation                                       [K8]
 */
#ifndef ILUG_H
#define ILUG_H

#include "iluamg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ilug_factors_s ilug_factors;
typedef struct ilug_dmatrix_s ilug_dmatrix;
typedef struct ilug_smoother_s ilug_smoother;
typedef struct ilug_hierarchy_s ilug_hierarchy;

ILUAMG_API const char* ilug_last_error(void);
ILUAMG_API int ilug_device_count(int* count);
ILUAMG_API int ilug_set_device(int device);
ILUAMG_API int ilug_synchronize(void* stream);

/* ---- host matrices (SparseMatrix::from_csr, src/sparse.cpp:88-118) ---- */
ILUAMG_API int ilug_matrix_from_csr(long long nrows, long long ncols, const long long* row_starts,
                                    const long long* col_indices, const double* values,
                                    iluamg_matrix** out);
/* Copies into caller arrays sized rows+1 / nnz / nnz. */
ILUAMG_API int ilug_matrix_copy_csr(const iluamg_matrix* A, long long* row_starts,
                                    long long* col_indices, double* values);

/* ---- host setup (no device needed; the north star keeps it on the host) ---- */
/* ILU(0)/ILUT per the config's ilu.* keys (src/ilu.cpp:56-265): L strict, U with diagonal. */
ILUAMG_API int ilug_ilu_factorize(const iluamg_matrix* A, const iluamg_config* cfg,
                                  iluamg_matrix** L, iluamg_matrix** U);
/* The factorisation the device objects use: ILU(0) (thread per row) and ILUT
 * (warp per row) on the device, level-free and dependency-flag scheduled;
 * bitwise equal to ilug_ilu_factorize. ILUG_ILU0_DEVICE=0 / ILUG_ILUT_DEVICE=0
 * force the host path. */
ILUAMG_API int ilug_ilu_factorize_device(const iluamg_matrix* A, const iluamg_config* cfg,
                                         iluamg_matrix** L, iluamg_matrix** U);
/* Device sparse products (kernels/spgemm.cu), bitwise equal to the host
 * SparseMatrix::multiply (src/sparse.cpp:176-231): C = A B, and the AMG
 * Galerkin operator C = R (A P) with A P kept on the device. */
ILUAMG_API int ilug_matmul_device(const iluamg_matrix* A, const iluamg_matrix* B, iluamg_matrix** C);
ILUAMG_API int ilug_galerkin_device(const iluamg_matrix* A, const iluamg_matrix* P, const iluamg_matrix* R,
                                    iluamg_matrix** C);

/* ---- K1-K5: factors ---- */
/* ILU(0)/ILUT per the config's ilu.* keys (on the device, bitwise the host and
 * reference factors), then K1 scaling per `scaling` (0 none, 1 row, 2 row_col).
 * upper_iteration: 0 scaled, 1 jacobi (unscaled). direct_plans != 0 also builds
 * the level schedules for ilug_solve_*. */
ILUAMG_API int ilug_factors_create(const iluamg_matrix* A, const iluamg_config* cfg, int scaling,
                                   int upper_iteration, int direct_plans, ilug_factors** out);
/* From explicit factors: L strictly lower (unit diagonal implicit), U upper with its diagonal. */
ILUAMG_API int ilug_factors_from_csr(long long n, const long long* L_rows, const long long* L_cols,
                                     const double* L_vals, const long long* U_rows,
                                     const long long* U_cols, const double* U_vals, int scaling,
                                     int upper_iteration, int direct_plans, ilug_factors** out);
/* Numeric refactorisation of ILU(0) factors (created by ilug_factors_create with
 * ilu.variant=ilu0) for a matrix with the same pattern (the time-stepping case,
 * P:636-648): the symbolic data stay on the device, only values are uploaded;
 * the result is bitwise the factors a fresh ilug_factors_create would build.
 * Status 2 if the pattern differs or the factors are not ILU(0). */
ILUAMG_API int ilug_factors_refactor(ilug_factors* f, const iluamg_matrix* A);
ILUAMG_API long long ilug_factors_rows(const ilug_factors* f);
/* nnz of L (strict) and of U (with diagonal). */
ILUAMG_API int ilug_factors_nnz(const ilug_factors* f, long long* nnz_L, long long* nnz_U);
/* Download U as scaled on the device (unit diagonal when scaled) and the scale
 * vectors (row_scale / col_scale may be NULL; flags bit0 = has row scale,
 * bit1 = has col scale). Synchronises. */
ILUAMG_API int ilug_factors_download_upper(const ilug_factors* f, long long* rows, long long* cols,
                                           double* vals, double* row_scale, double* col_scale,
                                           int* flags);
/* y = richardson_lower(L, b, m); x = richardson_upper_scaled(f, b, m) (or the Jacobi
 * form). Device pointers; b and the output must differ. */
ILUAMG_API int ilug_sweep_lower(const ilug_factors* f, const double* b, double* y, long long m,
                                void* stream);
ILUAMG_API int ilug_sweep_upper(const ilug_factors* f, const double* b, double* x, long long m,
                                void* stream);
/* Host-buffer variants (copy in, sweep, copy out; synchronous) for end-to-end timing. */
ILUAMG_API int ilug_sweep_upper_host(const ilug_factors* f, const double* b_host, double* x_host,
                                     long long m);
ILUAMG_API int ilug_solve_lower(const ilug_factors* f, const double* b, double* y, void* stream);
ILUAMG_API int ilug_solve_upper(const ilug_factors* f, const double* b, double* x, void* stream);
/* Sizes for the roofline: n, nnz of strict L, nnz of strict U, SELL padding. */
ILUAMG_API int ilug_factors_stats(const ilug_factors* f, long long* n, long long* nnz_Ls,
                                  long long* nnz_Us, long long* padded_Us, int* levels_L,
                                  int* levels_U);
/* Wavefront (temporally blocked) sweep plans: tile counts of L and U (0 = the
 * fused path is off for these factors, see ILUG_WAVEFRONT); whether a fused
 * launch hit its bounded-spin guard since the last query (*stalled = 1: a
 * scheduling bug, the affected results must be discarded); and how many work
 * items had to wait for their inputs (schedule diagnostic). Resets both. */
ILUAMG_API int ilug_factors_wave(const ilug_factors* f, long long* tiles_L, long long* tiles_U,
                                 int* stalled, long long* waits);
ILUAMG_API void ilug_factors_free(ilug_factors* f);

/* ---- K6: device operator ---- */
ILUAMG_API int ilug_dmatrix_create(const iluamg_matrix* A, ilug_dmatrix** out);
ILUAMG_API int ilug_spmv(const ilug_dmatrix* A, const double* x, double* y, void* stream);
ILUAMG_API int ilug_residual(const ilug_dmatrix* A, const double* x, const double* b, double* r,
                             void* stream);
ILUAMG_API void ilug_dmatrix_free(ilug_dmatrix* A);

/* ---- K4: smoother (which: 0 = finest-level config, 1 = fallback config) ---- */
ILUAMG_API int ilug_smoother_create(const iluamg_matrix* A, const iluamg_config* cfg, int which,
                                    ilug_smoother** out);
/* x <- smooth(A, b, x); resnorm (host, may be NULL) receives |b - A x|_2 like
 * the reference's return value (synchronises when requested). One in-flight
 * call per handle (the handle owns its workspace). */
ILUAMG_API int ilug_smooth(const ilug_smoother* s, const double* b, double* x, double* resnorm,
                           void* stream);
ILUAMG_API int ilug_ilu_smooth_sweep(const ilug_smoother* s, const double* b, double* x,
                                     void* stream);
/* Host-buffer smoother application (copy b, x in; smooth; copy x out; synchronous):
 * the end-to-end form of ilug_smooth used for e2e timing. */
ILUAMG_API int ilug_smooth_host(const ilug_smoother* s, const double* b_host, double* x_host);
/* count independent smoother applications x_i <- smooth(A, b_i, x_i) on host
 * buffers, pipelined: the copy-in of step i+1 and the copy-out of step i-1 run
 * on their own streams while step i smooths (two device slots). Pinned host
 * memory gives true overlap. Pairs may repeat only two or more positions
 * apart (slot reuse is ordered; adjacent steps are in flight together).
 * Returns after the last copy-out. */
ILUAMG_API int ilug_smooth_host_many(const ilug_smoother* s, long long count, const double* const* b_host,
                                     double* const* x_host);
/* Sizes for byte accounting: n, nnz(A), nnz(strict L), nnz(strict U) (ILU kinds; 0 otherwise),
 * SELL padded entries of strict U. */
ILUAMG_API int ilug_smoother_stats(const ilug_smoother* s, long long* n, long long* nnz_A,
                                   long long* nnz_Ls, long long* nnz_Us, long long* padded_Us);
/* Same as ilug_factors_wave for an ILU smoother's factors (zeros for other kinds). */
ILUAMG_API int ilug_smoother_wave(const ilug_smoother* s, long long* tiles_L, long long* tiles_U,
                                  int* stalled, long long* waits);
/* nsweeps (2..9) fused sweeps of one factor in one wavefront launch, for per-kernel
 * timing: x_{k+1} = rhs - T x_k from x_1 = x_in, T = strict L (which = 0) or strict
 * (scaled) U (which = 1); tmp: (nsweeps - 1) * n doubles; out = x_{nsweeps+1}.
 * ILUAMG_ERR_INVALID when the smoother has no wavefront plan. */
ILUAMG_API int ilug_smoother_sweeps_fused(const ilug_smoother* s, int which, int nsweeps,
                                          const double* x_in, const double* rhs, double* tmp,
                                          double* out, void* stream);
/* One bare sweep kernel of an ILU smoother's factor, for per-kernel timing:
 * out = rhs - T x_in with T = strict L (which = 0) or strict (scaled) U (which = 1). */
ILUAMG_API int ilug_smoother_sweep_once(const ilug_smoother* s, int which, const double* x_in,
                                        const double* rhs, double* out, void* stream);
ILUAMG_API void ilug_smoother_free(ilug_smoother* s);

/* ---- K6/K7: AMG hierarchy and V-cycle ---- */
ILUAMG_API int ilug_hierarchy_create(const iluamg_matrix* A, const iluamg_config* cfg,
                                     ilug_hierarchy** out);
/* Host-only setup (amg.* keys; src/amg.cpp:348-390): levels/matrices can be
 * inspected, ilug_vcycle/ilug_gmres refuse it. */
ILUAMG_API int ilug_hierarchy_create_host(const iluamg_matrix* A, const iluamg_config* cfg,
                                          ilug_hierarchy** out);
ILUAMG_API int ilug_hierarchy_levels(const ilug_hierarchy* h);
/* which: 0 A, 1 P, 2 R of `level` as a new host matrix (parity downloads). */
ILUAMG_API int ilug_hierarchy_level_matrix(const ilug_hierarchy* h, int level, int which,
                                           iluamg_matrix** out);
ILUAMG_API double ilug_hierarchy_operator_complexity(const ilug_hierarchy* h);
/* z = M(r): z zeroed, one cycle (the precond lambda of src/driver.cpp:182-185).
 * One in-flight call per handle. */
ILUAMG_API int ilug_vcycle(ilug_hierarchy* h, const double* r, double* z, void* stream);
/* Number of graph nodes (kernels + copies) one replayed V-cycle launches. */
ILUAMG_API long long ilug_vcycle_graph_nodes(const ilug_hierarchy* h);
ILUAMG_API void ilug_hierarchy_free(ilug_hierarchy* h);

/* ---- K8: preconditioned (F)GMRES, krylov.* keys of cfg; device b, x (x = x0 in,
 * solution out). iterations / final_relres may be NULL. Synchronises. Returns
 * ILUAMG_NOT_CONVERGED when the criterion was missed. ---- */
ILUAMG_API int ilug_gmres(ilug_hierarchy* h, const iluamg_config* cfg, const double* b, double* x,
                          long long* iterations, double* final_relres, void* stream);

/* ---- multi-GPU: row-block partition (src/schur.cpp:28-33 rule), halo plan,
 * NCCL communicator, block-Jacobi ILU smoother with a global residual.
 * One process per GPU; the caller moves the 128-byte NCCL id and the halo
 * request lists between ranks with its own plumbing (torch.distributed). ---- */
typedef struct ilug_dist_plan_s ilug_dist_plan;
typedef struct ilug_dist_comm_s ilug_dist_comm;
typedef struct ilug_dist_smoother_s ilug_dist_smoother;

/* starts[0..nranks] of the contiguous row blocks (last rank takes the remainder). */
ILUAMG_API int ilug_dist_partition(long long n, int nranks, long long* starts);
/* Rows [row0, row1) of a 3D generator spec, global column ids (ncols = n). */
ILUAMG_API int ilug_dist_generate_rows(const char* spec, long long row0, long long row1,
                                       iluamg_matrix** out);
/* This rank's rows (global columns) -> halo plan. */
ILUAMG_API int ilug_dist_plan_create(const iluamg_matrix* rows, long long n_global, int nranks, int rank,
                                     ilug_dist_plan** out);
ILUAMG_API int ilug_dist_plan_info(const ilug_dist_plan* p, long long* row0, long long* row1,
                                   long long* nhalo);
/* Global ids this rank needs from rank q; returns the count (ids may be NULL). */
ILUAMG_API long long ilug_dist_plan_requests(const ilug_dist_plan* p, int q, long long* ids);
/* Record what rank q requested from this rank (global ids). */
ILUAMG_API int ilug_dist_plan_set_sends(ilug_dist_plan* p, int q, const long long* ids, long long count);
/* Local row indices packed for rank q; returns the count (rows may be NULL). */
ILUAMG_API long long ilug_dist_plan_sends(const ilug_dist_plan* p, int q, long long* rows);
/* which: 0 extended local matrix (halo columns renumbered, global entry order), 1 diagonal block,
 * 2 off-block entries (halo columns, extended numbering). */
ILUAMG_API int ilug_dist_plan_matrix(const ilug_dist_plan* p, int which, iluamg_matrix** out);
ILUAMG_API void ilug_dist_plan_free(ilug_dist_plan* p);
ILUAMG_API int ilug_dist_unique_id(char* out128);
ILUAMG_API int ilug_dist_comm_create(int nranks, int rank, const char* id128, ilug_dist_comm** out);
/* In-process rank group: the ranks are host threads of one process (any
 * devices, several may share one GPU). Every collective synchronises the
 * caller's stream and meets the other ranks at a host barrier, so kernels
 * never wait on each other — the single-GPU stand-in for the NCCL path. */
typedef struct ilug_dist_group_s ilug_dist_group;
ILUAMG_API int ilug_dist_group_create(int nranks, ilug_dist_group** out);
ILUAMG_API void ilug_dist_group_free(ilug_dist_group* g);
/* A rank that failed releases the others: every pending and later collective of the group fails. */
ILUAMG_API void ilug_dist_group_abort(ilug_dist_group* g);
ILUAMG_API int ilug_dist_comm_create_local(ilug_dist_group* g, int rank, ilug_dist_comm** out);
/* Complete a plan's send lists over the communicator (collective; replaces
 * the caller-side request exchange). */
ILUAMG_API int ilug_dist_plan_exchange(ilug_dist_plan* p, const ilug_dist_comm* c);
ILUAMG_API int ilug_dist_allreduce_sum(const ilug_dist_comm* c, double* buf, long long count, void* stream);
ILUAMG_API void ilug_dist_comm_free(ilug_dist_comm* c);
/* Block-Jacobi ILU smoother of the plan's block (the config's ilu, scaling and trisolve keys). */
ILUAMG_API int ilug_dist_smoother_create(const ilug_dist_plan* p, const ilug_dist_comm* c,
                                         const iluamg_config* cfg, ilug_dist_smoother** out);
ILUAMG_API int ilug_dist_smooth(const ilug_dist_smoother* s, const double* b, double* x, void* stream);
ILUAMG_API int ilug_dist_residual(const ilug_dist_smoother* s, const double* x, const double* b, double* r,
                                  void* stream);
ILUAMG_API int ilug_dist_smoother_stats(const ilug_dist_smoother* s, long long* nloc, long long* nnz_A,
                                        long long* nnz_Ls, long long* nnz_Us);
/* Host-buffer application (copy this rank's b, x in; smooth; copy x out; synchronous). */
ILUAMG_API int ilug_dist_smooth_host(const ilug_dist_smoother* s, const double* b_host, double* x_host);
/* Pipelined multi-step form of ilug_dist_smooth_host (see ilug_smooth_host_many);
 * collective: every rank calls it with the same count. */
ILUAMG_API int ilug_dist_smooth_host_many(const ilug_dist_smoother* s, long long count,
                                          const double* const* b_host, double* const* x_host);
/* One bare L (which = 0) or U (which = 1) sweep kernel of the local factors, for kernel timing. */
ILUAMG_API int ilug_dist_smoother_sweep_once(const ilug_dist_smoother* s, int which, const double* x_in,
                                             const double* rhs, double* out, void* stream);
ILUAMG_API void ilug_dist_smoother_free(ilug_dist_smoother* s);

/* Distributed GMRES+AMG: the GLOBAL hierarchy `h` (a host
 * hierarchy handle, ilug_hierarchy_create_host; every rank passes the same
 * one) is row-block partitioned level by level: A_k / P_k rows by the level's
 * partition, R_k rows by the next level's, halo exchanges before every global
 * product, rank-local smoothers (block-Jacobi ILU / poly-GS, hybrid GS, global
 * Jacobi / l1), the coarsest rhs all-gathered and solved on every rank.
 * Global (F)GMRES over the ranks' rows with summed CGS2 reductions (replaces
 * gmres_impl + the V-cycle lambda, src/krylov.cpp:75-238, src/driver.cpp:182-185).
 * b, x, r, z: this rank's rows. All calls are collective. */
typedef struct ilug_dist_solver_s ilug_dist_solver;
ILUAMG_API int ilug_dist_solver_create(const ilug_hierarchy* h, const ilug_dist_comm* c, ilug_dist_solver** out);
ILUAMG_API int ilug_dist_gmres(ilug_dist_solver* s, const iluamg_config* cfg, const double* b, double* x,
                               long long* iterations, double* final_relres, void* stream);
ILUAMG_API int ilug_dist_vcycle(ilug_dist_solver* s, const double* r, double* z, void* stream);
ILUAMG_API int ilug_dist_solver_info(const ilug_dist_solver* s, long long* row0, long long* nloc, int* levels);
ILUAMG_API int ilug_dist_solver_levels(const ilug_dist_solver* s);
ILUAMG_API void ilug_dist_solver_free(ilug_dist_solver* s);

/* Host-only view of the per-level distribution (no device work): the halo
 * plans a rank's distributed V-cycle uses (tests, tooling). which: 0 A, 1 R,
 * 2 P (levels before the last smoothed one); ilug_dist_levels_last: the last
 * smoothed level's whole R (which 0) and its rows of P (which 1). */
typedef struct ilug_dist_levels_s ilug_dist_levels;
ILUAMG_API int ilug_dist_level_plans(const ilug_hierarchy* h, int nranks, int rank, ilug_dist_levels** out);
ILUAMG_API int ilug_dist_levels_count(const ilug_dist_levels* l);
ILUAMG_API int ilug_dist_levels_plan(const ilug_dist_levels* l, int k, int which, ilug_dist_plan** out);
ILUAMG_API int ilug_dist_levels_last(const ilug_dist_levels* l, int which, iluamg_matrix** out);
ILUAMG_API void ilug_dist_levels_free(ilug_dist_levels* l);

#ifdef __cplusplus
}
#endif

#endif /* ILUG_H */
