/*
 * bosp_b200.h -- C ABI of the B200-native BOSP core (libbosp_b200.so).
 *
 * Drop-in boundary for the reference's solver + matvec-callback plugin API
 * (/root/reference/proj, C++20).  Plain pointers and sizes only: every block is a host
 * column-major fp64 array (column j of an n x m block starts at j*n), every index is int64,
 * errors are status codes + a thread-local message (no C++ exception crosses this ABI).
 * Each entry point names the reference interface it replaces (file:line relative to
 * /root/reference/proj).  The C++ facade with the reference's own names (bosp::solve,
 * bosp::LinearOperator, ...) is paper_2506_08355_b200/csrc/api.hpp; this header is what an
 * FFI (ctypes / cgo / JNI / N-API) binds.
 */
#ifndef BOSP_B200_H
#define BOSP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: one per exception class of include/bosp/core/errors.hpp:9-69. */
typedef enum {
    BOSP_OK = 0,
    BOSP_CONTRACT_VIOLATION = 1,
    BOSP_INGESTION_ERROR = 2,
    BOSP_NULLSPACE_LEAK = 3,
    BOSP_DEGENERATE_SPECTRUM = 4,
    BOSP_RANK_MISMATCH = 5,
    BOSP_INVALID_NULLSPACE = 6,
    BOSP_INITIALIZATION_FAILURE = 7,
    BOSP_NOT_ENOUGH_SAMPLES = 8,
    BOSP_NUMERICAL_ABORT = 9,
    BOSP_CUDA_ERROR = 10,
    BOSP_ERROR = 11
} bosp_status;

/* Message of the last failing call on this thread. */
const char* bosp_last_error(void);
/* Library/device identification: writes the device name, returns the SM count (or <0). */
int bosp_device_info(char* name, int name_len);

/* ---------------------------------------------------------------------------------------
 * Operators -- replaces LinearOperator (include/bosp/core/linear_operator.hpp:15-48)
 * --------------------------------------------------------------------------------------- */
typedef struct bosp_op_s* bosp_op;

/* Host callback: y(:, j) = A x(:, j), x and y host n x ncols column-major (ld = n).
 * Replaces LinearOperator::ApplyFn / from_callback (linear_operator.hpp:19,25). */
typedef void (*bosp_host_apply_fn)(void* ctx, const double* x, double* y, int64_t n, int64_t ncols);
/* Device callback -- the device analog of ApplyFn / from_callback (linear_operator.hpp:19,25):
 * y(:, j) = A x(:, j) for j < ncols, x and y in HBM of `device` (column-major, leading dims
 * ldx, ldy, n rows each), work enqueued on `stream` (a cudaStream_t).  Same contract as ApplyFn:
 * overwrite all of y, accept any ncols >= 1.  Return 0 on success; any other value aborts the
 * solve with BOSP_ERROR ("device callback returned <status>"), the C analog of an exception
 * thrown from an ApplyFn. */
typedef int (*bosp_device_apply_fn)(void* ctx, int device, const double* x, int64_t ldx, double* y,
                                    int64_t ldy, int64_t n, int64_t ncols, void* stream);

/* from_dense (linear_operator.cpp:12-31): a is n x n column-major, copied to HBM. */
bosp_status bosp_op_dense(int64_t n, const double* a, bosp_op* out);
/* from_csr (linear_operator.cpp:33-43; SparseMatrixCSR sparse_csr.hpp:12-28). */
bosp_status bosp_op_csr(int64_t n, const int64_t* row_offsets, const int64_t* col_indices,
                        const double* values, bosp_op* out);
/* read_matrix_market (matrix_market.hpp:10-13, matrix_market.cpp:26-91): coordinate real
 * general|symmetric -> CSR (symmetric expanded, duplicates summed).  Call once with null
 * arrays for rows/cols/nnz, then with rowptr (rows+1), colidx and vals (nnz) to copy them out.
 * Malformed input -> BOSP_INGESTION_ERROR, message "<path>:<line>: <what>". */
bosp_status bosp_read_matrix_market(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz,
                                    int64_t* rowptr, int64_t* colidx, double* vals);
/* File -> device CSR operator (square matrices). */
bosp_status bosp_op_matrix_market(const char* path, bosp_op* out);
/* from_callback (linear_operator.cpp:45-47). */
bosp_status bosp_op_callback(int64_t n, bosp_host_apply_fn fn, void* ctx, bosp_op* out);
bosp_status bosp_op_device_callback(int64_t n, bosp_device_apply_fn fn, void* ctx, bosp_op* out);

/* Matrix-free structured-grid Laplacian family (new; the reference reaches such operators
 * only through from_callback):  y = scale * L_bc x + v .* x on nx*ny*nz nodes (nz=1: 5-point).
 * bc: 0 Neumann graph Laplacian, 1 Dirichlet.  potential: 0 none, 1 harmonic 0.5|x|^2 with
 * node coordinates origin + (i+1)*h, 2 explicit array v (n values). */
typedef struct {
    int64_t nx, ny, nz;
    int32_t bc;
    double scale;
    int32_t potential;
    double origin, h;
    const double* v;
    /* row partition along the slowest axis (z in 3-D, y in 2-D): local planes [s0, s0 + nz|ny)
     * of s_global, global z extent nz_global; s_global = 0 -> unpartitioned */
    int64_t s0, s_global, nz_global;
} bosp_stencil;
bosp_status bosp_op_stencil(const bosp_stencil* spec, bosp_op* out);

/* Row-partitioned operators: this rank's rows [row0, row0 + n_local) of an
 * n_global operator; requires a communicator on the calling thread (bosp_comm_init_nccl or
 * bosp_solve_multi).  CSR: rowptr has n_local + 1 entries (any base), colidx are global. */
bosp_status bosp_op_csr_rows(int64_t n_global, int64_t row0, int64_t n_local, const int64_t* rowptr,
                             const int64_t* colidx, const double* values, bosp_op* out);
/* a_rows: n_local x n_global column-major (ld n_local) */
bosp_status bosp_op_dense_rows(int64_t n_global, int64_t row0, int64_t n_local, const double* a_rows,
                               bosp_op* out);

/* identity / scaled_identity / diagonal / shifted (linear_operator.cpp:49-92). */
bosp_status bosp_op_identity(int64_t n, bosp_op* out);
bosp_status bosp_op_scaled_identity(int64_t n, double alpha, bosp_op* out);
bosp_status bosp_op_diagonal(int64_t n, const double* d, bosp_op* out);
bosp_status bosp_op_shifted(bosp_op base, double sigma, bosp_op* out);

/* LinearOperator::apply (linear_operator.cpp:94-106) on host blocks. */
bosp_status bosp_op_apply(bosp_op op, int64_t ncols, const double* x, double* y);
int64_t bosp_op_dim(bosp_op op);
/* 0 dense, 1 sparse_csr, 2 matrix_free_callback (LinearOperator::Kind). */
int bosp_op_kind(bosp_op op);
void bosp_op_free(bosp_op op);

/* ---------------------------------------------------------------------------------------
 * Solver -- replaces bosp::solve / BospConfig / SolverStats / EigenResult
 * (include/bosp/solver/bosp_solver.hpp:15-98)
 * --------------------------------------------------------------------------------------- */
typedef struct {
    int64_t nev, nb;
    double tol;
    int64_t ngs, s;
    int32_t moving;          /* -1 unset (default rule), 0 off, 1 on */
    int64_t max_outer_iter;
    uint64_t rng_seed;
    double inner_cg_tol;
    int64_t inner_cg_max_iter;
    double tol_null;
    int64_t rank_hint;       /* -1 unset */
} bosp_config;

/* BospConfig defaults (bosp_solver.hpp:15-34). */
void bosp_config_default(bosp_config* cfg);

typedef struct {
    int64_t iterations, matvec_count, step3_matvecs, step3_vecprods, max_width_u;
    double max_biorth_deviation, max_deflation_crossgram, final_biorth_deviation;
    int32_t nevconv_monotone;
    double wall_seconds;      /* host steady clock around the whole solve */
    int64_t nev_converged;
    int32_t converged;
    /* B200 additions */
    double device_seconds;    /* CUDA events on the solver stream around the whole solve */
    double host_small_seconds;
    int64_t repairs, cg_iterations, gpu_launches;
} bosp_stats;

/* bosp::solve (bosp_solver.cpp:513-536).  B may be NULL (Euclidean inner product).
 * Nullspace: r >= 0 with x0, y0 (n x r) supplies GeneralizedNullspace; r < 0 asks the solver
 * to compute it (compute_nullspace, nullspace.cpp:135).  Outputs have capacity `cap` pairs:
 * lambdas[cap], x and y (n x cap, may be NULL), residuals[cap]; *nout = pairs returned.
 * history (optional, history_cap x nev row-major) receives residual_history. */
bosp_status bosp_solve(bosp_op K, bosp_op M, bosp_op B, const bosp_config* cfg, int64_t r,
                       const double* x0, const double* y0, int64_t cap, double* lambdas,
                       double* x, double* y, double* residuals, int64_t* nout, bosp_stats* stats,
                       double* history, int64_t history_cap, int64_t* history_rows);

/* ---------------------------------------------------------------------------------------
 * Multi-GPU row partition (new; the reference is single address space).
 * --------------------------------------------------------------------------------------- */
/* One process per GPU: rank 0 creates an id (128 bytes), all ranks call init with it; the
 * communicator (NCCL) and this rank's row window attach to the calling thread.  After that,
 * bosp_solve on row-partitioned operators and local X0/Y0 rows returns local rows of x, y. */
bosp_status bosp_comm_nccl_unique_id(unsigned char* id128);
bosp_status bosp_comm_init_nccl(const unsigned char* id128, int32_t nranks, int32_t rank,
                                int64_t n_global, int64_t row0);
bosp_status bosp_comm_free(void);

/* A global operator for the in-process driver (each rank slices it). kind: 0 dense, 1 csr,
 * 2 stencil (the stencil's s0/s_global must be 0). */
typedef struct {
    int32_t kind;
    int64_t n;
    const double* dense;
    const int64_t* rowptr;
    const int64_t* colidx;
    const double* vals;
    bosp_stencil stencil;
} bosp_global_op;

/* nranks row-partitioned ranks as threads of this process over ngpus devices (round-robin;
 * <= 0: all visible).  Several ranks may share a GPU.  B (nullable): the inner-product weight,
 * partitioned like K and M.  Outputs as bosp_solve, eigenvectors in global row order; stats:
 * max wall/device time over ranks. */
bosp_status bosp_solve_multi(int32_t nranks, int32_t ngpus, const bosp_global_op* K,
                             const bosp_global_op* M, const bosp_global_op* B, const bosp_config* cfg, int64_t r,
                             const double* x0, const double* y0, int64_t cap, double* lambdas,
                             double* x, double* y, double* residuals, int64_t* nout,
                             bosp_stats* stats);

/* regression_coefficients (bosp_solver.cpp:538-580); history rows x cols row-major. */
bosp_status bosp_regression(const double* history, int64_t rows, int64_t cols, int64_t idx,
                            double tol, double* alpha, double* beta, int32_t* degenerate);

/* analytic_nullspace_T (nullspace.cpp:195-212): x0, y0 are n x 1. */
bosp_status bosp_analytic_nullspace_T(int64_t n, double* x0, double* y0);
/* compute_nullspace (nullspace.cpp:135-193): up to cap columns into x0/y0, rank in *r. */
bosp_status bosp_compute_nullspace(bosp_op K, bosp_op M, bosp_op B, int64_t rank_hint,
                                   double tol_null, uint64_t seed, int64_t cap, int64_t* r,
                                   double* x0, double* y0);

/* ---------------------------------------------------------------------------------------
 * Block kernels (device), host blocks in/out -- kernels.hpp:22-30, biorth.hpp:30-45, cg.hpp:17
 * --------------------------------------------------------------------------------------- */
/* G (a x b) = X^T B Y  (block_inner, kernels.cpp:47-68). */
bosp_status bosp_block_inner(bosp_op B, int64_t n, int64_t a, int64_t b, const double* x,
                             const double* y, double* g);
/* out (n x b) = X C  (block_product, kernels.cpp:70-87). */
/* Test hook (no reference counterpart): the solver's multi-job Gram launch, X split into nseg
 * column segments; out = [XᵀY | XᵀX | YᵀY] column-major. */
bosp_status bosp_test_gram_jobs(int64_t n, int64_t a, int64_t b, const double* x, const double* y, int32_t nseg,
                                int32_t njobs, double* out);
/* Test hook (no reference counterpart): the symmetric Gram.  same != 0: out (2a x 2a) = Z^T Z
 * for Z = [X | Y] (the MGS pair Gram); same == 0: out (a x a) = X^T Y computed as a symmetric
 * Gram (upper tiles mirrored -- the Ritz K^ = U^T (K U) path; X^T Y must be symmetric). */
bosp_status bosp_test_gram_sym(int64_t n, int64_t a, const double* x, const double* y, int32_t same, double* out);
/* Test hook (no reference counterpart): the solver's fused MGS-Biorth application -- P = X A,
 * Q = Y B (X, Y n x k; A, B k x kb; k, kb <= 32) and g = P^T Q (kb x kb) from the same kernel. */
bosp_status bosp_test_biorth_apply(int64_t n, int64_t k, int64_t kb, const double* x, const double* y,
                                   const double* a, const double* b, double* p, double* q, double* g);
/* Test hook (no reference counterpart): the solver's device MGS-Biorth (mgs_biorth,
 * biorth.cpp:102-109, as the outer iteration runs it: pair Gram, device or host coefficients,
 * fused application, second pass).  P, Q n x m get the kept columns; *nkept, *second_pass. */
bosp_status bosp_test_mgs_dev(int64_t n, int64_t m, const double* x, const double* y, double* p, double* q,
                              int64_t* nkept, int32_t* second_pass);
bosp_status bosp_block_product(int64_t n, int64_t a, int64_t b, const double* x, const double* c,
                               double* out);
/* Y (n x b) -= X C  (block_axpy, kernels.cpp:89-104). */
bosp_status bosp_block_axpy(int64_t n, int64_t a, int64_t b, const double* x, const double* c,
                            double* y);
/* mgs_biorth (classical=0) / cgs_biorth (classical=1) (biorth.cpp:102-114).  P, Q n x m
 * receive the kept columns; kept/dropped index lists (capacity m). */
bosp_status bosp_biorth(int32_t classical, bosp_op B, int64_t n, int64_t m, const double* x,
                        const double* y, double drop_tol, double* p, double* q, int64_t* kept,
                        int64_t* nkept, int64_t* dropped, int64_t* ndropped);
/* biorth_against (biorth.cpp:116-133): nbases pairs (ps[i], qs[i]) of widths[i] columns. */
bosp_status bosp_biorth_against(bosp_op B, int64_t n, int64_t nbases, const int64_t* widths,
                                const double* const* ps, const double* const* qs, int64_t m,
                                const double* x, const double* y, double* xo, double* yo);
/* biorth_residual (biorth.cpp:135-143). */
bosp_status bosp_biorth_residual(bosp_op B, int64_t n, int64_t m, const double* p,
                                 const double* q, double* out);
/* cg_solve (cg.cpp:11-58), batched over columns with per-column masks. */
bosp_status bosp_cg_solve(bosp_op A, int64_t m, const double* rhs, const double* x0, double tol,
                          int64_t max_iter, double* x, int32_t* breakdown, int64_t* max_it_used);

/* The initial random blocks exactly as initialize() draws them (bosp_solver.cpp:144-150):
 * U = [X|P|W] (n x d) then V = [Y|Q|Z] (n x d) from mt19937_64(seed), uniform [-1, 1),
 * generated on the device. */
bosp_status bosp_seed_blocks(uint64_t seed, int64_t n, int64_t d, double* u, double* v);

/* Host small dense (projected_lrep.cpp:48-80, dense_kernels.cpp:11-123). */
bosp_status bosp_solve_small_lrep(int64_t d, const double* khat, const double* mhat, int64_t k,
                                  double* lambdas, double* xhat, double* yhat);
bosp_status bosp_jacobi_svd(int64_t m, int64_t k, const double* a, double* u, double* sigma,
                            double* v, int64_t* sweeps, int32_t* converged);
bosp_status bosp_cholesky(int64_t n, const double* a, double* l, int32_t* ok);

/* ---------------------------------------------------------------------------------------
 * Measurement hooks (bench.py): kernel-family CUDA-event timing and launch counting.
 * --------------------------------------------------------------------------------------- */
/* Time every launch of one kernel family ("spmm", "gram", "product", "cg_vec", ...); NULL or
 * "" disables.  A composite-operation name ("mgs" = one MGS-Biorth call, biorth.cpp:102-109)
 * times every launch issued inside that operation. */
void bosp_profile_enable(const char* family);
/* Synchronises; returns launches, summed device ms, algorithmic bytes and flops since enable. */
void bosp_profile_collect(int64_t* launches, double* ms, double* bytes, double* flops);
/* As bosp_profile_collect, plus the number of composite operations profiled and their summed
 * algorithmic bytes (MGS-Biorth of n x m: 32 n m for X, Y in and P, Q out, + 16 n m for the
 * P^T Q check of the second-pass test).  Either extra pointer may be NULL. */
void bosp_profile_collect_regions(int64_t* launches, double* ms, double* bytes, double* flops,
                                  int64_t* region_calls, double* region_bytes);
/* After bosp_profile_enable("*") (every launch timed) and a collect: the collected totals split
 * by kernel family, one text line per family "<family> <launches> <ms> <bytes> <flops>\n"
 * into buf (NUL-terminated, truncated to len); returns the length the full report needs.  A
 * composite-operation profile ("mgs") adds "@region <calls> 0 <bytes> <flops>". */
int64_t bosp_profile_family_report(char* buf, int64_t len);
/* Microbenchmark: apply `op` to a device-resident random n x ncols block `reps` times (after
 * one warm-up); returns the mean device time per apply in *ms (CUDA events). */
bosp_status bosp_bench_apply(bosp_op op, int64_t ncols, int64_t reps, double* ms);
/* Microbenchmark of the tall-skinny kernels on device-resident random data: kind 0 = Gram
 * (n x a)^T (n x b), 1 = product (n x a)(a x b), 2 = axpy, 3 = the three Grams X^T X, X^T Y,
 * Y^T Y as three jobs, 4 = the same as one symmetric Gram of [X | Y], 5 = the fused MGS-Biorth
 * apply (P = X A, Q = Y B, P^T Q; a = b <= 32); mean ms per call. */
bosp_status bosp_bench_blas(int32_t kind, int64_t n, int64_t a, int64_t b, int64_t reps, double* ms);
/* Microbenchmark of the batched CG: `iters` iterations (tol 0, so every column runs all of
 * them) on a random n x ncols right-hand side; mean ms per CG iteration over `reps` solves. */
bosp_status bosp_bench_cg(bosp_op op, int64_t ncols, int64_t iters, int64_t reps, double* ms);
/* Kernel launches issued by this library since the last reset. */
int64_t bosp_launch_count(void);
void bosp_launch_reset(void);
/* Per-family launch counts as "family=count;..." into buf. */
int bosp_launch_families(char* buf, int len);
void bosp_device_sync(void);
/* cudaProfilerStart (on != 0) / cudaProfilerStop: brackets the launches an
 * `ncu --profile-from-start off` capture sees (tools/run_config.py --profile-range). */
void bosp_profiler_range(int on);
/* Select the CUDA device for this process (call before any other entry point; one process
 * per GPU).  Returns 0 on success. */
int bosp_set_device(int device);
/* Evict L2 by writing `bytes` (>= 2x the 126 MB L2) on the solver stream; synchronises. */
void bosp_flush_l2(int64_t bytes);
/* Pinned host memory for e2e measurements. */
void* bosp_host_alloc(int64_t bytes);
void bosp_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* BOSP_B200_H */
