// extern "C" boundary (include/bosp_b200.h): maps the C++ facade onto plain pointers and status
// codes.  No exception crosses this boundary.
#include "../../include/bosp_b200.h"

#include <cuda_profiler_api.h>

#include <cstdio>
#include <algorithm>
#include <cstring>
#include <string>

#include "api.hpp"
#include "comm.hpp"
#include "dense_ops.hpp"
#include "dev_algos.hpp"
#include "multi.hpp"
#include "operators.hpp"
#include "rng.hpp"
#include "runtime.hpp"

struct bosp_op_s {
    bosp::LinearOperator op;
};

namespace {

thread_local std::string g_err;

bosp_status status_of(const std::exception& e) {
    using namespace bosp;
    if (dynamic_cast<const ContractViolation*>(&e)) return BOSP_CONTRACT_VIOLATION;
    if (dynamic_cast<const IngestionError*>(&e)) return BOSP_INGESTION_ERROR;
    if (dynamic_cast<const NullspaceLeak*>(&e)) return BOSP_NULLSPACE_LEAK;
    if (dynamic_cast<const DegenerateSpectrum*>(&e)) return BOSP_DEGENERATE_SPECTRUM;
    if (dynamic_cast<const RankMismatch*>(&e)) return BOSP_RANK_MISMATCH;
    if (dynamic_cast<const InvalidNullspace*>(&e)) return BOSP_INVALID_NULLSPACE;
    if (dynamic_cast<const InitializationFailure*>(&e)) return BOSP_INITIALIZATION_FAILURE;
    if (dynamic_cast<const NotEnoughSamples*>(&e)) return BOSP_NOT_ENOUGH_SAMPLES;
    if (dynamic_cast<const NumericalAbort*>(&e)) return BOSP_NUMERICAL_ABORT;
    if (dynamic_cast<const CudaError*>(&e)) return BOSP_CUDA_ERROR;
    return BOSP_ERROR;
}

template <class F>
bosp_status guarded(F&& f) {
    try {
        f();
        return BOSP_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return status_of(e);
    } catch (...) {
        g_err = "unknown exception";
        return BOSP_ERROR;
    }
}

bosp::BlockVectors host_block(const double* p, int64_t n, int64_t m) {
    bosp::BlockVectors b(n, m);
    if (n * m > 0) std::memcpy(b.data(), p, sizeof(double) * n * m);
    return b;
}

void copy_out(const bosp::BlockVectors& b, double* out) {
    if (out && b.dim() * b.cols() > 0) std::memcpy(out, b.data(), sizeof(double) * b.dim() * b.cols());
}

bosp::DenseMatrix host_dense(const double* p, int64_t r, int64_t c) {
    bosp::DenseMatrix d(r, c);
    if (r * c > 0) std::memcpy(d.data(), p, sizeof(double) * r * c);
    return d;
}

bosp::InnerProduct ip_of(bosp_op b) {
    return b ? bosp::InnerProduct(b->op) : bosp::InnerProduct{};
}

bosp_op wrap(bosp::LinearOperator op) { return new bosp_op_s{std::move(op)}; }

void write_result(const bosp::EigenResult& res, const bosp::BospConfig& cfg, int64_t cap, double* lambdas,
                  double* x, double* y, double* residuals, int64_t* nout, bosp_stats* stats, double* history,
                  int64_t history_cap, int64_t* history_rows) {
    const int64_t h = static_cast<int64_t>(res.lambdas.size());
    bosp::require(h <= cap, "bosp_solve: output capacity too small");
    *nout = h;
    for (int64_t j = 0; j < h; ++j) {
        lambdas[j] = res.lambdas[j];
        residuals[j] = res.residuals[j];
    }
    copy_out(res.x, x);
    copy_out(res.y, y);
    if (stats) {
        const bosp::SolverStats& s = res.stats;
        stats->iterations = s.iterations;
        stats->matvec_count = s.matvec_count;
        stats->step3_matvecs = s.step3_matvecs;
        stats->step3_vecprods = s.step3_vecprods;
        stats->max_width_u = s.max_width_u;
        stats->max_biorth_deviation = s.max_biorth_deviation;
        stats->max_deflation_crossgram = s.max_deflation_crossgram;
        stats->final_biorth_deviation = s.final_biorth_deviation;
        stats->nevconv_monotone = s.nevconv_monotone ? 1 : 0;
        stats->wall_seconds = s.wall_seconds;
        stats->nev_converged = res.nev_converged;
        stats->converged = res.converged ? 1 : 0;
        stats->device_seconds = s.device_seconds;
        stats->host_small_seconds = s.host_small_seconds;
        stats->repairs = s.repairs;
        stats->cg_iterations = s.cg_iterations;
        stats->gpu_launches = s.gpu_launches;
    }
    if (history_rows) *history_rows = static_cast<int64_t>(res.history.size());
    if (history) {
        const int64_t rows = std::min<int64_t>(static_cast<int64_t>(res.history.size()), history_cap);
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t j = 0; j < cfg.nev; ++j)
                history[i * cfg.nev + j] = j < static_cast<int64_t>(res.history[i].size()) ? res.history[i][j] : 0.0;
    }
}

bosp::GlobalOp global_of(const bosp_global_op* g) {
    bosp::GlobalOp o;
    o.kind = static_cast<bosp::GlobalOp::Kind>(g->kind);
    o.n = g->n;
    o.dense = g->dense;
    o.rowptr = g->rowptr;
    o.colidx = g->colidx;
    o.vals = g->vals;
    if (g->kind == 2) {
        const bosp_stencil* s = &g->stencil;
        o.stencil.nx = s->nx;
        o.stencil.ny = s->ny;
        o.stencil.nz = s->nz;
        o.stencil.bc = static_cast<bosp::StencilSpec::Boundary>(s->bc);
        o.stencil.scale = s->scale;
        o.stencil.potential = static_cast<bosp::StencilSpec::Potential>(s->potential);
        o.stencil.origin = s->origin;
        o.stencil.h = s->h;
        if (s->potential == 2) o.stencil.v.assign(s->v, s->v + s->nx * s->ny * s->nz);
        o.n = s->nx * s->ny * s->nz;
    }
    return o;
}

void fill_random(const bosp::DMat& m, uint64_t seed) {
    bosp::DBlock tmp(m.rows, m.cols);
    bosp::mt_fill_uv(seed, m, tmp.view());
}

template <class F>
double time_reps(int64_t reps, F&& f) {
    bosp::Runtime& rt = bosp::Runtime::get();
    f();
    cudaEvent_t a, b;
    BOSP_CUDA(cudaEventCreate(&a));
    BOSP_CUDA(cudaEventCreate(&b));
    BOSP_CUDA(cudaEventRecord(a, rt.stream()));
    for (int64_t i = 0; i < reps; ++i) f();
    BOSP_CUDA(cudaEventRecord(b, rt.stream()));
    rt.sync();
    float ms = 0.f;
    BOSP_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / static_cast<double>(std::max<int64_t>(reps, 1));
}

// Mean device time of f() with the L2 flushed (a 512 MB memset) before every call; only the
// calls are timed (events per call).
template <class F>
double time_reps_cold(int64_t reps, F&& f) {
    bosp::Runtime& rt = bosp::Runtime::get();
    f();
    const size_t fl = size_t(512) << 20;
    void* buf = nullptr;
    BOSP_CUDA(cudaMalloc(&buf, fl));
    cudaEvent_t a, b;
    BOSP_CUDA(cudaEventCreate(&a));
    BOSP_CUDA(cudaEventCreate(&b));
    double total = 0.0;
    for (int64_t i = 0; i < reps; ++i) {
        BOSP_CUDA(cudaMemsetAsync(buf, static_cast<int>(i & 1), fl, rt.stream()));
        BOSP_CUDA(cudaEventRecord(a, rt.stream()));
        f();
        BOSP_CUDA(cudaEventRecord(b, rt.stream()));
        rt.sync();
        float ms = 0.f;
        BOSP_CUDA(cudaEventElapsedTime(&ms, a, b));
        total += ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    return total / static_cast<double>(std::max<int64_t>(reps, 1));
}

bosp::BospConfig cfg_of(const bosp_config* c) {
    bosp::BospConfig cfg;
    cfg.nev = c->nev;
    cfg.nb = c->nb;
    cfg.tol = c->tol;
    cfg.ngs = c->ngs;
    cfg.s = c->s;
    if (c->moving >= 0) cfg.moving = c->moving != 0;
    cfg.max_outer_iter = c->max_outer_iter;
    cfg.rng_seed = c->rng_seed;
    cfg.inner_cg_tol = c->inner_cg_tol;
    cfg.inner_cg_max_iter = c->inner_cg_max_iter;
    cfg.tol_null = c->tol_null;
    if (c->rank_hint >= 0) cfg.rank_hint = c->rank_hint;
    return cfg;
}

}  // namespace

extern "C" {

const char* bosp_last_error(void) { return g_err.c_str(); }

int bosp_device_info(char* name, int name_len) {
    int sms = -1;
    bosp_status st = guarded([&] {
        bosp::Runtime& rt = bosp::Runtime::get();
        cudaDeviceProp prop{};
        BOSP_CUDA(cudaGetDeviceProperties(&prop, rt.device()));
        if (name && name_len > 0) {
            std::strncpy(name, prop.name, static_cast<size_t>(name_len - 1));
            name[name_len - 1] = 0;
        }
        sms = rt.sm_count();
    });
    return st == BOSP_OK ? sms : -static_cast<int>(st);
}

bosp_status bosp_op_dense(int64_t n, const double* a, bosp_op* out) {
    return guarded([&] { *out = wrap(bosp::LinearOperator::from_dense(a, n)); });
}

bosp_status bosp_op_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv, bosp_op* out) {
    return guarded([&] {
        bosp::SparseMatrixCSR a;
        a.rows = a.cols = static_cast<size_t>(n);
        a.row_offsets.assign(rp, rp + n + 1);
        a.col_indices.assign(ci, ci + rp[n]);
        a.values.assign(vv, vv + rp[n]);
        *out = wrap(bosp::LinearOperator::from_csr(a));
    });
}

bosp_status bosp_op_callback(int64_t n, bosp_host_apply_fn fn, void* ctx, bosp_op* out) {
    return guarded([&] {
        *out = wrap(bosp::LinearOperator::from_callback(
            n, [fn, ctx](const bosp::BlockVectors& x, bosp::BlockVectors& y) {
                fn(ctx, x.data(), y.data(), x.dim(), x.cols());
            }));
    });
}

bosp_status bosp_op_device_callback(int64_t n, bosp_device_apply_fn fn, void* ctx, bosp_op* out) {
    return guarded([&] {
        *out = wrap(bosp::LinearOperator::from_device_callback(
            n, [fn, ctx, n](int dev, const double* x, int64_t ldx, double* y, int64_t ldy, int64_t m, cudaStream_t s) {
                return fn(ctx, dev, x, ldx, y, ldy, n, m, static_cast<void*>(s));
            }));
    });
}

bosp_status bosp_op_stencil(const bosp_stencil* s, bosp_op* out) {
    return guarded([&] {
        bosp::StencilSpec sp;
        sp.nx = s->nx;
        sp.ny = s->ny;
        sp.nz = s->nz;
        sp.bc = static_cast<bosp::StencilSpec::Boundary>(s->bc);
        sp.scale = s->scale;
        sp.potential = static_cast<bosp::StencilSpec::Potential>(s->potential);
        sp.origin = s->origin;
        sp.h = s->h;
        if (s->potential == 2) sp.v.assign(s->v, s->v + s->nx * s->ny * s->nz);
        sp.s0 = s->s0;
        sp.s_global = s->s_global;
        sp.nz_global = s->nz_global;
        *out = wrap(bosp::LinearOperator::stencil(sp));
    });
}

bosp_status bosp_op_identity(int64_t n, bosp_op* out) {
    return guarded([&] { *out = wrap(bosp::LinearOperator::identity(n)); });
}

bosp_status bosp_op_scaled_identity(int64_t n, double alpha, bosp_op* out) {
    return guarded([&] { *out = wrap(bosp::LinearOperator::scaled_identity(n, alpha)); });
}

bosp_status bosp_op_diagonal(int64_t n, const double* d, bosp_op* out) {
    return guarded([&] { *out = wrap(bosp::LinearOperator::diagonal(std::vector<double>(d, d + n))); });
}

bosp_status bosp_op_shifted(bosp_op base, double sigma, bosp_op* out) {
    return guarded([&] { *out = wrap(bosp::LinearOperator::shifted(base->op, sigma)); });
}

bosp_status bosp_op_apply(bosp_op op, int64_t ncols, const double* x, double* y) {
    return guarded([&] {
        const int64_t n = op->op.dim();
        bosp::BlockVectors out(n, ncols);
        op->op.apply(host_block(x, n, ncols), out);
        copy_out(out, y);
    });
}

int64_t bosp_op_dim(bosp_op op) { return op ? op->op.dim() : 0; }
int bosp_op_kind(bosp_op op) { return op ? static_cast<int>(op->op.kind()) : -1; }
void bosp_op_free(bosp_op op) { delete op; }

void bosp_config_default(bosp_config* c) {
    const bosp::BospConfig d;
    c->nev = d.nev;
    c->nb = d.nb;
    c->tol = d.tol;
    c->ngs = d.ngs;
    c->s = d.s;
    c->moving = -1;
    c->max_outer_iter = d.max_outer_iter;
    c->rng_seed = d.rng_seed;
    c->inner_cg_tol = d.inner_cg_tol;
    c->inner_cg_max_iter = d.inner_cg_max_iter;
    c->tol_null = d.tol_null;
    c->rank_hint = -1;
}

bosp_status bosp_solve(bosp_op K, bosp_op M, bosp_op B, const bosp_config* c, int64_t r,
                       const double* x0, const double* y0, int64_t cap, double* lambdas,
                       double* x, double* y, double* residuals, int64_t* nout, bosp_stats* stats,
                       double* history, int64_t history_cap, int64_t* history_rows) {
    return guarded([&] {
        bosp::require(K && M, "bosp_solve: K and M are required");
        const bosp::BospConfig cfg = cfg_of(c);
        const int64_t n = K->op.dim();
        std::optional<bosp::GeneralizedNullspace> ns;
        if (r >= 0) {
            bosp::GeneralizedNullspace g;
            g.r = r;
            g.x0 = host_block(x0, n, r);
            g.y0 = host_block(y0, n, r);
            ns = std::move(g);
        }
        // null x / y: eigenvectors stay in HBM (no host copy); otherwise straight into x, y
        const bosp::HostVectorsOut hv{x, y, cap, !(x && y)};
        bosp::EigenResult res = bosp::solve(K->op, M->op, ip_of(B), cfg, std::move(ns), &hv);
        write_result(res, cfg, cap, lambdas, x, y, residuals, nout, stats, history, history_cap, history_rows);
    });
}

bosp_status bosp_read_matrix_market(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz, int64_t* rowptr,
                                    int64_t* colidx, double* vals) {
    thread_local std::string last_path;
    thread_local bosp::SparseMatrixCSR last;
    return guarded([&] {
        bosp::require(path != nullptr, "read_matrix_market: null path");
        if (last_path != path || !rowptr) {  // the size call parses; the copy call reuses it
            last = bosp::read_matrix_market(path);
            last_path = path;
        }
        *rows = static_cast<int64_t>(last.rows);
        *cols = static_cast<int64_t>(last.cols);
        *nnz = static_cast<int64_t>(last.nnz());
        if (rowptr) std::memcpy(rowptr, last.row_offsets.data(), sizeof(int64_t) * last.row_offsets.size());
        if (colidx) std::memcpy(colidx, last.col_indices.data(), sizeof(int64_t) * last.col_indices.size());
        if (vals) std::memcpy(vals, last.values.data(), sizeof(double) * last.values.size());
        if (rowptr) last_path.clear();
    });
}

bosp_status bosp_op_matrix_market(const char* path, bosp_op* out) {
    return guarded([&] {
        bosp::require(path != nullptr, "op_matrix_market: null path");
        const bosp::SparseMatrixCSR a = bosp::read_matrix_market(path);
        *out = wrap(bosp::LinearOperator::from_csr(a));
    });
}

bosp_status bosp_op_csr_rows(int64_t n_global, int64_t row0, int64_t n_local, const int64_t* rp, const int64_t* ci,
                             const double* vv, bosp_op* out) {
    return guarded([&] { *out = wrap(bosp::LinearOperator::from_csr_rows(n_global, row0, n_local, rp, ci, vv)); });
}

bosp_status bosp_op_dense_rows(int64_t n_global, int64_t row0, int64_t n_local, const double* a, bosp_op* out) {
    return guarded([&] { *out = wrap(bosp::LinearOperator::from_dense_rows(n_global, row0, n_local, a)); });
}

bosp_status bosp_comm_nccl_unique_id(unsigned char* id128) {
    return guarded([&] { bosp::NcclComm::unique_id(id128); });
}

bosp_status bosp_comm_init_nccl(const unsigned char* id128, int32_t nranks, int32_t rank, int64_t n_global,
                                int64_t row0) {
    return guarded([&] {
        bosp::Runtime& rt = bosp::Runtime::get();
        rt.set_comm(std::make_shared<bosp::NcclComm>(id128, nranks, rank));
        rt.set_rows(n_global, row0);
    });
}

bosp_status bosp_comm_free(void) {
    return guarded([&] {
        bosp::Runtime& rt = bosp::Runtime::get();
        rt.sync();
        rt.set_comm(nullptr);
        rt.set_rows(0, 0);
    });
}

bosp_status bosp_solve_multi(int32_t nranks, int32_t ngpus, const bosp_global_op* K, const bosp_global_op* M,
                             const bosp_global_op* B,
                             const bosp_config* c, int64_t r, const double* x0, const double* y0, int64_t cap,
                             double* lambdas, double* x, double* y, double* residuals, int64_t* nout,
                             bosp_stats* stats) {
    return guarded([&] {
        const bosp::BospConfig cfg = cfg_of(c);
        bosp::GlobalOp k = global_of(K), m = global_of(M);
        std::optional<bosp::GeneralizedNullspace> ns;
        if (r >= 0) {
            ns.emplace();
            ns->r = r;
            ns->x0 = host_block(x0, k.n, r);
            ns->y0 = host_block(y0, k.n, r);
        }
        bosp::GlobalOp bg;
        if (B) bg = global_of(B);
        bosp::EigenResult res = bosp::solve_multi(nranks, ngpus, k, m, B ? &bg : nullptr, cfg, ns);
        write_result(res, cfg, cap, lambdas, x, y, residuals, nout, stats, nullptr, 0, nullptr);
    });
}

bosp_status bosp_regression(const double* history, int64_t rows, int64_t cols, int64_t idx, double tol,
                            double* alpha, double* beta, int32_t* degenerate) {
    return guarded([&] {
        std::vector<std::vector<double>> h(static_cast<size_t>(rows));
        for (int64_t i = 0; i < rows; ++i) h[i].assign(history + i * cols, history + (i + 1) * cols);
        bosp::RegressionFit f = bosp::regression_coefficients(h, idx, tol);
        *alpha = f.alpha;
        *beta = f.beta;
        *degenerate = f.degenerate ? 1 : 0;
    });
}

bosp_status bosp_analytic_nullspace_T(int64_t n, double* x0, double* y0) {
    return guarded([&] {
        bosp::GeneralizedNullspace ns = bosp::analytic_nullspace_T(n);
        copy_out(ns.x0, x0);
        copy_out(ns.y0, y0);
    });
}

bosp_status bosp_compute_nullspace(bosp_op K, bosp_op M, bosp_op B, int64_t rank_hint, double tol_null,
                                   uint64_t seed, int64_t cap, int64_t* r, double* x0, double* y0) {
    return guarded([&] {
        std::optional<int64_t> hint;
        if (rank_hint >= 0) hint = rank_hint;
        bosp::GeneralizedNullspace ns = bosp::compute_nullspace(K->op, M->op, hint, tol_null, ip_of(B), seed);
        *r = ns.r;
        if (ns.r <= cap) {
            copy_out(ns.x0, x0);
            copy_out(ns.y0, y0);
        }
    });
}

bosp_status bosp_block_inner(bosp_op B, int64_t n, int64_t a, int64_t b, const double* x, const double* y, double* g) {
    return guarded([&] {
        bosp::DenseMatrix r = bosp::block_inner(ip_of(B), host_block(x, n, a), host_block(y, n, b));
        if (a * b > 0) std::memcpy(g, r.data(), sizeof(double) * a * b);
    });
}

// Test hook: the multi-job Gram launch the solver uses (XᵀY, XᵀX, YᵀY in one launch) with X
// split into nseg separately allocated column segments.  out = [XᵀY (a x b) | XᵀX (a x a) | YᵀY (b x b)].
bosp_status bosp_test_gram_jobs(int64_t n, int64_t a, int64_t b, const double* x, const double* y, int32_t nseg,
                                int32_t njobs, double* out) {
    return guarded([&] {
        bosp::require(nseg >= 1 && nseg <= 4 && njobs >= 1 && njobs <= 3 && a >= nseg, "test_gram_jobs: bad arguments");
        std::vector<bosp::DBlock> xs;
        bosp::ColList xl;
        int64_t c0 = 0;
        for (int s = 0; s < nseg; ++s) {
            const int64_t w = (a - c0) / (nseg - s);
            xs.emplace_back(n, w);
            bosp::to_device(x + c0 * n, n, w, n, xs.back().view());
            c0 += w;
        }
        for (auto& blk : xs) xl.add(blk.view());
        bosp::DBlock yd(n, b);
        bosp::to_device(y, n, b, n, yd.view());
        bosp::DBlock g1(a, b), g2(a, a), g3(b, b);
        const bosp::ColList yl(yd.view());
        const bosp::GramJob jobs[3] = {{xl, yl, g1.data(), g1.ld()}, {xl, xl, g2.data(), g2.ld()}, {yl, yl, g3.data(), g3.ld()}};
        bosp::gram(jobs, njobs, n);
        bosp::to_host(g1.view(), out, a);
        if (njobs > 1) bosp::to_host(g2.view(), out + a * b, a);
        if (njobs > 2) bosp::to_host(g3.view(), out + a * b + a * a, b);
    });
}

bosp_status bosp_test_gram_sym(int64_t n, int64_t a, const double* x, const double* y, int32_t same, double* out) {
    return guarded([&] {
        bosp::DBlock xd(n, a), yd(n, a), gd(same ? 2 * a : a, same ? 2 * a : a);
        bosp::to_device(x, n, a, n, xd.view());
        bosp::to_device(y, n, a, n, yd.view());
        bosp::GramJob job = same ? bosp::GramJob{bosp::ColList(xd.view()).add(yd.view()),
                                                 bosp::ColList(xd.view()).add(yd.view()), gd.data(), gd.ld()}
                                 : bosp::GramJob{bosp::ColList(xd.view()), bosp::ColList(yd.view()), gd.data(), gd.ld()};
        job.sym = true;
        bosp::gram(&job, 1, n);
        bosp::to_host(gd.view(), out, gd.rows());
    });
}

bosp_status bosp_test_biorth_apply(int64_t n, int64_t k, int64_t kb, const double* x, const double* y,
                                   const double* a, const double* b, double* p, double* q, double* g) {
    return guarded([&] {
        bosp::DBlock xd(n, k), yd(n, k), pd(n, kb), qd(n, kb), cd(k, 2 * kb), gd(kb, kb);
        bosp::to_device(x, n, k, n, xd.view());
        bosp::to_device(y, n, k, n, yd.view());
        bosp::to_device(a, k, kb, k, cd.cols(0, kb));
        bosp::to_device(b, k, kb, k, cd.cols(kb, kb));
        // K bound of every coefficient column (its last nonzero row in A or B): upper-triangular
        // inputs take the kernels' triangular K loops, as the solver's calls do
        std::vector<int32_t> ke(static_cast<size_t>(kb), 0);
        for (int64_t c = 0; c < kb; ++c)
            for (int64_t r = 0; r < k; ++r)
                if (a[r + c * k] != 0.0 || b[r + c * k] != 0.0) ke[c] = static_cast<int32_t>(r + 1);
        bosp::biorth_apply(xd.view(), yd.view(), cd.data(), cd.data() + kb * cd.ld(), cd.ld(), static_cast<int>(kb),
                           pd.view(), qd.view(), gd.data(), gd.ld(), ke.data());
        bosp::to_host(pd.view(), p, n);
        bosp::to_host(qd.view(), q, n);
        bosp::to_host(gd.view(), g, kb);
    });
}

bosp_status bosp_test_mgs_dev(int64_t n, int64_t m, const double* x, const double* y, double* p, double* q,
                              int64_t* nkept, int32_t* second_pass) {
    return guarded([&] {
        bosp::DBlock xd(n, m), yd(n, m), pd(n, m), qd(n, m);
        bosp::to_device(x, n, m, n, xd.view());
        bosp::to_device(y, n, m, n, yd.view());
        const bosp::DevBiorthOutcome o = bosp::dev_mgs_biorth(xd.view(), yd.view(), pd.view(), qd.view(),
                                                              bosp::InnerProduct(), 1e-12);
        *nkept = o.kept;
        *second_pass = o.second_pass ? 1 : 0;
        if (o.kept > 0) {
            bosp::to_host(pd.view().cols_range(0, o.kept), p, n);
            bosp::to_host(qd.view().cols_range(0, o.kept), q, n);
        }
    });
}

bosp_status bosp_block_product(int64_t n, int64_t a, int64_t b, const double* x, const double* c, double* out) {
    return guarded([&] { copy_out(bosp::block_product(host_block(x, n, a), host_dense(c, a, b)), out); });
}

bosp_status bosp_block_axpy(int64_t n, int64_t a, int64_t b, const double* x, const double* c, double* y) {
    return guarded([&] {
        bosp::BlockVectors yy = host_block(y, n, b);
        bosp::block_axpy(host_block(x, n, a), host_dense(c, a, b), yy);
        copy_out(yy, y);
    });
}

bosp_status bosp_biorth(int32_t classical, bosp_op B, int64_t n, int64_t m, const double* x, const double* y,
                        double drop_tol, double* p, double* q, int64_t* kept, int64_t* nkept,
                        int64_t* dropped, int64_t* ndropped) {
    return guarded([&] {
        bosp::BiorthOutcome o = classical
            ? bosp::cgs_biorth(host_block(x, n, m), host_block(y, n, m), ip_of(B), drop_tol)
            : bosp::mgs_biorth(host_block(x, n, m), host_block(y, n, m), ip_of(B), drop_tol);
        copy_out(o.basis.p, p);
        copy_out(o.basis.q, q);
        *nkept = static_cast<int64_t>(o.kept_columns.size());
        *ndropped = static_cast<int64_t>(o.dropped_columns.size());
        for (size_t i = 0; i < o.kept_columns.size(); ++i) kept[i] = o.kept_columns[i];
        for (size_t i = 0; i < o.dropped_columns.size(); ++i) dropped[i] = o.dropped_columns[i];
    });
}

bosp_status bosp_biorth_against(bosp_op B, int64_t n, int64_t nbases, const int64_t* widths,
                                const double* const* ps, const double* const* qs, int64_t m,
                                const double* x, const double* y, double* xo, double* yo) {
    return guarded([&] {
        std::vector<bosp::BiorthBasis> store;
        store.reserve(static_cast<size_t>(nbases));
        for (int64_t i = 0; i < nbases; ++i)
            store.push_back({host_block(ps[i], n, widths[i]), host_block(qs[i], n, widths[i])});
        std::vector<const bosp::BiorthBasis*> bases;
        for (auto& b : store) bases.push_back(&b);
        auto [w, z] = bosp::biorth_against(bases, host_block(x, n, m), host_block(y, n, m), ip_of(B));
        copy_out(w, xo);
        copy_out(z, yo);
    });
}

bosp_status bosp_biorth_residual(bosp_op B, int64_t n, int64_t m, const double* p, const double* q, double* out) {
    return guarded([&] { *out = bosp::biorth_residual(host_block(p, n, m), host_block(q, n, m), ip_of(B)); });
}

bosp_status bosp_cg_solve(bosp_op A, int64_t m, const double* rhs, const double* x0, double tol,
                          int64_t max_iter, double* x, int32_t* breakdown, int64_t* max_it_used) {
    return guarded([&] {
        const int64_t n = A->op.dim();
        bosp::BlockVectors xx0 = x0 ? host_block(x0, n, m) : bosp::BlockVectors(n, m);
        bosp::CgResult r = bosp::cg_solve(A->op, host_block(rhs, n, m), xx0, tol, max_iter);
        copy_out(r.x, x);
        *breakdown = r.breakdown ? 1 : 0;
        *max_it_used = r.max_iterations_used;
    });
}

bosp_status bosp_seed_blocks(uint64_t seed, int64_t n, int64_t d, double* u, double* v) {
    return guarded([&] {
        bosp::DBlock du(n, std::max<int64_t>(d, 1)), dv(n, std::max<int64_t>(d, 1));
        du.set_cols(d);
        dv.set_cols(d);
        bosp::mt_fill_uv(seed, du.view(), dv.view());
        bosp::to_host(du.view(), u, n);
        bosp::to_host(dv.view(), v, n);
    });
}

bosp_status bosp_solve_small_lrep(int64_t d, const double* khat, const double* mhat, int64_t k,
                                  double* lambdas, double* xhat, double* yhat) {
    return guarded([&] {
        bosp::ProjectedLrep p = bosp::finish_assembly(host_dense(khat, d, d), host_dense(mhat, d, d));
        bosp::SmallEigenSolution s = bosp::solve_small_lrep(p, k);
        for (int64_t j = 0; j < k; ++j) lambdas[j] = s.lambdas[j];
        std::memcpy(xhat, s.xhat.data(), sizeof(double) * d * k);
        std::memcpy(yhat, s.yhat.data(), sizeof(double) * d * k);
    });
}

bosp_status bosp_jacobi_svd(int64_t m, int64_t k, const double* a, double* u, double* sigma, double* v,
                            int64_t* sweeps, int32_t* converged) {
    return guarded([&] {
        bosp::JacobiSvdResult r = bosp::jacobi_svd(host_dense(a, m, k));
        std::memcpy(u, r.u.data(), sizeof(double) * m * k);
        std::memcpy(v, r.v.data(), sizeof(double) * k * k);
        for (int64_t j = 0; j < k; ++j) sigma[j] = r.sigma[j];
        *sweeps = r.sweeps;
        *converged = r.converged ? 1 : 0;
    });
}

bosp_status bosp_cholesky(int64_t n, const double* a, double* l, int32_t* ok) {
    return guarded([&] {
        auto r = bosp::cholesky_lower(host_dense(a, n, n));
        *ok = r ? 1 : 0;
        if (r) std::memcpy(l, r->data(), sizeof(double) * n * n);
    });
}

void bosp_profile_enable(const char* family) {
    try {
        bosp::Runtime::get().prof_enable(family ? family : "");
    } catch (...) {
    }
}

int64_t bosp_profile_family_report(char* buf, int64_t len) {
    std::string s;
    try {
        char line[256];
        const bosp::Runtime& rt = bosp::Runtime::get();
        for (const auto& kv : rt.prof_by_family()) {
            std::snprintf(line, sizeof(line), "%s %lld %.9g %.17g %.17g\n", kv.first.c_str(),
                          (long long)kv.second.launches, kv.second.ms, kv.second.bytes, kv.second.flops);
            s += line;
        }
        if (rt.last_regions_.launches > 0) {  // composite operations: calls, -, bytes, flops
            std::snprintf(line, sizeof(line), "@region %lld 0 %.17g %.17g\n", (long long)rt.last_regions_.launches,
                          rt.last_regions_.bytes, rt.last_regions_.flops);
            s += line;
        }
    } catch (...) {
    }
    if (buf && len > 0) {
        const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(len - 1));
        std::memcpy(buf, s.data(), n);
        buf[n] = '\0';
    }
    return static_cast<int64_t>(s.size()) + 1;
}

void bosp_profile_collect(int64_t* launches, double* ms, double* bytes, double* flops) {
    bosp_profile_collect_regions(launches, ms, bytes, flops, nullptr, nullptr);
}

void bosp_profile_collect_regions(int64_t* launches, double* ms, double* bytes, double* flops,
                                  int64_t* region_calls, double* region_bytes) {
    try {
        auto r = bosp::Runtime::get().prof_collect();
        *launches = r.launches;
        *ms = r.ms;
        *bytes = r.bytes;
        *flops = r.flops;
        if (region_calls) *region_calls = r.region_calls;
        if (region_bytes) *region_bytes = r.region_bytes;
    } catch (...) {
        *launches = 0;
        *ms = *bytes = *flops = 0.0;
        if (region_calls) *region_calls = 0;
        if (region_bytes) *region_bytes = 0.0;
    }
}

int64_t bosp_launch_count(void) {
    try {
        return bosp::Runtime::get().launches();
    } catch (...) {
        return -1;
    }
}

void bosp_launch_reset(void) {
    try {
        bosp::Runtime::get().reset_launches();
    } catch (...) {
    }
}

int bosp_launch_families(char* buf, int len) {
    std::string s;
    try {
        for (auto& kv : bosp::Runtime::get().family_launches()) s += kv.first + "=" + std::to_string(kv.second) + ";";
    } catch (...) {
        return -1;
    }
    if (buf && len > 0) {
        std::strncpy(buf, s.c_str(), static_cast<size_t>(len - 1));
        buf[len - 1] = 0;
    }
    return static_cast<int>(s.size());
}

void bosp_profiler_range(int on) {
    if (on) cudaProfilerStart();
    else cudaProfilerStop();
}

void bosp_device_sync(void) {
    try {
        bosp::Runtime::get().sync();
    } catch (...) {
    }
}

bosp_status bosp_bench_apply(bosp_op op, int64_t ncols, int64_t reps, double* ms) {
    return guarded([&] {
        const int64_t n = op->op.dim();
        bosp::DBlock x(n, ncols), y(n, ncols);
        fill_random(x.view(), 1);
        *ms = time_reps(reps, [&] { op->op.apply_device(x.view(), y.view()); });
    });
}

bosp_status bosp_bench_cg(bosp_op op, int64_t ncols, int64_t iters, int64_t reps, double* ms) {
    return guarded([&] {
        const int64_t n = op->op.dim();
        bosp::DBlock b(n, ncols), x(n, ncols);
        fill_random(b.view(), 7);
        bosp::CgWorkspace ws;
        *ms = time_reps(reps, [&] { bosp::dev_cg(op->op, b.view(), x.view(), 0.0, iters, ws); }) /
              static_cast<double>(std::max<int64_t>(iters, 1));
    });
}

bosp_status bosp_bench_blas(int32_t kind, int64_t n, int64_t a, int64_t b, int64_t reps, double* ms) {
    return guarded([&] {
        bosp::DBlock x(n, a), y(n, b), c(std::max<int64_t>(a, b), std::max<int64_t>(a, b));
        fill_random(x.view(), 1);
        fill_random(y.view(), 2);
        fill_random(c.view(), 3);
        if (kind == 0)
            *ms = time_reps(reps, [&] { bosp::gram(bosp::ColList(x.view()), bosp::ColList(y.view()), n, c.data(), c.ld()); });
        else if (kind == 3) {  // the MGS triple XᵀX, XᵀY, YᵀY in one launch
            bosp::DBlock c2(std::max<int64_t>(a, b), std::max<int64_t>(a, b)), c3(std::max<int64_t>(a, b), std::max<int64_t>(a, b));
            const bosp::GramJob jobs[3] = {{bosp::ColList(x.view()), bosp::ColList(x.view()), c.data(), c.ld()},
                                           {bosp::ColList(x.view()), bosp::ColList(y.view()), c2.data(), c2.ld()},
                                           {bosp::ColList(y.view()), bosp::ColList(y.view()), c3.data(), c3.ld()}};
            *ms = time_reps(reps, [&] { bosp::gram(jobs, 3, n); });
        } else if (kind == 5) {  // fused MGS-Biorth apply (a = b <= 32): P = X A, Q = Y B, P^T Q
            bosp::DBlock p(n, a), q(n, a), z(a, 2 * a), g(a, a);
            fill_random(z.view(), 4);
            *ms = time_reps(reps, [&] {
                bosp::biorth_apply(x.view(), y.view().cols_range(0, a), z.data(), z.data() + a * z.ld(), z.ld(),
                                   static_cast<int>(a), p.view(), q.view(), g.data(), g.ld());
            });
        } else if (kind == 6) {  // one whole MGS-Biorth call (a = b columns): pair Gram, coefficient
                                 // recurrence, fused apply + check Gram (48 n m bytes)
            bosp::DBlock p(n, a), q(n, a);
            *ms = time_reps(reps, [&] {
                bosp::dev_mgs_biorth(x.view(), y.view().cols_range(0, a), p.view(), q.view(), bosp::InnerProduct(), 1e-12);
            });
        } else if (kind == 7) {  // kind 6 with the L2 flushed before every call
            bosp::DBlock p(n, a), q(n, a);
            *ms = time_reps_cold(reps, [&] {
                bosp::dev_mgs_biorth(x.view(), y.view().cols_range(0, a), p.view(), q.view(), bosp::InnerProduct(), 1e-12);
            });
        } else if (kind == 4) {  // the same three blocks as one symmetric Gram of Z = [X | Y]
            bosp::DBlock z(a + b, a + b);
            bosp::GramJob job{bosp::ColList(x.view()).add(y.view()), bosp::ColList(x.view()).add(y.view()),
                              z.data(), z.ld()};
            job.sym = true;
            *ms = time_reps(reps, [&] { bosp::gram(&job, 1, n); });
        }
        else
            *ms = time_reps(reps, [&] {
                bosp::product(bosp::ColList(x.view()), c.data(), c.ld(), static_cast<int32_t>(b), y.view(),
                              kind == 1 ? 1.0 : -1.0, kind == 1 ? 0.0 : 1.0);
            });
    });
}

int bosp_set_device(int device) {
    return cudaSetDevice(device) == cudaSuccess ? 0 : -1;
}

void bosp_flush_l2(int64_t bytes) {
    try {
        bosp::Runtime& rt = bosp::Runtime::get();
        static void* buf = nullptr;
        static int64_t cap = 0;
        if (bytes > cap) {
            if (buf) cudaFree(buf);
            BOSP_CUDA(cudaMalloc(&buf, static_cast<size_t>(bytes)));
            cap = bytes;
        }
        BOSP_CUDA(cudaMemsetAsync(buf, cap & 1, static_cast<size_t>(bytes), rt.stream()));
        rt.sync();
    } catch (...) {
    }
}

void* bosp_host_alloc(int64_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, static_cast<size_t>(bytes)) != cudaSuccess) return nullptr;
    return p;
}

void bosp_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

}  // extern "C"
