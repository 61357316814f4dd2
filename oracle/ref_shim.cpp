// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the UNMODIFIED reference BOSP library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libbosp_ref.so).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference leg may load this; the product (paper_2506_08355_b200) never does.
//
// Every entry point forwards to the reference's public C++ API:
//   bosp::solve / initialize / iterate_once      proj/include/bosp/solver/bosp_solver.hpp:85-98
//   LinearOperator::from_dense / from_csr / ...  proj/include/bosp/core/linear_operator.hpp:24-31
//   mgs_biorth / cgs_biorth / biorth_against     proj/include/bosp/biorth/biorth.hpp:30-45
//   block_inner / block_product / block_axpy     proj/include/bosp/core/kernels.hpp:22-30
//   cg_solve                                     proj/include/bosp/core/cg.hpp:17-18
//   solve_small_lrep / jacobi_svd / cholesky     proj/include/bosp/projected/*.hpp
//   compute_nullspace / analytic_nullspace_T     proj/include/bosp/nullspace/nullspace.hpp:27-39
// It also supplies the one symbol the reference cannot build here
// (dense_lrep_oracle needs Eigen, which is absent; proj/src/projected/lrep_oracle.cpp:1).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "bosp/biorth/biorth.hpp"
#include "bosp/core/cg.hpp"
#include "bosp/core/errors.hpp"
#include "bosp/core/kernels.hpp"
#include "bosp/core/linear_operator.hpp"
#include "bosp/core/matrix_market.hpp"
#include "bosp/nullspace/nullspace.hpp"
#include "bosp/projected/dense_kernels.hpp"
#include "bosp/projected/projected_lrep.hpp"
#include "bosp/solver/bosp_solver.hpp"

namespace bosp {
// Eigen-backed test oracle is not buildable in this image; the solver never calls it.
SmallEigenSolution dense_lrep_oracle(const DenseMatrix&, const DenseMatrix&) {
    throw Error("dense_lrep_oracle: Eigen is not available in this build");
}
}  // namespace bosp

namespace {

thread_local std::string g_err;

enum RefKind { REF_DENSE = 0, REF_CSR = 1, REF_DIAG = 2, REF_IDENTITY = 3 };

int status_of(const std::exception& e) {
    if (dynamic_cast<const bosp::ContractViolation*>(&e)) return 1;
    if (dynamic_cast<const bosp::IngestionError*>(&e)) return 2;
    if (dynamic_cast<const bosp::NullspaceLeak*>(&e)) return 3;
    if (dynamic_cast<const bosp::DegenerateSpectrum*>(&e)) return 4;
    if (dynamic_cast<const bosp::RankMismatch*>(&e)) return 5;
    if (dynamic_cast<const bosp::InvalidNullspace*>(&e)) return 6;
    if (dynamic_cast<const bosp::InitializationFailure*>(&e)) return 7;
    if (dynamic_cast<const bosp::NotEnoughSamples*>(&e)) return 8;
    if (dynamic_cast<const bosp::NumericalAbort*>(&e)) return 9;
    return 11;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return status_of(e);
    }
}

bosp::BlockVectors block_from(const double* p, int64_t n, int64_t m) {
    bosp::BlockVectors b(static_cast<size_t>(n), static_cast<size_t>(m));
    if (n * m > 0) std::memcpy(b.data(), p, sizeof(double) * n * m);
    return b;
}

void block_to(const bosp::BlockVectors& b, double* out) {
    if (b.dim() * b.cols() > 0) std::memcpy(out, b.data(), sizeof(double) * b.dim() * b.cols());
}

bosp::DenseMatrix dense_from(const double* p, int64_t r, int64_t c) {
    bosp::DenseMatrix d(static_cast<size_t>(r), static_cast<size_t>(c));
    if (r * c > 0) std::memcpy(d.data(), p, sizeof(double) * r * c);
    return d;
}

void dense_to(const bosp::DenseMatrix& d, double* out) {
    if (d.rows() * d.cols() > 0) std::memcpy(out, d.data(), sizeof(double) * d.rows() * d.cols());
}

}  // namespace

extern "C" {

struct ref_op_desc {
    int32_t kind;
    int64_t n;
    const double* dense;     // n*n column-major (REF_DENSE)
    const int64_t* rowptr;   // n+1 (REF_CSR)
    const int64_t* colidx;   // nnz
    const double* vals;      // nnz (REF_CSR) or n (REF_DIAG)
    int64_t nnz;
};

struct ref_config {
    int64_t nev, nb;
    double tol;
    int64_t ngs, s;
    int32_t moving;  // -1 unset, 0 off, 1 on
    int64_t max_outer_iter;
    uint64_t rng_seed;
    double inner_cg_tol;
    int64_t inner_cg_max_iter;
    double tol_null;
    int64_t rank_hint;  // -1 unset
};

struct ref_stats {
    int64_t iterations, matvec_count, step3_matvecs, step3_vecprods, max_width_u;
    double max_biorth_deviation, max_deflation_crossgram, final_biorth_deviation;
    int32_t nevconv_monotone;
    double wall_seconds;
    int64_t nev_converged;
    int32_t converged;
};

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int t) { bosp::set_kernel_threads(t); }
int ref_threads() { return bosp::kernel_threads(); }

// read_matrix_market (matrix_market.cpp:26-91).  Two calls: sizes first (arrays null), then
// the arrays; the parse of the first call is kept for the second.
int ref_read_matrix_market(const char* path, int64_t* rows, int64_t* cols, int64_t* nnz, int64_t* rowptr,
                           int64_t* colidx, double* vals) {
    static std::string last_path;
    static bosp::SparseMatrixCSR last;
    return guarded([&] {
        if (last_path != path || !rowptr) {
            last = bosp::read_matrix_market(path);
            last_path = path;
        }
        *rows = static_cast<int64_t>(last.rows);
        *cols = static_cast<int64_t>(last.cols);
        *nnz = static_cast<int64_t>(last.values.size());
        if (rowptr)
            for (size_t i = 0; i < last.row_offsets.size(); ++i) rowptr[i] = static_cast<int64_t>(last.row_offsets[i]);
        if (colidx)
            for (size_t i = 0; i < last.col_indices.size(); ++i) colidx[i] = static_cast<int64_t>(last.col_indices[i]);
        if (vals) std::memcpy(vals, last.values.data(), sizeof(double) * last.values.size());
        if (rowptr) last_path.clear();
    });
}

}  // extern "C"

namespace {

bosp::LinearOperator make_op(const ref_op_desc* d) {
    using bosp::LinearOperator;
    switch (d->kind) {
        case REF_DENSE:
            return LinearOperator::from_dense(dense_from(d->dense, d->n, d->n));
        case REF_CSR: {
            bosp::SparseMatrixCSR a;
            a.rows = a.cols = static_cast<size_t>(d->n);
            a.row_offsets.assign(d->rowptr, d->rowptr + d->n + 1);
            a.col_indices.assign(d->colidx, d->colidx + d->nnz);
            a.values.assign(d->vals, d->vals + d->nnz);
            return LinearOperator::from_csr(std::move(a));
        }
        case REF_DIAG:
            return LinearOperator::diagonal(std::vector<double>(d->vals, d->vals + d->n));
        case REF_IDENTITY:
            return LinearOperator::identity(static_cast<size_t>(d->n));
    }
    throw bosp::ContractViolation("ref_shim: unknown operator kind");
}

bosp::BospConfig make_cfg(const ref_config* c) {
    bosp::BospConfig cfg;
    cfg.nev = static_cast<size_t>(c->nev);
    cfg.nb = static_cast<size_t>(c->nb);
    cfg.tol = c->tol;
    cfg.ngs = static_cast<size_t>(c->ngs);
    cfg.s = static_cast<size_t>(c->s);
    if (c->moving >= 0) cfg.moving = (c->moving != 0);
    cfg.max_outer_iter = static_cast<size_t>(c->max_outer_iter);
    cfg.rng_seed = c->rng_seed;
    cfg.inner_cg_tol = c->inner_cg_tol;
    cfg.inner_cg_max_iter = static_cast<size_t>(c->inner_cg_max_iter);
    cfg.tol_null = c->tol_null;
    if (c->rank_hint >= 0) cfg.rank_hint = static_cast<size_t>(c->rank_hint);
    return cfg;
}

bosp::InnerProduct make_ip(const ref_op_desc* b) {
    if (b == nullptr) return bosp::InnerProduct{};
    return bosp::InnerProduct(make_op(b));
}

bosp::GeneralizedNullspace make_ns(int64_t n, int64_t r, const double* x0, const double* y0) {
    bosp::GeneralizedNullspace ns;
    ns.r = static_cast<size_t>(r);
    ns.x0 = block_from(x0, r > 0 ? n : n, r);
    ns.y0 = block_from(y0, r > 0 ? n : n, r);
    return ns;
}

void fill_stats(const bosp::SolverStats& s, ref_stats* o) {
    o->iterations = static_cast<int64_t>(s.iterations);
    o->matvec_count = static_cast<int64_t>(s.matvec_count);
    o->step3_matvecs = static_cast<int64_t>(s.step3_matvecs);
    o->step3_vecprods = static_cast<int64_t>(s.step3_vecprods);
    o->max_width_u = static_cast<int64_t>(s.max_width_u);
    o->max_biorth_deviation = s.max_biorth_deviation;
    o->max_deflation_crossgram = s.max_deflation_crossgram;
    o->final_biorth_deviation = s.final_biorth_deviation;
    o->nevconv_monotone = s.nevconv_monotone ? 1 : 0;
    o->wall_seconds = s.wall_seconds;
}

}  // namespace

extern "C" {

// Full solve through bosp::solve (bosp_solver.cpp:513-536).  have_ns=0 lets the
// reference compute the nullspace itself (compute_nullspace, nullspace.cpp:135).
// Outputs (capacity nev): lambdas, x, y (n x nev col-major), residuals,
// history (iterations x nev, row per iteration; may be null), nevconv history.
int ref_solve(const ref_op_desc* K, const ref_op_desc* M, const ref_op_desc* B,
              const ref_config* c, int32_t have_ns, int64_t r, const double* x0,
              const double* y0, double* lambdas, double* x, double* y, double* residuals,
              int64_t* nout, ref_stats* st, double* history, int64_t history_cap,
              int64_t* history_rows) {
    return guarded([&] {
        bosp::LinearOperator k = make_op(K), m = make_op(M);
        bosp::InnerProduct ip = make_ip(B);
        bosp::BospConfig cfg = make_cfg(c);
        std::optional<bosp::GeneralizedNullspace> ns;
        if (have_ns) ns = make_ns(K->n, r, x0, y0);
        bosp::EigenResult res = bosp::solve(k, m, ip, cfg, std::move(ns));
        const size_t have = res.lambdas.size();
        *nout = static_cast<int64_t>(have);
        for (size_t j = 0; j < have; ++j) {
            lambdas[j] = res.lambdas[j];
            residuals[j] = res.residuals[j];
        }
        if (x) block_to(res.x, x);
        if (y) block_to(res.y, y);
        fill_stats(res.stats, st);
        st->nev_converged = static_cast<int64_t>(res.nev_converged);
        st->converged = res.converged ? 1 : 0;
        if (history_rows) *history_rows = static_cast<int64_t>(res.history.size());
        if (history) {
            const size_t rows = std::min<size_t>(res.history.size(), static_cast<size_t>(history_cap));
            for (size_t i = 0; i < rows; ++i)
                for (size_t j = 0; j < static_cast<size_t>(c->nev); ++j)
                    history[i * c->nev + j] = j < res.history[i].size() ? res.history[i][j] : 0.0;
        }
    });
}

// Bounded-sample CPU timing: initialize + up to k_iters iterate_once calls through
// the public API (bosp_solver.hpp:85-93).  Times are steady_clock seconds.
int ref_time_iterations(const ref_op_desc* K, const ref_op_desc* M, const ref_op_desc* B,
                        const ref_config* c, int64_t r, const double* x0, const double* y0,
                        int64_t k_iters, double* t_init, double* t_iters, int64_t* iters_done,
                        int32_t* converged, int64_t* nev_conv) {
    return guarded([&] {
        bosp::LinearOperator k = make_op(K), m = make_op(M);
        bosp::InnerProduct ip = make_ip(B);
        bosp::BospConfig cfg = make_cfg(c);
        bosp::GeneralizedNullspace ns = make_ns(K->n, r, x0, y0);
        auto t0 = std::chrono::steady_clock::now();
        bosp::SolverState st = bosp::initialize(k, m, ip, ns, cfg);
        auto t1 = std::chrono::steady_clock::now();
        int64_t done = 0;
        bool conv = false;
        while (done < k_iters) {
            ++done;
            if (bosp::iterate_once(st, k, m, ip, ns, cfg)) {
                conv = true;
                break;
            }
        }
        auto t2 = std::chrono::steady_clock::now();
        *t_init = std::chrono::duration<double>(t1 - t0).count();
        *t_iters = std::chrono::duration<double>(t2 - t1).count();
        *iters_done = done;
        *converged = conv ? 1 : 0;
        *nev_conv = static_cast<int64_t>(st.nev_conv);
    });
}

// The initial random fill, exactly as initialize() draws it (bosp_solver.cpp:144-150,
// block_vectors.cpp:27-30): one mt19937_64(seed) stream, uniform [-1,1).
int ref_fill_uniform(uint64_t seed, int64_t count, double* out) {
    return guarded([&] {
        std::mt19937_64 rng(seed);
        bosp::BlockVectors b(static_cast<size_t>(count), 1);
        b.fill_uniform(rng);
        block_to(b, out);
    });
}

int ref_op_apply(const ref_op_desc* A, int64_t m, const double* x, double* y) {
    return guarded([&] {
        bosp::LinearOperator op = make_op(A);
        bosp::BlockVectors out = op.apply(block_from(x, A->n, m));
        block_to(out, y);
    });
}

int ref_block_inner(const ref_op_desc* B, int64_t n, int64_t a, int64_t b, const double* x,
                    const double* y, double* g) {
    return guarded([&] {
        bosp::InnerProduct ip = make_ip(B);
        dense_to(bosp::block_inner(ip, block_from(x, n, a), block_from(y, n, b)), g);
    });
}

int ref_block_product(int64_t n, int64_t a, int64_t b, const double* x, const double* c,
                      double* out) {
    return guarded([&] {
        block_to(bosp::block_product(block_from(x, n, a), dense_from(c, a, b)), out);
    });
}

int ref_block_axpy(int64_t n, int64_t a, int64_t b, const double* x, const double* c,
                   double* y) {
    return guarded([&] {
        bosp::BlockVectors yy = block_from(y, n, b);
        bosp::block_axpy(block_from(x, n, a), dense_from(c, a, b), yy);
        block_to(yy, y);
    });
}

// mgs_biorth / cgs_biorth (biorth.cpp:102-114). P, Q receive kept columns (n x nkept).
int ref_biorth(int32_t classical, const ref_op_desc* B, int64_t n, int64_t m, const double* x,
               const double* y, double drop_tol, double* p, double* q, int64_t* kept,
               int64_t* nkept, int64_t* dropped, int64_t* ndropped) {
    return guarded([&] {
        bosp::InnerProduct ip = make_ip(B);
        bosp::BiorthOutcome o = classical
            ? bosp::cgs_biorth(block_from(x, n, m), block_from(y, n, m), ip, drop_tol)
            : bosp::mgs_biorth(block_from(x, n, m), block_from(y, n, m), ip, drop_tol);
        block_to(o.basis.p, p);
        block_to(o.basis.q, q);
        *nkept = static_cast<int64_t>(o.kept_columns.size());
        *ndropped = static_cast<int64_t>(o.dropped_columns.size());
        for (size_t i = 0; i < o.kept_columns.size(); ++i) kept[i] = static_cast<int64_t>(o.kept_columns[i]);
        for (size_t i = 0; i < o.dropped_columns.size(); ++i) dropped[i] = static_cast<int64_t>(o.dropped_columns[i]);
    });
}

// biorth_against (biorth.cpp:116-133) with nbases pairs; widths[i] columns each.
int ref_biorth_against(const ref_op_desc* B, int64_t n, int64_t nbases, const int64_t* widths,
                       const double* const* ps, const double* const* qs, int64_t m,
                       const double* x, const double* y, double* xo, double* yo) {
    return guarded([&] {
        bosp::InnerProduct ip = make_ip(B);
        std::vector<bosp::BiorthBasis> store;
        store.reserve(static_cast<size_t>(nbases));
        for (int64_t i = 0; i < nbases; ++i)
            store.push_back(bosp::BiorthBasis{block_from(ps[i], n, widths[i]),
                                              block_from(qs[i], n, widths[i]), ip});
        std::vector<const bosp::BiorthBasis*> bases;
        for (auto& b : store) bases.push_back(&b);
        auto [w, z] = bosp::biorth_against(bases, block_from(x, n, m), block_from(y, n, m), ip);
        block_to(w, xo);
        block_to(z, yo);
    });
}

int ref_biorth_residual(const ref_op_desc* B, int64_t n, int64_t m, const double* p,
                        const double* q, double* out) {
    return guarded([&] {
        *out = bosp::biorth_residual(block_from(p, n, m), block_from(q, n, m), make_ip(B));
    });
}

int ref_cg_solve(const ref_op_desc* A, int64_t m, const double* rhs, const double* x0,
                 double tol, int64_t max_iter, double* x, int32_t* breakdown,
                 int64_t* max_it_used) {
    return guarded([&] {
        bosp::LinearOperator op = make_op(A);
        bosp::CgResult r = bosp::cg_solve(op, block_from(rhs, A->n, m), block_from(x0, A->n, m),
                                          tol, static_cast<size_t>(max_iter));
        block_to(r.x, x);
        *breakdown = r.breakdown ? 1 : 0;
        *max_it_used = static_cast<int64_t>(r.max_iterations_used);
    });
}

// assemble (finish_assembly, projected_lrep.cpp:13-25) of already-projected d x d
// blocks + solve_small_lrep (projected_lrep.cpp:48-80).
int ref_solve_small_lrep(int64_t d, const double* khat, const double* mhat, int64_t k,
                         double* lambdas, double* xhat, double* yhat) {
    return guarded([&] {
        bosp::BlockVectors eye(static_cast<size_t>(d), static_cast<size_t>(d));
        for (int64_t i = 0; i < d; ++i) eye(i, i) = 1.0;
        bosp::ProjectedLrep p = bosp::assemble_projected_applied(
            eye, block_from(khat, d, d), eye, block_from(mhat, d, d));
        bosp::SmallEigenSolution s = bosp::solve_small_lrep(p, static_cast<size_t>(k));
        for (int64_t j = 0; j < k; ++j) lambdas[j] = s.lambdas[j];
        dense_to(s.xhat, xhat);
        dense_to(s.yhat, yhat);
    });
}

int ref_jacobi_svd(int64_t m, int64_t k, const double* a, double* u, double* sigma, double* v,
                   int64_t* sweeps, int32_t* conv) {
    return guarded([&] {
        bosp::JacobiSvdResult r = bosp::jacobi_svd(dense_from(a, m, k));
        dense_to(r.u, u);
        dense_to(r.v, v);
        for (int64_t j = 0; j < k; ++j) sigma[j] = r.sigma[j];
        *sweeps = static_cast<int64_t>(r.sweeps);
        *conv = r.converged ? 1 : 0;
    });
}

int ref_cholesky(int64_t n, const double* a, double* l, int32_t* ok) {
    return guarded([&] {
        auto r = bosp::cholesky_lower(dense_from(a, n, n));
        *ok = r ? 1 : 0;
        if (r) dense_to(*r, l);
    });
}

int ref_spectral_norm(int64_t r, int64_t c, const double* a, double* out) {
    return guarded([&] { *out = bosp::spectral_norm(dense_from(a, r, c)); });
}

int ref_compute_nullspace(const ref_op_desc* K, const ref_op_desc* M, const ref_op_desc* B,
                          int64_t rank_hint, double tol_null, uint64_t seed, int64_t cap,
                          int64_t* r, double* x0, double* y0) {
    return guarded([&] {
        std::optional<size_t> hint;
        if (rank_hint >= 0) hint = static_cast<size_t>(rank_hint);
        bosp::GeneralizedNullspace ns = bosp::compute_nullspace(make_op(K), make_op(M), hint,
                                                                tol_null, make_ip(B), seed);
        *r = static_cast<int64_t>(ns.r);
        if (static_cast<int64_t>(ns.r) <= cap) {
            block_to(ns.x0, x0);
            block_to(ns.y0, y0);
        }
    });
}

int ref_analytic_nullspace_T(int64_t n, double* x0, double* y0) {
    return guarded([&] {
        bosp::GeneralizedNullspace ns = bosp::analytic_nullspace_T(static_cast<size_t>(n));
        block_to(ns.x0, x0);
        block_to(ns.y0, y0);
    });
}

int ref_regression(const double* history, int64_t rows, int64_t cols, int64_t idx, double tol,
                   double* alpha, double* beta, int32_t* degenerate) {
    return guarded([&] {
        std::vector<std::vector<double>> h(static_cast<size_t>(rows));
        for (int64_t i = 0; i < rows; ++i) h[i].assign(history + i * cols, history + (i + 1) * cols);
        bosp::RegressionFit f = bosp::regression_coefficients(h, static_cast<size_t>(idx), tol);
        *alpha = f.alpha;
        *beta = f.beta;
        *degenerate = f.degenerate ? 1 : 0;
    });
}

}  // extern "C"
