// Tall-skinny fp64 contractions on the sm_100a DMMA tensor pipe (mma.sync m8n8k4 f64 ->
// SASS DMMA.8x8x4; tcgen05 has no f64 kind) plus the column-wise reductions and element-wise
// kernels of the BOSP outer iteration.
#pragma once

#include "common.hpp"

namespace bosp {
inline namespace b200 {

// ---- Gram: G(a x b) = A^T B over n rows (reference block_inner, kernels.cpp:47-68) ----------
// Up to 4 independent Grams in one launch.  G is column-major with leading dim ldg (device).
struct GramJob {
    ColList a, b;
    double* g;
    int64_t ldg;
    // G is symmetric (A^T A, or U^T (K U) with K symmetric): only the upper-triangular tiles
    // are computed and G(i, j), i <= j, is mirrored to G(j, i) -- G exactly symmetric, ~half
    // the DMMA work.  Requires a.cols() == b.cols().
    bool sym = false;
};
void gram(const GramJob* jobs, int njobs, int64_t n);
inline void gram(const ColList& a, const ColList& b, int64_t n, double* g, int64_t ldg) {
    GramJob j{a, b, g, ldg};
    gram(&j, 1, n);
}

// ---- Product: Out(n x b) = alpha * A(n x k) * C(k x b) + beta * Out -------------------------
// reference block_product / block_axpy (kernels.cpp:70-104); also the dense operator K*X
// (linear_operator.cpp:12-31) with A = K.  C is a device matrix (ldc).  Up to 4 jobs/launch.
struct ProductJob {
    ColList a;          // k columns of n rows
    const double* c;    // k x b
    int64_t ldc;
    int32_t ncols;      // b
    double* out;
    int64_t ldo;
    double alpha, beta;
    // optional (host array of ncols): rows of C that can be nonzero in each column (e.g. the
    // upper-triangular coefficient matrices of MGS-Biorth) -- the K loop of a column tile stops
    // there.  Read at launch time only.
    const int32_t* col_kend = nullptr;
};
void product(const ProductJob* jobs, int njobs, int64_t n);
// MGS-Biorth application fused with its check Gram (x, y widths and kb <= 32): P = X A,
// Q = Y B for the k x kb coefficient matrices A (ca) and B (cb) with leading dimension ldc, and
// G = P^T Q (kb x kb, ldg) from the same pass -- one launch + the split reduction.
// col_kend (optional host array of kb): rows of A and B that can be nonzero per column (the
// triangular coefficients of the first pass) -- the K loop of a column block stops there.
// status_dev (optional device int): nonzero at run time -> the kernel does nothing (coefficients
// produced on the device that turned out invalid; the caller redoes the block).
void biorth_apply(const DMat& x, const DMat& y, const double* ca, const double* cb, int64_t ldc, int kb,
                  const DMat& p, const DMat& q, double* g, int64_t ldg, const int32_t* col_kend = nullptr,
                  const int* status_dev = nullptr);
// MGS-Biorth coefficients of an m <= 32 column block on the device (coef_dev.cu): reads Gxx, Gxy,
// Gyy from the pair Gram z = [X | Y]^T [X | Y] (2m x 2m, ldz), writes A | B (m x 2m, ldc; upper
// triangular) and *status = 0, or *status = 1 when a pivot is zero / a column would be dropped
// or cancels (the host's column-sequential recurrence must decide those).
void coef_mgs_dev(const double* z, int64_t ldz, int m, double* c, int64_t ldc, int* status, double drop_tol,
                  double cancel_tol);
// The pair Gram g = Z^T Z of Z = [X | Y] (2m <= 56 columns, single rank, n >= 8192) with the
// coefficients of coef_mgs_dev fused into its split reduction.  false: not applicable (the
// caller runs gram + allreduce + coef_mgs_dev).
bool gram_pair_coef(const ColList& z, int64_t n, double* g, int64_t ldg, double* c, int64_t ldc, int* status,
                    double drop_tol, double cancel_tol);
inline void product(const ColList& a, const double* c, int64_t ldc, int32_t b, const DMat& out,
                    double alpha, double beta) {
    ProductJob j{a, c, ldc, b, out.p, out.ld, alpha, beta};
    product(&j, 1, out.rows);
}

// ---- Column reductions (deterministic two-level, no atomics on values) ------------------------
// out[j] = sum_i x[i,j] * y[i,j]
void col_dots(const DMat& x, const DMat& y, double* out_dev);
// Normalised residuals of the Ritz window (bosp_solver.cpp:256-272, 487-497):
// num_j = ||kx_j - lam_j yb_j||^2 + ||my_j - lam_j xb_j||^2,  den_j = ||x_j||^2 + ||y_j||^2
void residual_sums(const DMat& kx, const DMat& my, const DMat& xb, const DMat& yb,
                   const DMat& x, const DMat& y, const double* lam_dev, double* num_dev,
                   double* den_dev);

// ---- Element-wise ---------------------------------------------------------------------------
// out[:,j] = lam_j * a[:,j] - b[:,j]   (Step-6 right-hand sides, bosp_solver.cpp:337-350)
void lam_axmy(const DMat& a, const DMat& b, const double* lam_dev, const DMat& out);
// y[:,j] += lam_j * x[:,j]             (Gauss-Seidel coupling, bosp_solver.cpp:354-371)
void lam_axpy(const DMat& x, const double* lam_dev, const DMat& y);
// y = x + sigma * y  (shifted operator epilogue) / y = alpha * x / y = d .* x
void axpby(double a, const DMat& x, double b, const DMat& y);
// y -= s[0] * x with s a device scalar (one column)
void sub_scaled(const DMat& x, const double* s_dev, const DMat& y);
void diag_scale(const double* d_dev, const DMat& x, const DMat& y);
// t = a^T (square or rectangular; t.rows == a.cols, t.cols == a.rows)
void transpose(const DMat& a, const DMat& t);

// ---- Batched multi-RHS CG kernels (reference cg_solve, cg.cpp:11-58) -------------------------
// Per-column scalars live on the device in CgScalars; every kernel honours the column masks, so
// the iterates equal those of the reference's per-column loop.
struct CgScalars {
    double* rr;       // current r^T r
    double* bnorm;    // ||b||
    double* pap;      // p^T A p (this iteration)
    double* beta;     // rr_new / rr (this iteration)
    double* alpha;    // rr / p^T A p of this iteration (0: column not updated), applied to x by
                      // the direction kernel
    int* active;      // column still iterating
    int* broken;      // p^T A p <= 0 hit
    int* iters;       // iterations taken
    int* any_active;  // scalar: number of active columns (device)
    int* loops;       // scalar: batched iterations executed (device)
    unsigned long long* total = nullptr;  // running count of batched iterations over all solves
    double* parts;    // scratch for per-block partial sums (fused SpMM dots)
    int parts_cap;    // doubles available at `parts`
    // When the CG runs as a CUDA graph with a `while` conditional node, the start/update
    // epilogues set the loop condition to (any column still active).
    cudaGraphConditionalHandle cond = 0;
    int has_cond = 0;
    // Optional device scalar: columns >= *m_live are not part of this solve (never read or
    // written, inactive from the start).  Lets one recorded graph serve every narrower call.
    const int* m_live = nullptr;
};
// *p = v on the stream (sets a graph's live width before its launch)
void set_device_int(int* p, int v);
// x = 0, r = b, p = b, rr = ||b||^2, bnorm = ||b||, active = (bnorm != 0 && sqrt(rr) > tol*bnorm)
void cg_start(const DMat& b, const DMat& x, const DMat& r, const DMat& p, const CgScalars& s,
              double tol, int max_iter);
// General start with x0: x = x0, r = b - ax0, p = r, rr = ||r||^2, bnorm = ||b|| (cg.cpp:22-31)
void cg_start_x0(const DMat& b, const DMat& x0, const DMat& ax0, const DMat& x, const DMat& r,
                 const DMat& p, const CgScalars& s, double tol, int max_iter);
// pap_j = p_j^T ap_j (active columns)
void cg_pap(const DMat& p, const DMat& ap, const CgScalars& s);
// active & pap>0: x += a p, r -= a ap, rr_new; pap<=0 -> broken, inactive.  Then
// p = r + beta p, rr = rr_new, active = sqrt(rr) > tol*bnorm && iters < max_iter.
// pap_parts != nullptr: p^T A p is still in per-block partials (pap_parts[j * nparts + b], the
// SpMM's unfolded dots) and every update block folds its column itself.
void cg_update(const DMat& x, const DMat& r, const DMat& p, const DMat& ap, const CgScalars& s,
               double tol, int max_iter, const double* pap_parts = nullptr, int nparts = 0);

}  // namespace b200
}  // namespace bosp
