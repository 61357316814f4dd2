// Host-side small dense algebra of the projected problem (stays on the host per the north
// star): Cholesky, one-sided Jacobi SVD, the small LREP solve, the Step-5 Euclidean
// MGS-Biorth, and the coefficient-space form of MGS-Biorth that drives the device kernels.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "common.hpp"

namespace bosp {
inline namespace b200 {

// Column-major host matrix (the reference's DenseMatrix, dense_matrix.hpp:9-56).
class DenseMatrix {
public:
    DenseMatrix() = default;
    DenseMatrix(int64_t rows, int64_t cols) : rows_(rows), cols_(cols), data_(static_cast<size_t>(rows * cols), 0.0) {}
    static DenseMatrix identity(int64_t n);
    static DenseMatrix diagonal(const std::vector<double>& d);

    int64_t rows() const { return rows_; }
    int64_t cols() const { return cols_; }
    double& operator()(int64_t i, int64_t j) { return data_[static_cast<size_t>(i + j * rows_)]; }
    double operator()(int64_t i, int64_t j) const { return data_[static_cast<size_t>(i + j * rows_)]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    double* col(int64_t j) { return data_.data() + j * rows_; }
    const double* col(int64_t j) const { return data_.data() + j * rows_; }

    DenseMatrix transposed() const;
    DenseMatrix symmetrized() const;
    void mirror_lower();
    double max_abs() const;
    double frobenius_norm() const;
    bool is_symmetric(double tol_rel) const;

private:
    int64_t rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

// a_lower: a is lower triangular (its structural zeros are skipped).
DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b, bool a_lower = false);
DenseMatrix matmul_tn(const DenseMatrix& a, const DenseMatrix& b);
// L^T R for square lower-triangular L, R.
DenseMatrix matmul_tn_lower(const DenseMatrix& l, const DenseMatrix& r);

// A = L L^T, or nullopt when a pivot is <= 0 / non-finite (dense_kernels.cpp:11-28).
std::optional<DenseMatrix> cholesky_lower(const DenseMatrix& a);
// cholesky_lower of two matrices of one order at once (threads; bitwise the serial factors).
void cholesky_lower_pair(const DenseMatrix& a, const DenseMatrix& b, std::optional<DenseMatrix>& la,
                         std::optional<DenseMatrix>& lb);

struct JacobiSvdResult {
    DenseMatrix u;
    std::vector<double> sigma;  // ascending
    DenseMatrix v;
    bool converged = true;
    int64_t sweeps = 0;
};
// One-sided Hestenes Jacobi, same rotation formula, threshold (1e-15) and sweep cap (40) as
// dense_kernels.cpp:30-113; the sweep is executed in a parallel round-robin ordering so that
// column pairs of one round rotate concurrently (threads when d is large).
JacobiSvdResult jacobi_svd(DenseMatrix a, int64_t max_sweeps = 40);
// The same with the orthogonality test |x^T y| <= tol ||x|| ||y|| (jacobi_svd: tol = 1e-15).
// accumulate = false: the rotations are not accumulated (res.v empty; U and sigma only).
JacobiSvdResult jacobi_svd_tol(DenseMatrix a, int64_t max_sweeps, double tol, bool accumulate = true);
// Square W: QR-preconditioned one-sided Jacobi (Householder QR with column pivoting, then the
// same Jacobi on R^T); used by solve_small_lrep for d >= 96.  0 <= nvec < k: only the nvec
// smallest singular pairs' vectors (u, v are k x nvec; sigma is complete).
JacobiSvdResult jacobi_svd_qr(const DenseMatrix& w, int64_t max_sweeps = 40, int64_t nvec = -1);
double spectral_norm(const DenseMatrix& a);
DenseMatrix lu_inverse(const DenseMatrix& a);

// Small LREP (projected_lrep.cpp:48-80): W = L^T R, SVD, Yhat = L Phi S^-1/2, Xhat = R Psi S^-1/2.
struct SmallEigenSolution {
    std::vector<double> lambdas;
    DenseMatrix xhat, yhat;
};
struct ProjectedLrep {
    int64_t d = 0;
    DenseMatrix khat, mhat, chol_k, chol_m;
};
// symmetrize + 2 Cholesky (throws NullspaceLeak), projected_lrep.cpp:13-25
ProjectedLrep finish_assembly(const DenseMatrix& khat, const DenseMatrix& mhat);
SmallEigenSolution solve_small_lrep(const ProjectedLrep& p, int64_t k);

// Euclidean column-space MGS-Biorth on host (Step 5 small problem, bosp_solver.cpp:322),
// same semantics as biorth.cpp:19-109.
struct HostBiorth {
    DenseMatrix p, q;
    std::vector<int64_t> kept, dropped;
};
HostBiorth host_mgs_biorth(const DenseMatrix& x, const DenseMatrix& y, double drop_tol = 1e-12);
HostBiorth host_cgs_biorth(const DenseMatrix& x, const DenseMatrix& y, double drop_tol = 1e-12);

// ||G - I||_2 > thr, decided exactly: Frobenius bound first, Jacobi spectral norm only when the
// bound does not settle it (biorth_residual, biorth.cpp:135-143, compared at mgs_biorth :104).
bool biorth_loss_exceeds(const DenseMatrix& g, double thr);
double biorth_loss(const DenseMatrix& g);  // exact spectral ||G - I||_2

// MGS-Biorth in coefficient space.  Given the Grams of the input pair (X, Y) under the inner
// product -- Gxx = <X,X>, Gxy = <X,Y>, Gyy = <Y,Y> -- run the exact column-sequential recurrence
// of gs_biorth (biorth.cpp:19-69: modified projections, norms, drop test, sign/sqrt|eta|
// scaling) on coefficient vectors, so that P = X A and Q = Y B reproduce its output.
struct CoefBiorth {
    DenseMatrix a, b;  // m x k
    std::vector<int64_t> kept, dropped;
};
// The Gram route squares the conditioning of a column that is nearly dependent on the kept
// ones (catastrophic cancellation in a^T Gxx a).  coef_mgs therefore stops at the first column
// whose residual norm^2 falls below cancel_tol x its naive magnitude; `stop` returns that
// column (m when all were processed) so the caller can materialise it in n-space exactly as the
// reference does.  cancel_tol = 0 disables the check.
CoefBiorth coef_mgs(const DenseMatrix& gxx, const DenseMatrix& gxy, const DenseMatrix& gyy,
                    double drop_tol, bool classical = false, double cancel_tol = 0.0,
                    int64_t* stop = nullptr);
// rebiorth_pass (biorth.cpp:72-98) in coefficient space given Gpq = <P, Q> (k x k).
CoefBiorth coef_rebiorth(const DenseMatrix& gpq);

}  // namespace b200
}  // namespace bosp
