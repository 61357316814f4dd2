// The remaining public helpers of the reference's headers, so that reference callers compile
// and link against this library unchanged (tests/test_compat.py):
// kernels.hpp:13-21 (vector helpers, kernel thread count), sparse_csr.hpp:24-32 (single-column
// host apply, csr_from_triplets), inner_product.hpp:20-27, projected_lrep.hpp:27-36,
// dense_kernels.hpp:24-40 (estimate_operator_norm, nullspace.hpp:21-23, is nullspace_dev.cpp).  None of these is on the solver's path: the
// solver's block kernels, Grams and applies run on the GPU; what runs here is host algebra on
// host data (spans, small dense matrices) exactly where the reference's caller has it.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>

#include "api.hpp"

namespace bosp {
inline namespace b200 {

// ---- kernels.hpp ------------------------------------------------------------------------
double vdot(std::span<const double> x, std::span<const double> y) {
    require(x.size() == y.size(), "vdot: length mismatch");
    double s = 0.0;
    for (size_t i = 0; i < x.size(); ++i) s += x[i] * y[i];
    return s;
}

double vnorm2(std::span<const double> x) { return std::sqrt(vdot(x, x)); }

void vaxpy(double alpha, std::span<const double> x, std::span<double> y) {
    require(x.size() == y.size(), "vaxpy: length mismatch");
    for (size_t i = 0; i < x.size(); ++i) y[i] += alpha * x[i];
}

void vscale(double alpha, std::span<double> x) {
    for (double& v : x) v *= alpha;
}

namespace {
int g_host_threads = 0;  // 0: OpenMP default
}

void set_kernel_threads(int nthreads) {
    g_host_threads = std::max(0, nthreads);
    if (nthreads > 0) omp_set_num_threads(nthreads);
}

int kernel_threads() { return g_host_threads > 0 ? g_host_threads : omp_get_max_threads(); }

// ---- sparse_csr.hpp ---------------------------------------------------------------------
void SparseMatrixCSR::apply(std::span<const double> x, std::span<double> y) const {
    require(x.size() == cols && y.size() == rows, "SparseMatrixCSR::apply: shape mismatch");
    for (size_t r = 0; r < rows; ++r) {
        double s = 0.0;
        for (size_t k = row_offsets[r]; k < row_offsets[r + 1]; ++k) s += values[k] * x[col_indices[k]];
        y[r] = s;
    }
}

SparseMatrixCSR csr_from_triplets(std::size_t rows, std::size_t cols, std::vector<std::size_t> ti,
                                  std::vector<std::size_t> tj, std::vector<double> tv) {
    require(ti.size() == tj.size() && ti.size() == tv.size(), "csr_from_triplets: length mismatch");
    std::vector<size_t> order(ti.size());
    std::iota(order.begin(), order.end(), size_t(0));
    for (size_t k = 0; k < ti.size(); ++k)
        require(ti[k] < rows && tj[k] < cols, "csr_from_triplets: index out of range");
    std::stable_sort(order.begin(), order.end(),
                     [&](size_t a, size_t b) { return ti[a] != ti[b] ? ti[a] < ti[b] : tj[a] < tj[b]; });
    SparseMatrixCSR m;
    m.rows = rows;
    m.cols = cols;
    m.row_offsets.assign(rows + 1, 0);
    for (size_t k = 0; k < order.size();) {
        const size_t r = ti[order[k]], c = tj[order[k]];
        double v = 0.0;
        while (k < order.size() && ti[order[k]] == r && tj[order[k]] == c) v += tv[order[k++]];
        m.col_indices.push_back(c);
        m.values.push_back(v);
        m.row_offsets[r + 1] = m.values.size();
    }
    for (size_t r = 1; r <= rows; ++r) m.row_offsets[r] = std::max(m.row_offsets[r], m.row_offsets[r - 1]);
    return m;
}

// ---- inner_product.hpp ------------------------------------------------------------------
BlockVectors InnerProduct::apply_weight(const BlockVectors& y) const {
    if (!weighted()) return y.columns(0, y.cols());
    return weight_->apply(y);
}

double InnerProduct::dot(std::span<const double> x, std::span<const double> y) const {
    require(x.size() == y.size(), "InnerProduct::dot: length mismatch");
    if (!weighted()) return vdot(x, y);
    BlockVectors yb(static_cast<int64_t>(y.size()), 1);
    std::copy(y.begin(), y.end(), yb.data());
    const BlockVectors by = weight_->apply(yb);
    return vdot(x, by.col(0));
}

double InnerProduct::norm(std::span<const double> x) const { return std::sqrt(std::max(0.0, dot(x, x))); }

// ---- projected_lrep.hpp -----------------------------------------------------------------
ProjectedLrep assemble_projected_applied(const BlockVectors& u, const BlockVectors& ku, const BlockVectors& v,
                                         const BlockVectors& mv) {
    const InnerProduct euclid;
    return finish_assembly(block_inner(euclid, u, ku), block_inner(euclid, v, mv));
}

ProjectedLrep assemble_projected(const LinearOperator& k, const LinearOperator& m, const BlockVectors& u,
                                 const BlockVectors& v, const InnerProduct& ip) {
    (void)ip;  // (U, V) biorthonormal under ip is the caller's precondition (projected_lrep.cpp:31-33)
    require(u.dim() == k.dim() && v.dim() == m.dim() && u.cols() == v.cols(), "assemble_projected: shape mismatch");
    return assemble_projected_applied(u, k.apply(u), v, m.apply(v));
}

// ---- dense_kernels.hpp ------------------------------------------------------------------
double condition_number_2(const DenseMatrix& a) {
    const JacobiSvdResult s = jacobi_svd(a.rows() >= a.cols() ? a : a.transposed());
    if (s.sigma.empty() || s.sigma.front() == 0.0) return std::numeric_limits<double>::infinity();
    return s.sigma.back() / s.sigma.front();
}

LuFactors lu_factor(DenseMatrix a) {
    require(a.rows() == a.cols(), "lu_factor: matrix not square");
    const int64_t n = a.rows();
    LuFactors f;
    f.perm.resize(static_cast<size_t>(n));
    std::iota(f.perm.begin(), f.perm.end(), size_t(0));
    for (int64_t c = 0; c < n; ++c) {
        int64_t piv = c;
        for (int64_t r = c + 1; r < n; ++r)
            if (std::fabs(a(r, c)) > std::fabs(a(piv, c))) piv = r;
        if (a(piv, c) == 0.0) throw ContractViolation("lu_factor: singular matrix");
        if (piv != c) {
            for (int64_t j = 0; j < n; ++j) std::swap(a(c, j), a(piv, j));
            std::swap(f.perm[c], f.perm[piv]);
        }
        for (int64_t r = c + 1; r < n; ++r) {
            a(r, c) /= a(c, c);
            const double l = a(r, c);
            for (int64_t j = c + 1; j < n; ++j) a(r, j) -= l * a(c, j);
        }
    }
    f.lu = std::move(a);
    return f;
}

std::vector<double> lu_solve(const LuFactors& f, std::vector<double> b) {
    const int64_t n = f.lu.rows();
    require(static_cast<int64_t>(b.size()) == n, "lu_solve: length mismatch");
    std::vector<double> x(b.size());
    for (int64_t i = 0; i < n; ++i) x[i] = b[f.perm[i]];
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = 0; j < i; ++j) x[i] -= f.lu(i, j) * x[j];
    for (int64_t i = n - 1; i >= 0; --i) {
        for (int64_t j = i + 1; j < n; ++j) x[i] -= f.lu(i, j) * x[j];
        x[i] /= f.lu(i, i);
    }
    return x;
}

DenseMatrix lu_solve(const LuFactors& f, const DenseMatrix& b) {
    DenseMatrix x(b.rows(), b.cols());
    for (int64_t c = 0; c < b.cols(); ++c) {
        const std::vector<double> col(b.col(c), b.col(c) + b.rows());
        const std::vector<double> s = lu_solve(f, col);
        std::copy(s.begin(), s.end(), x.col(c));
    }
    return x;
}

DenseMatrix transpose_times(const DenseMatrix& l, const DenseMatrix& r) { return matmul_tn(l, r); }

}  // namespace b200
}  // namespace bosp
