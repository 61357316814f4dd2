// A reference-API caller written the way a user of the reference library writes one: only the
// reference's public headers and names (proj/include/bosp/...), size_t everywhere, spans from
// BlockVectors::col, CSR built with csr_from_triplets, a matrix-free ApplyFn operator.  The
// same file compiles against the reference headers and, unchanged, against the B200 build
// (include/bosp/* -> paper_2506_08355_b200/csrc/api.hpp); tests/test_compat.py does both and
// runs the B200 binary on the GPU.
//
// Problem: K = M = T(0), n = 400, the 6 smallest positive eigenvalues,
// whose closed form is 4 sin^2(pi l / (2 (n + 1))).  K comes in as CSR, M as a callback.
#include <cmath>
#include <cstdio>
#include <span>
#include <vector>

#include "bosp/core/block_vectors.hpp"
#include "bosp/core/errors.hpp"
#include "bosp/core/inner_product.hpp"
#include "bosp/core/kernels.hpp"
#include "bosp/core/linear_operator.hpp"
#include "bosp/core/sparse_csr.hpp"
#include "bosp/solver/bosp_solver.hpp"

int main() {
    const std::size_t n = 400, nev = 6;
    std::vector<std::size_t> ti, tj;
    std::vector<double> tv;
    for (std::size_t i = 0; i < n; ++i) {
        ti.push_back(i); tj.push_back(i); tv.push_back(2.0);
        if (i > 0) { ti.push_back(i); tj.push_back(i - 1); tv.push_back(-1.0); }
        if (i + 1 < n) { ti.push_back(i); tj.push_back(i + 1); tv.push_back(-1.0); }
    }
    bosp::SparseMatrixCSR t = bosp::csr_from_triplets(n, n, ti, tj, tv);
    t.check_invariants();
    const bosp::SparseMatrixCSR t_copy = t;

    bosp::LinearOperator k = bosp::LinearOperator::from_csr(std::move(t));
    bosp::LinearOperator m = bosp::LinearOperator::from_callback(
        n, [&t_copy](const bosp::BlockVectors& x, bosp::BlockVectors& y) {
            for (std::size_t j = 0; j < x.cols(); ++j) t_copy.apply(x.col(j), y.col(j));
        });

    bosp::BospConfig cfg;
    cfg.nev = nev;
    cfg.nb = nev;
    cfg.tol = 1e-10;
    bosp::EigenResult r = bosp::solve(k, m, bosp::InnerProduct{}, cfg);
    if (!r.converged || r.lambdas.size() != nev) {
        std::printf("FAIL not converged\n");
        return 1;
    }
    const double pi = std::acos(-1.0);
    double worst = 0.0;
    for (std::size_t l = 0; l < nev; ++l) {
        const double exact = 4.0 * std::pow(std::sin(pi * double(l + 1) / (2.0 * double(n + 1))), 2);
        worst = std::fmax(worst, std::fabs(r.lambdas[l] - exact) / exact);
    }
    // biorthogonality through the public span helpers: x_j^T y_j = 1
    double bi = 0.0;
    for (std::size_t j = 0; j < r.x.cols(); ++j) {
        std::span<const double> xj = r.x.col(j), yj = r.y.col(j);
        bi = std::fmax(bi, std::fabs(bosp::vdot(xj, yj) - 1.0));
    }
    const bosp::InnerProduct ip;
    const double nx = ip.norm(r.x.col(0));
    std::printf("lambda_max_rel_err=%.3e biorth=%.3e iterations=%zu norm_x0=%.6f\n", worst, bi,
                static_cast<std::size_t>(r.iterations), nx);
    try {
        bosp::BospConfig bad;
        bad.nev = 0;
        bosp::solve(k, m, bosp::InnerProduct{}, bad);
        std::printf("FAIL no ContractViolation\n");
        return 1;
    } catch (const bosp::ContractViolation&) {
    }
    return (worst < 1e-11 && bi < 1e-10) ? 0 : 1;
}
