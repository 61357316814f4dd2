// Generalized nullspace detection on the device (nullspace.cpp:14-193): power iteration for
// ||K||, shifted block inverse iteration with the batched CG -- made robust by a Rayleigh-Ritz
// step per sweep and an early shift schedule (the reference misdetects
// rank 0 on T(-1)/T(0) at n >= 1000) -- CG for M y = B x and the Cholesky normalisation
// X0 = X C^-1, Y0 = Y C^-1.  One-time setup, not the hot loop.
#include <cmath>
#include <limits>

#include "api.hpp"
#include "dev_algos.hpp"
#include "operators.hpp"

namespace bosp {
inline namespace b200 {

namespace {

double col_norm(const DMat& v) {
    DBlock s(1, 1);
    col_dots(v, v, s.data());
    double h = 0.0;
    to_host(s.view(), &h, 1);
    return std::sqrt(h);
}

// Euclidean orthonormalisation, two classical passes per column (nullspace.cpp:38-50 does
// two modified passes; same span and normalisation).
void orthonormalize(const DMat& v) {
    for (int64_t j = 0; j < v.cols; ++j) {
        const DMat vj = v.cols_range(j, 1);
        if (j > 0) {
            const DMat prev = v.cols_range(0, j);
            DBlock c(j, 1);
            for (int pass = 0; pass < 2; ++pass) {
                gram(ColList(prev), ColList(vj), v.rows, c.data(), c.ld());
                Runtime::get().allreduce(c.data(), c.ld());
                product(ColList(prev), c.data(), c.ld(), 1, vj, -1.0, 1.0);
            }
        }
        const double nrm = col_norm(vj);
        if (nrm > 0.0) axpby(1.0 / nrm, vj, 0.0, vj);
    }
}

// Global row count (row-partitioned ranks) or the local one.
int64_t global_dim(int64_t n) {
    const Runtime& rt = Runtime::get();
    return rt.nranks() > 1 ? rt.n_global() : n;
}

// The full n_global x cols random block is drawn on every rank and each keeps its own rows, so
// a partitioned run starts from exactly the serial run's vectors.
void fill_host_uniform(DBlock& b, std::mt19937_64& rng) {
    const Runtime& rt = Runtime::get();
    const int64_t ng = global_dim(b.rows());
    BlockVectors h(ng, b.ncols());
    h.fill_uniform(rng);
    const int64_t r0 = rt.nranks() > 1 ? rt.row0() : 0;
    to_device(h.data() + r0, b.rows(), b.ncols(), ng, b.view());
}

}  // namespace

double estimate_operator_norm(const LinearOperator& op, int64_t iters, uint64_t seed) {
    const int64_t n = op.dim();
    std::mt19937_64 rng(seed);
    DBlock v(n, 1), av(n, 1);
    fill_host_uniform(v, rng);
    double nrm = col_norm(v.view());
    if (nrm == 0.0) return 0.0;
    axpby(1.0 / nrm, v.view(), 0.0, v.view());
    double est = 0.0;
    for (int64_t it = 0; it < iters; ++it) {
        op.apply_device(v.view(), av.view());
        est = col_norm(av.view());
        if (est == 0.0) return 0.0;
        axpby(1.0 / est, av.view(), 0.0, v.view());
    }
    return est;
}

GeneralizedNullspace compute_nullspace(const LinearOperator& k, const LinearOperator& m,
                                       std::optional<int64_t> r_hint, double tol_null,
                                       const InnerProduct& ip, uint64_t seed) {
    const int64_t n = k.dim();
    if (m.dim() != n) throw ContractViolation("compute_nullspace: K and M dimension mismatch");
    const double knorm = std::max(estimate_operator_norm(k, 50, 12345), 1e-300);
    const double zero_thresh = tol_null * knorm;
    const int64_t ng = global_dim(n);
    int64_t block = std::min<int64_t>(r_hint ? *r_hint + 1 : 3, ng);
    std::mt19937_64 rng(seed);
    CgWorkspace ws;
    for (;;) {
        // smallest_eigenpairs (nullspace.cpp:61-131)
        double sigma = 1e-3 * knorm;
        LinearOperator shifted = LinearOperator::shifted(k, sigma);
        DBlock v(n, block), kv(n, block), tmp(n, block), sc(block, 2);
        fill_host_uniform(v, rng);
        orthonormalize(v.view());
        std::vector<double> rayleigh(static_cast<size_t>(block), knorm), resid(static_cast<size_t>(block), knorm);
        double prev_min = std::numeric_limits<double>::infinity();
        double refine_prev = std::numeric_limits<double>::infinity();
        int refine_sweeps = 0;
        for (int outer = 0; outer < 300; ++outer) {
            dev_cg(shifted, v.view(), tmp.view(), 1e-10, 10 * ng, ws);
            copy_block(tmp.view(), v.view());
            orthonormalize(v.view());
            k.apply_device(v.view(), kv.view());
            // Rayleigh-Ritz on the block (new vs nullspace.cpp:78-93, which takes per-vector
            // Rayleigh quotients): a null direction spread over several iterates shows up as one
            // Ritz value ~ 0 instead of several mixed quotients above zero_thresh -- the reason
            // the reference misdetects rank 0 on T(-1)/T(0) at n >= 1000
            {
                DenseMatrix h = ip_gram_host(InnerProduct{}, v.view(), kv.view()).symmetrized();
                JacobiSvdResult e = jacobi_svd(h);  // H is PSD: singular = eigen pairs, ascending
                DBlock z(block, block);
                to_device(e.v.data(), block, block, block, z.view());
                product(ColList(v.view()), z.data(), z.ld(), static_cast<int32_t>(block), tmp.view(), 1.0, 0.0);
                copy_block(tmp.view(), v.view());
                product(ColList(kv.view()), z.data(), z.ld(), static_cast<int32_t>(block), tmp.view(), 1.0, 0.0);
                copy_block(tmp.view(), kv.view());
            }
            col_dots(v.view(), kv.view(), sc.data());
            to_host(sc.cols(0, 1), rayleigh.data(), block);
            // residual ||K v - theta v||
            std::vector<double> neg(rayleigh.size());
            for (size_t j = 0; j < neg.size(); ++j) neg[j] = -rayleigh[j];
            DBlock th(block, 1);
            to_device(neg.data(), block, 1, block, th.view());
            copy_block(kv.view(), tmp.view());
            lam_axpy(v.view(), th.data(), tmp.view());
            col_dots(tmp.view(), tmp.view(), sc.data() + sc.ld());
            to_host(sc.cols(1, 1), resid.data(), block);
            for (auto& r : resid) r = std::sqrt(r);

            double theta_min = std::numeric_limits<double>::infinity();
            double theta_pos = std::numeric_limits<double>::infinity();  // smallest non-null Ritz value
            bool null_converged = true, any_null = false;
            for (int64_t j = 0; j < block; ++j) {
                theta_min = std::min(theta_min, std::fabs(rayleigh[j]));
                if (std::fabs(rayleigh[j]) < zero_thresh) {
                    any_null = true;
                    if (resid[j] > zero_thresh) null_converged = false;
                } else {
                    theta_pos = std::min(theta_pos, std::fabs(rayleigh[j]));
                }
            }
            if (any_null && null_converged && outer >= 2) {
                // Detected (the reference stops here).  A residual <= zero_thresh leaves the null
                // vectors accurate only to ~zero_thresh / lambda_1 (1e-5 for T(-1) at n = 1000,
                // too loose to deflate a 1e-10 solve), so keep sweeping while the largest null
                // residual still halves, down to ~1e-14 ||K||.
                double worst = 0.0;
                for (int64_t j = 0; j < block; ++j)
                    if (std::fabs(rayleigh[j]) < zero_thresh) worst = std::max(worst, resid[j]);
                if (worst <= 1e-14 * knorm || !(worst < 0.5 * refine_prev) || ++refine_sweeps > 12) break;
                refine_prev = worst;
            }
            if (!any_null) {
                int64_t jmin = 0;
                for (int64_t j = 1; j < block; ++j)
                    if (std::fabs(rayleigh[j]) < std::fabs(rayleigh[jmin])) jmin = j;
                const double theta = std::fabs(rayleigh[jmin]);
                if (outer >= 4 && theta - resid[jmin] > zero_thresh && resid[jmin] < 1e-2 * theta &&
                    std::fabs(theta - prev_min) < 1e-4 * theta)
                    break;
            }
            // Shift a decade below the smallest non-null Ritz value from the third sweep on
            // (the reference moves it only after a stall, ~1e-3 relative change, which at
            // n = 4000 never happens within 300 sweeps): the null directions then gain ~10x
            // per sweep over the smallest positive eigenvalue.  The batched CG solves
            // (K + sigma I) to 1e-10 regardless of the conditioning.
            if (outer >= 2 && std::isfinite(theta_pos)) {
                const double target = std::max({theta_pos / 10.0, 1e-14 * knorm, 1e-300});
                if (target < sigma / 2.0) {
                    sigma = target;
                    shifted = LinearOperator::shifted(k, sigma);
                }
            }
            prev_min = theta_min;
        }
        int64_t r = 0;
        for (int64_t j = 0; j < block; ++j)
            if (std::fabs(rayleigh[j]) < zero_thresh) ++r;
        if (r == block && block < ng) {
            block = std::min(ng, block * 2);
            continue;
        }
        if (r_hint && r != *r_hint)
            throw RankMismatch("compute_nullspace: detected rank " + std::to_string(r) + " but hint was " +
                               std::to_string(*r_hint));
        GeneralizedNullspace ns;
        ns.r = r;
        ns.x0 = BlockVectors(n, r);
        ns.y0 = BlockVectors(n, r);
        if (r == 0) return ns;
        DBlock xr(n, r), yr(n, r), rhs(n, r);
        int64_t at = 0;
        for (int64_t j = 0; j < block; ++j)
            if (std::fabs(rayleigh[j]) < zero_thresh) copy_block(v.cols(j, 1), xr.cols(at++, 1));
        apply_weight(ip, xr.view(), rhs.view());
        dev_cg(m, rhs.view(), yr.view(), 1e-12, 10 * ng, ws);
        DenseMatrix gram_h = ip_gram_host(ip, xr.view(), yr.view()).symmetrized();
        auto chol = cholesky_lower(gram_h);
        if (!chol) throw InvalidNullspace("compute_nullspace: nullspace Gram matrix is not SPD");
        DenseMatrix cinv = lu_inverse(chol->transposed());
        DBlock cd(r, r), xo(n, r), yo(n, r);
        to_device(cinv.data(), r, r, r, cd.view());
        product(ColList(xr.view()), cd.data(), cd.ld(), static_cast<int32_t>(r), xo.view(), 1.0, 0.0);
        product(ColList(yr.view()), cd.data(), cd.ld(), static_cast<int32_t>(r), yo.view(), 1.0, 0.0);
        to_host(xo.view(), ns.x0.data(), n);
        to_host(yo.view(), ns.y0.data(), n);
        return ns;
    }
}

}  // namespace b200
}  // namespace bosp
