// Kernel-level API on host blocks (same signatures as the reference's kernels.hpp / biorth.hpp /
// cg.hpp): inputs are staged to HBM, the device kernels run, outputs come back.  Used by the
// parity tests and by callers that want single building blocks.
#include <cmath>

#include <cstdlib>

#include "api.hpp"
#include "dev_algos.hpp"
#include "operators.hpp"

namespace bosp {
inline namespace b200 {

namespace {

DBlock up(const BlockVectors& b) {
    DBlock d(b.dim(), std::max<int64_t>(b.cols(), 1));
    d.set_cols(b.cols());
    to_device(b.data(), b.dim(), b.cols(), b.dim(), d.view());
    return d;
}

BlockVectors down(const DMat& m) {
    BlockVectors b(m.rows, m.cols);
    to_host(m, b.data(), m.rows);
    return b;
}

DBlock up_dense(const DenseMatrix& c) {
    DBlock d(c.rows(), std::max<int64_t>(c.cols(), 1));
    d.set_cols(c.cols());
    to_device(c.data(), c.rows(), c.cols(), c.rows(), d.view());
    return d;
}

}  // namespace

DenseMatrix block_inner(const InnerProduct& ip, const BlockVectors& x, const BlockVectors& y) {
    require(x.dim() == y.dim(), "block_inner: dimension mismatch");
    DBlock dx = up(x), dy = up(y);
    return ip_gram_host(ip, dx.view(), dy.view());
}

BlockVectors block_product(const BlockVectors& x, const DenseMatrix& c) {
    require(x.cols() == c.rows(), "block_product: shape mismatch");
    DBlock dx = up(x), dc = up_dense(c);
    DBlock out(x.dim(), std::max<int64_t>(c.cols(), 1));
    out.set_cols(c.cols());
    product(ColList(dx.view()), dc.data(), dc.ld(), static_cast<int32_t>(c.cols()), out.view(), 1.0, 0.0);
    return down(out.view());
}

void block_axpy(const BlockVectors& x, const DenseMatrix& c, BlockVectors& y) {
    require(x.cols() == c.rows() && c.cols() == y.cols() && x.dim() == y.dim(), "block_axpy: shape mismatch");
    DBlock dx = up(x), dc = up_dense(c), dy = up(y);
    product(ColList(dx.view()), dc.data(), dc.ld(), static_cast<int32_t>(c.cols()), dy.view(), -1.0, 1.0);
    to_host(dy.view(), y.data(), y.dim());
}

namespace {
BiorthOutcome biorth_common(const BlockVectors& x, const BlockVectors& y, const InnerProduct& ip,
                            double drop_tol, bool classical) {
    require(x.dim() == y.dim() && x.cols() == y.cols(), "biorth: X and Y must have equal shape");
    DBlock dx = up(x), dy = up(y);
    DBlock p(x.dim(), std::max<int64_t>(x.cols(), 1)), q(x.dim(), std::max<int64_t>(x.cols(), 1));
    // small blocks: the reference's column-sequential recurrence itself (exact order, robust on
    // ill-conditioned input); wide blocks: the level-3 coefficient-space path of the solver
    constexpr int64_t seq_max = 64;
    DevBiorthOutcome o = x.cols() <= seq_max
        ? dev_gs_biorth_seq(dx.view(), dy.view(), p.view(), q.view(), ip, drop_tol, classical)
        : dev_mgs_biorth(dx.view(), dy.view(), p.view(), q.view(), ip, drop_tol, classical);
    BiorthOutcome out;
    out.basis.p = down(p.cols(0, o.kept));
    out.basis.q = down(q.cols(0, o.kept));
    out.kept_columns = o.kept_columns;
    out.dropped_columns = o.dropped_columns;
    return out;
}
}  // namespace

BiorthOutcome mgs_biorth(const BlockVectors& x, const BlockVectors& y, const InnerProduct& ip, double drop_tol) {
    return biorth_common(x, y, ip, drop_tol, false);
}

BiorthOutcome cgs_biorth(const BlockVectors& x, const BlockVectors& y, const InnerProduct& ip, double drop_tol) {
    return biorth_common(x, y, ip, drop_tol, true);
}

std::pair<BlockVectors, BlockVectors> biorth_against(const std::vector<const BiorthBasis*>& bases,
                                                     const BlockVectors& x, const BlockVectors& y,
                                                     const InnerProduct& ip) {
    require(x.dim() == y.dim(), "biorth_against: X and Y dimension mismatch");
    std::vector<DBlock> store;
    std::vector<DevBasis> db;
    for (const BiorthBasis* b : bases) {
        if (b == nullptr || b->p.empty()) continue;
        require(b->p.dim() == x.dim(), "biorth_against: basis dimension mismatch");
        store.push_back(up(b->p));
        store.push_back(up(b->q));
    }
    for (size_t i = 0; i + 1 < store.size(); i += 2) db.push_back({store[i].view(), store[i + 1].view()});
    DBlock dw = up(x), dz = up(y);
    dev_biorth_against(db, dw.view(), dz.view(), ip);
    return {down(dw.view()), down(dz.view())};
}

double biorth_residual(const BlockVectors& p, const BlockVectors& q, const InnerProduct& ip) {
    require(p.dim() == q.dim() && p.cols() == q.cols(), "biorth_residual: shape mismatch");
    if (p.cols() == 0) return 0.0;
    DBlock dp = up(p), dq = up(q);
    return dev_biorth_residual(dp.view(), dq.view(), ip);
}

CgResult cg_solve(const LinearOperator& op, const BlockVectors& rhs, const BlockVectors& x0,
                  double tol, int64_t max_iter) {
    require(rhs.dim() == op.dim() && x0.dim() == op.dim() && rhs.cols() == x0.cols(), "cg_solve: shape mismatch");
    DBlock db = up(rhs), dx0 = up(x0);
    DBlock dx(rhs.dim(), std::max<int64_t>(rhs.cols(), 1));
    dx.set_cols(rhs.cols());
    CgWorkspace ws;
    const DMat x0v = dx0.view();
    DevCgOutcome o = dev_cg(op, db.view(), dx.view(), tol, max_iter, ws, &x0v, true);
    CgResult r;
    r.x = down(dx.view());
    r.breakdown = o.breakdown;
    r.max_iterations_used = o.max_iterations_used;
    return r;
}

GeneralizedNullspace analytic_nullspace_T(int64_t n) {
    if (n < 2) throw ContractViolation("analytic_nullspace_T: n must be >= 2");
    GeneralizedNullspace ns;
    ns.r = 1;
    ns.x0 = BlockVectors(n, 1);
    ns.y0 = BlockVectors(n, 1);
    double eta = 0.0;
    for (int64_t l = 1; l <= n; ++l) {
        const double a = static_cast<double>(l) * static_cast<double>(n - l + 1) / 2.0;
        ns.x0(l - 1, 0) = 1.0;
        ns.y0(l - 1, 0) = a;
        eta += a;
    }
    const double s = 1.0 / std::sqrt(eta);
    for (int64_t i = 0; i < n; ++i) {
        ns.x0(i, 0) *= s;
        ns.y0(i, 0) *= s;
    }
    return ns;
}

}  // namespace b200
}  // namespace bosp
