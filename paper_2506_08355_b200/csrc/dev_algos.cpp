// Device orchestration of the biorthogonalization and inner-CG building blocks.
#include "dev_algos.hpp"

#include <atomic>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>

#include "operators.hpp"

namespace bosp {
inline namespace b200 {

namespace {
bool debug_on() {
    static const bool on = std::getenv("BOSP_DEBUG") != nullptr;
    return on;
}
}  // namespace

// ---------------------------------------------------------------------------------------------
// Grams under the inner product
// ---------------------------------------------------------------------------------------------
void apply_weight(const InnerProduct& ip, const DMat& b, const DMat& out) {
    if (ip.weighted()) ip.weight()->apply_device(b, out);
    else copy_block(b, out);
}

void ip_gram_dev(const InnerProduct& ip, const DMat& a, const DMat& b, const DMat& g) {
    Runtime& rt = Runtime::get();
    if (!ip.weighted()) {
        gram(ColList(a), ColList(b), a.rows, g.p, g.ld);
    } else {
        DBlock wb(b.rows, b.cols);
        ip.weight()->apply_device(b, wb.view());
        gram(ColList(a), ColList(wb.view()), a.rows, g.p, g.ld);
    }
    rt.allreduce(g.p, g.ld * g.cols);  // row-partitioned: sum the per-rank partial Grams
}

DenseMatrix ip_gram_host(const InnerProduct& ip, const DMat& a, const DMat& b) {
    DenseMatrix h(a.cols, b.cols);
    if (a.cols == 0 || b.cols == 0) return h;
    DBlock g(a.cols, b.cols);
    ip_gram_dev(ip, a, b, g.view());
    to_host(g.view(), h.data(), h.rows());
    return h;
}

std::vector<DenseMatrix> ip_grams_host(const InnerProduct& ip, const std::vector<std::pair<DMat, DMat>>& pairs) {
    std::vector<DenseMatrix> out;
    std::vector<int64_t> off;
    int64_t total = 0;
    for (const auto& pr : pairs) {
        out.emplace_back(pr.first.cols, pr.second.cols);
        off.push_back(total);
        total += pr.first.cols * pr.second.cols;
    }
    if (total == 0) return out;
    Runtime& rt = Runtime::get();
    DBlock g(total, 1);
    std::vector<DBlock> weighted;
    // Jobs are launched in shape classes (a launch's tile shape follows its widest job): square-
    // ish Grams together, and skinny cross-Grams (Q^T U with Q <= 32 columns, U >= 128) computed
    // as U^T Q on the 128 x 32 tiles and transposed on the host -- in a 320-wide launch a 1 x 320
    // job would cost 5 full 64 x 64 tiles per row split.
    std::vector<GramJob> wide, skinny;
    std::vector<char> swapped(pairs.size(), 0);
    for (size_t i = 0; i < pairs.size(); ++i) {
        const DMat& a = pairs[i].first;
        DMat b = pairs[i].second;
        if (a.cols == 0 || b.cols == 0) continue;
        if (ip.weighted()) {
            weighted.emplace_back(b.rows, b.cols);
            ip.weight()->apply_device(b, weighted.back().view());
            b = weighted.back().view();
        }
        if (a.cols <= 32 && b.cols >= 128) {
            swapped[i] = 1;
            skinny.push_back({ColList(b), ColList(a), g.data() + off[i], b.cols});
        } else {
            wide.push_back({ColList(a), ColList(b), g.data() + off[i], a.cols});
        }
    }
    for (const std::vector<GramJob>* js : {&wide, &skinny})
        for (size_t i = 0; i < js->size(); i += 4)
            gram(js->data() + i, static_cast<int>(std::min<size_t>(4, js->size() - i)), pairs[0].first.rows);
    rt.allreduce(g.data(), total);
    std::vector<double> h(static_cast<size_t>(total));
    BOSP_CUDA(cudaMemcpyAsync(h.data(), g.data(), sizeof(double) * total, cudaMemcpyDeviceToHost, rt.stream()));
    rt.sync();
    for (size_t i = 0; i < pairs.size(); ++i) {
        const double* src = h.data() + off[i];
        DenseMatrix& o = out[i];
        if (!swapped[i]) {
            std::copy(src, src + o.rows() * o.cols(), o.data());
        } else {  // src holds (b^T a), o.cols() x o.rows()
            for (int64_t c = 0; c < o.cols(); ++c)
                for (int64_t r = 0; r < o.rows(); ++r) o(r, c) = src[c + r * o.cols()];
        }
    }
    return out;
}

// ---------------------------------------------------------------------------------------------
// biorth_against: per basis two Grams (one launch) and two in-place axpy products (one launch)
// ---------------------------------------------------------------------------------------------
void dev_biorth_against(const std::vector<DevBasis>& bases, const DMat& w, const DMat& z,
                        const InnerProduct& ip) {
    if (w.cols == 0) return;
    const int64_t m = w.cols;
    size_t i = 0;
    while (i < bases.size()) {
        if (bases[i].p.cols == 0) {
            ++i;
            continue;
        }
        // Concatenated pass: a run of `group` bases (the locked pairs, mutually
        // biorthogonal by construction) is projected at once, W -= [P_1..P_s] ([Q_1..Q_s]^T W),
        // which equals the reference's basis-by-basis order (biorth.cpp:116-133) up to products
        // of cross-Grams (~1e-26): one Gram and one product launch per run of up to kMaxSeg
        // bases instead of one each per basis (config 5 locks up to three 128-column pairs).
        // Other bases (null basis, window X, P~) stay separate: measured faster on config 3.
        ColList pl, ql;
        int64_t k = 0;
        const bool grouped = bases[i].group && !ip.weighted();
        do {
            const DevBasis& b = bases[i];
            require(b.p.rows == w.rows, "biorth_against: basis dimension mismatch");
            if (b.p.cols > 0) {
                pl.add(b.p);
                ql.add(b.q);
                k += b.p.cols;
            }
            ++i;
        } while (grouped && i < bases.size() && bases[i].group && pl.nseg < kMaxSeg);
        DBlock c(k, 2 * m);  // [Cw | Cz]
        const DMat cw = c.cols(0, m), cz = c.cols(m, m);
        if (!ip.weighted()) {
            GramJob jobs[2] = {{ql, ColList(w), cw.p, cw.ld}, {pl, ColList(z), cz.p, cz.ld}};
            gram(jobs, 2, w.rows);
            Runtime::get().allreduce(c.data(), c.ld() * 2 * m);
        } else {  // one basis at a time (grouped is off)
            ip_gram_dev(ip, bases[i - 1].q, w, cw);
            ip_gram_dev(ip, bases[i - 1].p, z, cz);
        }
        ProductJob pj[2] = {{pl, cw.p, cw.ld, static_cast<int32_t>(m), w.p, w.ld, -1.0, 1.0},
                            {ql, cz.p, cz.ld, static_cast<int32_t>(m), z.p, z.ld, -1.0, 1.0}};
        product(pj, 2, w.rows);
    }
}

void dev_project_sampled(const std::vector<DevBasis>& bases, const DMat& w, const DMat& z,
                         const std::vector<DenseMatrix>& cross) {
    const int64_t m = w.cols;
    if (m == 0) return;
    require(cross.size() == 2 * bases.size(), "project_sampled: one Gram pair per basis");
    size_t i = 0;
    while (i < bases.size()) {
        ColList pl, ql;
        std::vector<size_t> idx;
        int64_t k = 0;
        for (; i < bases.size() && pl.nseg < kMaxSeg; ++i) {
            if (bases[i].p.cols == 0) continue;
            pl.add(bases[i].p);
            ql.add(bases[i].q);
            idx.push_back(i);
            k += bases[i].p.cols;
        }
        if (k == 0) continue;
        DenseMatrix cw(k, m), cz(k, m);  // the bases' Grams stacked in segment order
        int64_t r0 = 0;
        for (size_t b : idx) {
            const DenseMatrix& gw = cross[2 * b];
            const DenseMatrix& gz = cross[2 * b + 1];
            require(gw.cols() == m && gz.cols() == m, "project_sampled: Gram width mismatch");
            for (int64_t c = 0; c < m; ++c)
                for (int64_t r = 0; r < gw.rows(); ++r) {
                    cw(r0 + r, c) = gw(r, c);
                    cz(r0 + r, c) = gz(r, c);
                }
            r0 += gw.rows();
        }
        DBlock c(k, 2 * m);
        to_device(cw.data(), k, m, k, c.cols(0, m));
        to_device(cz.data(), k, m, k, c.cols(m, m));
        ProductJob pj[2] = {{pl, c.data(), c.ld(), static_cast<int32_t>(m), w.p, w.ld, -1.0, 1.0},
                            {ql, c.data() + m * c.ld(), c.ld(), static_cast<int32_t>(m), z.p, z.ld, -1.0, 1.0}};
        product(pj, 2, w.rows);
    }
}

// ---------------------------------------------------------------------------------------------
// MGS-Biorth: Grams of the pair -> exact column recurrence on the host in coefficient space
// -> P = X A, Q = Y B on the DMMA pipe -> conditional second pass from the Gram of (P, Q).
// ---------------------------------------------------------------------------------------------
namespace {

// rows of each column of a (m x k) up to its last nonzero: the K bound of a triangular product
std::vector<int32_t> last_nonzero_rows(const DenseMatrix& a) {
    std::vector<int32_t> ke(static_cast<size_t>(a.cols()), 0);
    for (int64_t c = 0; c < a.cols(); ++c)
        for (int64_t r = a.rows() - 1; r >= 0; --r)
            if (a(r, c) != 0.0) {
                ke[c] = static_cast<int32_t>(r + 1);
                break;
            }
    return ke;
}

void apply_coefs(const DMat& x, const DMat& y, const DenseMatrix& a, const DenseMatrix& b,
                 const DMat& p, const DMat& q) {
    const int64_t m = a.rows(), k = a.cols();
    DBlock c(m, 2 * k);
    to_device(a.data(), m, k, m, c.cols(0, k));
    to_device(b.data(), m, k, m, c.cols(k, k));
    // the recurrence's coefficients are upper triangular (column j of P combines x_0..x_j):
    // wide products skip the zero K blocks (about half the DMMA work at d = 320)
    const std::vector<int32_t> ka = last_nonzero_rows(a), kb = last_nonzero_rows(b);
    ProductJob pj[2] = {{ColList(x), c.data(), c.ld(), static_cast<int32_t>(k), p.p, p.ld, 1.0, 0.0},
                        {ColList(y), c.data() + k * c.ld(), c.ld(), static_cast<int32_t>(k), q.p, q.ld, 1.0, 0.0}};
    pj[0].col_kend = ka.data();
    pj[1].col_kend = kb.data();
    product(pj, 2, x.rows);
}

// apply_coefs fused with the P^T Q Gram of the written columns (widths <= 32, unweighted):
// returns P^T Q on the host (allreduced across ranks).
DenseMatrix apply_coefs_gram(const DMat& x, const DMat& y, const DenseMatrix& a, const DenseMatrix& b,
                             const DMat& p, const DMat& q) {
    const int64_t m = a.rows(), k = a.cols();
    DBlock c(m, 2 * k), g(k, k);
    to_device(a.data(), m, k, m, c.cols(0, k));
    to_device(b.data(), m, k, m, c.cols(k, k));
    // triangular coefficients: each column block's K loop stops at its last nonzero row
    std::vector<int32_t> ke = last_nonzero_rows(a);
    const std::vector<int32_t> kbr = last_nonzero_rows(b);
    for (size_t i = 0; i < ke.size(); ++i) ke[i] = std::max(ke[i], kbr[i]);
    biorth_apply(x, y, c.data(), c.data() + k * c.ld(), c.ld(), static_cast<int>(k), p, q, g.data(), g.ld(), ke.data());
    Runtime::get().allreduce(g.data(), g.ld() * k);
    DenseMatrix h(k, k);
    to_host(g.view(), h.data(), k);
    return h;
}

// Gxx = X^T X and Gyy = Y^T Y only (unweighted): two symmetric jobs in one launch.
void self_grams(const DMat& x, const DMat& y, DenseMatrix& gxx, DenseMatrix& gyy) {
    const int64_t m = x.cols;
    DBlock g(m, 2 * m);
    GramJob jobs[2] = {{ColList(x), ColList(x), g.data(), g.ld()}, {ColList(y), ColList(y), g.data() + m * g.ld(), g.ld()}};
    jobs[0].sym = jobs[1].sym = true;
    gram(jobs, 2, x.rows);
    Runtime::get().allreduce(g.data(), g.ld() * 2 * m);
    DenseMatrix both(m, 2 * m);
    to_host(g.view().cols_range(0, 2 * m), both.data(), m);
    gxx = DenseMatrix(m, m);
    gyy = DenseMatrix(m, m);
    std::copy(both.data(), both.data() + m * m, gxx.data());
    std::copy(both.data() + m * m, both.data() + 2 * m * m, gyy.data());
}

// Gxx, Gxy, Gyy of the pair under ip.
void pair_grams(const DMat& x, const DMat& y, const InnerProduct& ip, DenseMatrix& gxx,
                DenseMatrix& gxy, DenseMatrix& gyy) {
    const int64_t m = x.cols;
    if (!ip.weighted()) {
        // one symmetric Gram of Z = [X | Y]: X and Y streamed once, upper tiles only;
        // Z^T Z = [[X^T X, X^T Y], [., Y^T Y]]
        DBlock g(2 * m, 2 * m);
        GramJob job{ColList(x).add(y), ColList(x).add(y), g.data(), g.ld()};
        job.sym = true;
        gram(&job, 1, x.rows);
        Runtime::get().allreduce(g.data(), g.ld() * 2 * m);
        DenseMatrix z(2 * m, 2 * m);
        to_host(g.view(), z.data(), 2 * m);
        gxx = DenseMatrix(m, m);
        gxy = DenseMatrix(m, m);
        gyy = DenseMatrix(m, m);
        for (int64_t j = 0; j < m; ++j)
            for (int64_t i = 0; i < m; ++i) {
                gxx(i, j) = z(i, j);
                gxy(i, j) = z(i, m + j);
                gyy(i, j) = z(m + i, m + j);
            }
        return;
    }
    DBlock g(m, 3 * m);
    if (!ip.weighted()) {
        GramJob jobs[3] = {{ColList(x), ColList(x), g.data(), g.ld()},
                           {ColList(x), ColList(y), g.data() + m * g.ld(), g.ld()},
                           {ColList(y), ColList(y), g.data() + 2 * m * g.ld(), g.ld()}};
        gram(jobs, 3, x.rows);
    } else {
        DBlock wx(x.rows, m), wy(y.rows, m);
        ip.weight()->apply_device(x, wx.view());
        ip.weight()->apply_device(y, wy.view());
        GramJob jobs[3] = {{ColList(x), ColList(wx.view()), g.data(), g.ld()},
                           {ColList(x), ColList(wy.view()), g.data() + m * g.ld(), g.ld()},
                           {ColList(y), ColList(wy.view()), g.data() + 2 * m * g.ld(), g.ld()}};
        gram(jobs, 3, x.rows);
    }
    Runtime::get().allreduce(g.data(), g.ld() * 3 * m);
    DenseMatrix all(m, 3 * m);
    to_host(g.view().cols_range(0, 3 * m), all.data(), m);
    gxx = DenseMatrix(m, m);
    gxy = DenseMatrix(m, m);
    gyy = DenseMatrix(m, m);
    std::copy(all.data(), all.data() + m * m, gxx.data());
    std::copy(all.data() + m * m, all.data() + 2 * m * m, gxy.data());
    std::copy(all.data() + 2 * m * m, all.data() + 3 * m * m, gyy.data());
}

}  // namespace

DevBiorthOutcome dev_mgs_biorth(const DMat& x, const DMat& y, const DMat& p, const DMat& q,
                                const InnerProduct& ip, double drop_tol, bool classical,
                                const DenseMatrix* gxy_hint, bool inputs_scratch) {
    require(x.rows == y.rows && x.cols == y.cols, "biorth: X and Y must have equal shape");
    DevBiorthOutcome out;
    const int64_t m = x.cols, n = x.rows;
    if (m == 0) return out;
    // profiled as one unit ("mgs"): X, Y in and P, Q out (32 n m) + the P^T Q check (16 n m)
    // 4 n m^2 flops of the recurrence + 2 n m^2 for the P^T Q check
    ProfRegion region("mgs", classical ? 32.0 * n * m : 48.0 * n * m,
                      classical ? 4.0 * n * m * m : 6.0 * n * m * m);
    // Columns are processed in order.  Runs of well-conditioned columns go through the Gram /
    // coefficient recurrence (level-3 on the DMMA pipe); a column whose residual cancels
    // (nearly dependent on the kept pairs) is materialised in n-space and projected
    // explicitly, exactly as gs_biorth would, then the remaining columns are projected against
    // the pairs kept so far and the recurrence resumes on them.
    constexpr double kCancel = 1e-8;
    const int passes = classical ? 1 : 2;
    DMat cx = x, cy = y;
    DBlock wx, wy;
    int64_t start = 0, kept = 0;
    DenseMatrix gpq_fused;
    bool have_fused = false;
    // m <= 32, unweighted first pass: pair Gram -> device LDU coefficients -> fused application
    // and check Gram, with no host round trip between the kernels; one read-back (P^T Q and the
    // coefficient status) at the end.  A block the LDU cannot decide exactly (a drop, a
    // cancelling column, a zero pivot) is redone below by the host's column recurrence.
    static const bool dev_coef = !std::getenv("BOSP_DEV_COEF") || std::atoi(std::getenv("BOSP_DEV_COEF")) != 0;
    if (dev_coef && !classical && !ip.weighted() && !gxy_hint && m >= 2 && m <= 32 && n >= 8192) {
        Runtime& rt = Runtime::get();
        DBlock z(2 * m, 2 * m), c(m, 2 * m), g(m, m + 1);
        int* status = reinterpret_cast<int*>(g.data() + m * g.ld());
        if (!gram_pair_coef(ColList(x).add(y), n, z.data(), z.ld(), c.data(), c.ld(), status, drop_tol, kCancel)) {
            GramJob job{ColList(x).add(y), ColList(x).add(y), z.data(), z.ld()};
            job.sym = true;
            gram(&job, 1, n);
            rt.allreduce(z.data(), z.ld() * 2 * m);
            coef_mgs_dev(z.data(), z.ld(), static_cast<int>(m), c.data(), c.ld(), status, drop_tol, kCancel);
        }
        std::vector<int32_t> ke(static_cast<size_t>(m));
        std::iota(ke.begin(), ke.end(), 1);  // upper triangular
        biorth_apply(x, y, c.data(), c.data() + m * c.ld(), c.ld(), static_cast<int>(m), p, q, g.data(), g.ld(),
                     ke.data(), status);
        rt.allreduce(g.data(), g.ld() * m);  // P^T Q (every rank took the same decision)
        std::vector<double> h(static_cast<size_t>(g.ld() * (m + 1)));
        BOSP_CUDA(cudaMemcpyAsync(h.data(), g.data(), sizeof(double) * h.size(), cudaMemcpyDeviceToHost, rt.stream()));
        rt.sync();
        int st = 0;
        std::memcpy(&st, h.data() + m * g.ld(), sizeof(int));
        if (st == 0) {
            gpq_fused = DenseMatrix(m, m);
            for (int64_t j = 0; j < m; ++j)
                for (int64_t i = 0; i < m; ++i) gpq_fused(i, j) = h[i + j * g.ld()];
            have_fused = true;
            kept = m;
            for (int64_t j = 0; j < m; ++j) out.kept_columns.push_back(j);
        }
    }
    for (; !have_fused;) {
        const int64_t mr = cx.cols;
        if (mr == 0) break;
        DenseMatrix gxx, gxy, gyy;
        if (start == 0 && gxy_hint && !ip.weighted() && gxy_hint->rows() == mr && gxy_hint->cols() == mr) {
            self_grams(cx, cy, gxx, gyy);
            gxy = *gxy_hint;
        } else {
            pair_grams(cx, cy, ip, gxx, gxy, gyy);
        }
        int64_t stop = mr;
        const auto tc0 = std::chrono::steady_clock::now();
        CoefBiorth cb = coef_mgs(gxx, gxy, gyy, drop_tol, classical, kCancel, &stop);
        if (debug_on())
            std::fprintf(stderr, "[bosp] mgs m=%lld coef %.2f ms stop=%lld\n", (long long)mr,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count() * 1e3,
                         (long long)stop);
        const int64_t kb = static_cast<int64_t>(cb.kept.size());
        // whole block in one recurrence pass: the check Gram P^T Q comes out of the same kernel
        const bool fuse = !classical && !ip.weighted() && start == 0 && stop >= mr && mr <= 32 && kb >= 2;
        if (fuse) {
            gpq_fused = apply_coefs_gram(cx, cy, cb.a, cb.b, p.cols_range(0, kb), q.cols_range(0, kb));
            have_fused = true;
        } else if (kb > 0) {
            apply_coefs(cx, cy, cb.a, cb.b, p.cols_range(kept, kb), q.cols_range(kept, kb));
        }
        for (int64_t c : cb.kept) out.kept_columns.push_back(start + c);
        for (int64_t c : cb.dropped) out.dropped_columns.push_back(start + c);
        kept += kb;
        if (stop >= mr) break;
        // materialise column `stop`: p~ = x - P_k (Q_k^T x) (twice for MGS), q~ likewise
        DBlock tp(n, 1), tq(n, 1);
        copy_block(cx.cols_range(stop, 1), tp.view());
        copy_block(cy.cols_range(stop, 1), tq.view());
        const std::vector<DevBasis> kb_basis{{p.cols_range(0, kept), q.cols_range(0, kept)}};
        if (kept > 0)
            for (int ps = 0; ps < passes; ++ps) dev_biorth_against(kb_basis, tp.view(), tq.view(), ip);
        DenseMatrix sxx, sxy, syy;
        pair_grams(tp.view(), tq.view(), ip, sxx, sxy, syy);
        const double pn = std::sqrt(std::max(0.0, sxx(0, 0))), qn = std::sqrt(std::max(0.0, syy(0, 0)));
        const double eta = sxy(0, 0);
        if (pn == 0.0 || qn == 0.0 || std::fabs(eta) < drop_tol * pn * qn) {
            out.dropped_columns.push_back(start + stop);
        } else {
            const double sc = 1.0 / std::sqrt(std::fabs(eta)), sg = eta < 0.0 ? -1.0 : 1.0;
            axpby(sg * sc, tp.view(), 0.0, p.cols_range(kept, 1));
            axpby(sc, tq.view(), 0.0, q.cols_range(kept, 1));
            out.kept_columns.push_back(start + stop);
            ++kept;
        }
        const int64_t rest = mr - stop - 1;
        if (rest == 0) break;
        DBlock nx(n, rest), ny(n, rest);
        copy_block(cx.cols_range(stop + 1, rest), nx.view());
        copy_block(cy.cols_range(stop + 1, rest), ny.view());
        const std::vector<DevBasis> all{{p.cols_range(0, kept), q.cols_range(0, kept)}};
        if (kept > 0)
            for (int ps = 0; ps < passes; ++ps) dev_biorth_against(all, nx.view(), ny.view(), ip);
        wx = std::move(nx);
        wy = std::move(ny);
        cx = wx.view();
        cy = wy.view();
        start += stop + 1;
    }
    out.kept = kept;
    if (out.kept == 0) return out;
    const DMat pk = p.cols_range(0, out.kept), qk = q.cols_range(0, out.kept);
    if (classical || out.kept <= 1) return out;
    const DenseMatrix gpq = have_fused ? std::move(gpq_fused) : ip_gram_host(ip, pk, qk);
    if (!biorth_loss_exceeds(gpq, 1e-10)) return out;
    // second subtraction pass (biorth.cpp:104-107)
    out.second_pass = true;
    if (debug_on()) std::fprintf(stderr, "[bosp] mgs m=%lld second pass\n", (long long)out.kept);
    CoefBiorth cb2 = coef_rebiorth(gpq);
    if (inputs_scratch && start == 0) {  // X, Y (never re-pointed) take the result: no copy back
        apply_coefs(pk, qk, cb2.a, cb2.b, x.cols_range(0, out.kept), y.cols_range(0, out.kept));
        out.result_in_inputs = true;
        return out;
    }
    DBlock tp(x.rows, out.kept), tq(x.rows, out.kept);
    apply_coefs(pk, qk, cb2.a, cb2.b, tp.view(), tq.view());
    copy_block(tp.view(), pk);
    copy_block(tq.view(), qk);
    return out;
}

namespace {
// ip.dot(a, b) = a^T B b into a device scalar (one column each)
void ip_dot_dev(const InnerProduct& ip, const DMat& a, const DMat& b, DBlock& wb, double* out) {
    if (ip.weighted()) {
        ip.weight()->apply_device(b, wb.view());
        col_dots(a, wb.view(), out);
    } else {
        col_dots(a, b, out);
    }
}
}  // namespace

DevBiorthOutcome dev_gs_biorth_seq(const DMat& x, const DMat& y, const DMat& p, const DMat& q,
                                   const InnerProduct& ip, double drop_tol, bool classical) {
    require(x.rows == y.rows && x.cols == y.cols, "biorth: X and Y must have equal shape");
    DevBiorthOutcome out;
    const int64_t n = x.rows, m = x.cols;
    if (m == 0) return out;
    Runtime& rt = Runtime::get();
    DBlock pl(n, 1), ql(n, 1), wb(n, 1), sc(8, 1);
    double* r = sc.data();
    double* s = sc.data() + 1;
    double h[3];
    auto norms_eta = [&](const DMat& a, const DMat& b) {  // (a^T B a, b^T B b, a^T B b)
        ip_dot_dev(ip, a, a, wb, sc.data() + 2);
        ip_dot_dev(ip, b, b, wb, sc.data() + 3);
        ip_dot_dev(ip, a, b, wb, sc.data() + 4);
        BOSP_CUDA(cudaMemcpyAsync(h, sc.data() + 2, sizeof(h), cudaMemcpyDeviceToHost, rt.stream()));
        rt.sync();
    };
    int64_t kept = 0;
    for (int64_t l = 0; l < m; ++l) {
        const DMat xl = x.cols_range(l, 1), yl = y.cols_range(l, 1);
        copy_block(xl, pl.view());
        copy_block(yl, ql.view());
        for (int64_t kk = 0; kk < kept; ++kk) {
            const DMat pj = p.cols_range(kk, 1), qj = q.cols_range(kk, 1);
            ip_dot_dev(ip, qj, classical ? xl : pl.view(), wb, r);
            sub_scaled(pj, r, pl.view());
            ip_dot_dev(ip, pj, classical ? yl : ql.view(), wb, s);
            sub_scaled(qj, s, ql.view());
        }
        norms_eta(pl.view(), ql.view());
        const double pn = std::sqrt(h[0]), qn = std::sqrt(h[1]), eta = h[2];
        if (pn == 0.0 || qn == 0.0 || std::fabs(eta) < drop_tol * pn * qn) {
            out.dropped_columns.push_back(l);
            continue;
        }
        const double scale = 1.0 / std::sqrt(std::fabs(eta)), sgn = eta < 0.0 ? -1.0 : 1.0;
        axpby(sgn * scale, pl.view(), 0.0, p.cols_range(kept, 1));
        axpby(scale, ql.view(), 0.0, q.cols_range(kept, 1));
        out.kept_columns.push_back(l);
        ++kept;
    }
    out.kept = kept;
    if (classical || kept <= 1) return out;
    const DMat pk = p.cols_range(0, kept), qk = q.cols_range(0, kept);
    if (!(biorth_loss(ip_gram_host(ip, pk, qk)) > 1e-10)) return out;
    // rebiorth_pass (biorth.cpp:73-99)
    out.second_pass = true;
    for (int64_t l = 0; l < kept; ++l) {
        copy_block(p.cols_range(l, 1), pl.view());
        copy_block(q.cols_range(l, 1), ql.view());
        for (int64_t j = 0; j < l; ++j) {
            const DMat pj = p.cols_range(j, 1), qj = q.cols_range(j, 1);
            ip_dot_dev(ip, qj, pl.view(), wb, r);
            sub_scaled(pj, r, pl.view());
            ip_dot_dev(ip, pj, ql.view(), wb, s);
            sub_scaled(qj, s, ql.view());
        }
        norms_eta(pl.view(), ql.view());
        const double eta = h[2];
        if (eta == 0.0) continue;
        const double scale = 1.0 / std::sqrt(std::fabs(eta)), sgn = eta < 0.0 ? -1.0 : 1.0;
        axpby(sgn * scale, pl.view(), 0.0, p.cols_range(l, 1));
        axpby(scale, ql.view(), 0.0, q.cols_range(l, 1));
    }
    return out;
}

double dev_biorth_residual(const DMat& p, const DMat& q, const InnerProduct& ip) {
    require(p.rows == q.rows && p.cols == q.cols, "biorth_residual: shape mismatch");
    if (p.cols == 0) return 0.0;
    return biorth_loss(ip_gram_host(ip, p, q));
}

// ---------------------------------------------------------------------------------------------
// Batched multi-RHS CG
// ---------------------------------------------------------------------------------------------
namespace {
constexpr int64_t kCgUnrollMax = 32;

void drop_graphs(std::vector<CgGraph>& gs) {
    for (CgGraph& g : gs) {
        if (g.exec) cudaGraphExecDestroy(g.exec);
        if (g.graph) cudaGraphDestroy(g.graph);
    }
    gs.clear();
}
}  // namespace

void CgWorkspace::ensure(int64_t n, int64_t m) {
    if (r.rows() != n || r.capacity() < m) {
        drop_graphs(graphs);  // recorded launches point at the old buffers
        r = DBlock(n, m);
        p = DBlock(n, m);
        ap = DBlock(n, m);
    }
    r.set_cols(m);
    p.set_cols(m);
    ap.set_cols(m);
    if (m > m_cap_) {
        drop_graphs(graphs);
        Runtime& rt = Runtime::get();
        if (scal_) rt.free(scal_);
        m_cap_ = m;
        const size_t bytes = sizeof(double) * 5 * m + sizeof(int) * (3 * m + 4);
        scal_ = rt.alloc(bytes);
        double* d = static_cast<double*>(scal_);
        s.rr = d;
        s.bnorm = d + m;
        s.pap = d + 2 * m;
        s.beta = d + 3 * m;
        s.alpha = d + 4 * m;
        int* iv = reinterpret_cast<int*>(d + 5 * m);
        s.active = iv;
        s.broken = iv + m;
        s.iters = iv + 2 * m;
        s.any_active = iv + 3 * m;
        s.loops = iv + 3 * m + 1;
        m_live = iv + 3 * m + 2;
    }
    if (!parts_) {  // [pap partials | r^T r partials], 160 columns x 512 blocks each
        parts_ = static_cast<double*>(Runtime::get().alloc(sizeof(double) * 2 * kPartsPerRegion));
        ticket_ = static_cast<unsigned*>(Runtime::get().alloc(sizeof(unsigned) * 4 + sizeof(unsigned long long)));
        BOSP_CUDA(cudaMemsetAsync(ticket_, 0, sizeof(unsigned) * 4 + sizeof(unsigned long long), Runtime::get().stream()));
    }
    s.total = reinterpret_cast<unsigned long long*>(ticket_ + 4);
    s.parts = parts_ + kPartsPerRegion;
    s.parts_cap = static_cast<int>(kPartsPerRegion);
    if (!host_active) {
        BOSP_CUDA(cudaMallocHost(&host_active, 4 * sizeof(int)));
        BOSP_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        BOSP_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    }
}

int64_t CgWorkspace::total_sweeps() {
    if (!s.total) return 0;
    unsigned long long t = 0;
    BOSP_CUDA(cudaMemcpyAsync(&t, s.total, sizeof(t), cudaMemcpyDeviceToHost, Runtime::get().stream()));
    Runtime::get().sync();
    return static_cast<int64_t>(t);
}

CgWorkspace::~CgWorkspace() {
    // Every workspace (one per solve, per nullspace detection, per API CG call) returns what it
    // owns.  At process exit the CUDA runtime may already be unloading: the calls then fail
    // with cudaErrorCudartUnloading and are ignored (the driver reclaims everything).
    drop_graphs(graphs);
    Runtime& rt = Runtime::get();
    if (cudaStreamQuery(rt.stream()) == cudaErrorCudartUnloading) return;
    if (scal_) rt.free(scal_);
    if (parts_) rt.free(parts_);
    if (ticket_) rt.free(ticket_);
    if (host_active) {
        cudaStreamSynchronize(rt.stream());  // a pending publish() may still target it
        cudaFreeHost(host_active);
    }
    for (cudaEvent_t& e : ev)
        if (e) cudaEventDestroy(e);
    cudaGetLastError();  // clear any teardown error
}

namespace {
// One batched CG iteration: ap = A p with p^T A p fused into the operator when it can
// (SELL / stencil), then the cooperative fused update; unfused kernels otherwise.
// (Measured and dropped: a row-major "interleaved" CG layout, 15-20 % slower on config 2, and
// a cooperative single-kernel update with a grid barrier, slower than the 2-kernel form.)
void cg_iteration(const LinearOperator& a, const DMat& x, const DMat& r, const DMat& p, const DMat& ap,
                  const CgScalars& sc, CgWorkspace& ws, double tol, int mi) {
    if (Runtime::get().nranks() == 1) {
        // the SpMM leaves p^T A p as per-block partials; each update block folds its column
        const SpmmDot dot{ws.pap_parts(), nullptr, sc.pap, sc.active, CgWorkspace::kPartsPerRegion};
        if (const int nparts = a.impl()->apply_dot(p, ap, dot)) {
            cg_update(x, r, p, ap, sc, tol, mi, ws.pap_parts(), nparts);
            return;
        }
    }
    const SpmmDot dot{ws.pap_parts(), ws.ticket(), sc.pap, sc.active, CgWorkspace::kPartsPerRegion};
    if (a.impl()->apply_dot(p, ap, dot) > 0) {
        Runtime::get().allreduce(sc.pap, p.cols);  // per-rank p^T A p -> global
        cg_update(x, r, p, ap, sc, tol, mi);
        return;
    }
    a.apply_device(p, ap);
    cg_pap(p, ap, sc);
    cg_update(x, r, p, ap, sc, tol, mi);
}
}  // namespace

DevCgOutcome dev_cg(const LinearOperator& a, const DMat& rhs, const DMat& x, double tol,
                    int64_t max_iter, CgWorkspace& ws, const DMat* x0, bool want_stats, bool defer_sweeps) {
    require(rhs.rows == a.dim() && x.rows == a.dim() && rhs.cols == x.cols, "cg_solve: shape mismatch");
    DevCgOutcome out;
    const int64_t m = rhs.cols;
    if (m == 0) return out;
    Runtime& rt = Runtime::get();
    ws.ensure(rhs.rows, m);
    const DMat r = ws.r.view(), p = ws.p.view(), ap = ws.ap.view();
    const int mi = static_cast<int>(std::min<int64_t>(max_iter, 1 << 30));
    // one rank: the whole solve is a CUDA graph.  Several ranks: also a graph when the
    // communicator is stream-ordered (NCCL: the allreduces of p^T A p / r^T r and the halo
    // send/recv are recorded with the kernels); ThreadComm's host barriers keep the loop
    // host-driven.  A multi-rank capture that fails falls back to the host loop for good.
    // Graphs pay off where launch overhead matters (config 2: 262144 x 20); on the large blocks
    // of configs 3/5 graph and host loop measured within run-to-run noise (config 3: 14.2-19.4 s
    // vs 17.1-18.8 s over several boxes), so graphs stay the default.  BOSP_NO_GRAPHS=1 forces
    // the host loop (per-kernel ncu captures).
    static const bool no_graphs = std::getenv("BOSP_NO_GRAPHS") != nullptr;
    static std::atomic<bool> multi_capture_failed{false};
    const bool multi = rt.nranks() > 1;
    const bool comm_ok = !multi || (rt.comm()->stream_capturable() && !multi_capture_failed.load());
    CgGraph* g = nullptr;
    const bool unrolled = max_iter <= kCgUnrollMax && a.impl()->has_masked_dot();
    if (!x0 && comm_ok && a.impl()->capturable() && !no_graphs) {
        // ---- graph path: the whole solve is one launch, the loop runs on the device ----
        // Operators whose apply honours the column mask record the unrolled graph once at the
        // workspace width and serve every narrower call through the live-width scalar (the
        // solver's GS sweeps shrink 20 -> 19 -> 16 -> ... -> 1 as columns converge).
        // Recorded width: the next power of two (capped at the workspace width), so a graph
        // serves widths within 2x of its own and the kernels' grids stay sized for them
        // (recording at the full width for every call measured 8 % slower: narrow solves then
        // run on grids split for 20 columns).
        int64_t mg = m;
        if (unrolled) {
            mg = 1;
            while (mg < m) mg *= 2;
            mg = std::max<int64_t>(m, std::min<int64_t>(mg, ws.r.capacity()));
        }
        for (CgGraph& c : ws.graphs)
            if (c.op == a.impl()->uid() && c.scratch_gen == rt.scratch_generation() && c.rhs == rhs.p && c.ldr == rhs.ld && c.x == x.p && c.ldx == x.ld &&
                c.m == mg && c.tol == tol && c.max_iter == max_iter && c.prof_family == rt.prof_family())
                g = &c;
        if (!g) {
            const auto tb = std::chrono::steady_clock::now();
            if (ws.graphs.size() >= 16) drop_graphs(ws.graphs);
            ws.graphs.emplace_back();
            g = &ws.graphs.back();
            g->op = a.impl()->uid();
            g->rhs = rhs.p;
            g->ldr = rhs.ld;
            g->x = x.p;
            g->ldx = x.ld;
            g->m = mg;
            g->tol = tol;
            g->max_iter = max_iter;
            g->prof_family = rt.prof_family();
            rt.set_capture_prof(&g->prof_pairs);
            rt.scratch(1 << 16);  // no pool growth while recording
            rt.tickets(64);
            g->scratch_gen = rt.scratch_generation();
            a.impl()->reserve(unrolled ? mg : m);  // halo buffers exist before the capture
            rt.sync();
            try {
            BOSP_CUDA(cudaGraphCreate(&g->graph, 0));
            // Short solves (the solver's inner CG: max_iter 20) are unrolled into a straight
            // graph -- every kernel early-outs once its columns are done, no conditional node,
            // and every launch keeps its own profiling slot.  Long solves use a device while loop.
            if (unrolled) {
                CgScalars sc = ws.s;
                sc.has_cond = 0;
                sc.m_live = ws.m_live;
                const DMat rg = ws.r.cols(0, mg), pg = ws.p.cols(0, mg), apg = ws.ap.cols(0, mg);
                DMat rhsg = rhs, xg = x;
                rhsg.cols = xg.cols = mg;  // columns >= the live width are never touched
                rt.set_capture_sink(&g->start_launches);
                BOSP_CUDA(cudaStreamBeginCaptureToGraph(rt.stream(), g->graph, nullptr, nullptr, 0,
                                                        cudaStreamCaptureModeRelaxed));
                rt.timer_reserve(3 * max_iter + 2);  // one memset node for every timed launch below
                cg_start(rhsg, xg, rg, pg, sc, tol, mi);
                for (int64_t it = 0; it < max_iter; ++it) cg_iteration(a, xg, rg, pg, apg, sc, ws, tol, mi);
                rt.timer_reserve(0);
                BOSP_CUDA(cudaStreamEndCapture(rt.stream(), &g->graph));
            } else {
            cudaGraphConditionalHandle h;
            BOSP_CUDA(cudaGraphConditionalHandleCreate(&h, g->graph, 0, 0));
            CgScalars sc = ws.s;
            sc.cond = h;
            sc.has_cond = 1;
            // prologue: x = 0, r = p = b, norms, loop condition
            rt.set_capture_sink(&g->start_launches);
            BOSP_CUDA(cudaStreamBeginCaptureToGraph(rt.stream(), g->graph, nullptr, nullptr, 0,
                                                    cudaStreamCaptureModeRelaxed));
            cg_start(rhs, x, r, p, sc, tol, mi);
            BOSP_CUDA(cudaStreamEndCapture(rt.stream(), &g->graph));
            size_t nn = 0;
            BOSP_CUDA(cudaGraphGetNodes(g->graph, nullptr, &nn));
            std::vector<cudaGraphNode_t> deps(nn);
            BOSP_CUDA(cudaGraphGetNodes(g->graph, deps.data(), &nn));
            cudaGraphNodeParams cp{};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t cnode;
            BOSP_CUDA(cudaGraphAddNode(&cnode, g->graph, deps.data(), nn, &cp));
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            rt.set_capture_sink(&g->body_launches);
            BOSP_CUDA(cudaStreamBeginCaptureToGraph(rt.stream(), body, nullptr, nullptr, 0,
                                                    cudaStreamCaptureModeRelaxed));
            cg_iteration(a, x, r, p, ap, sc, ws, tol, mi);
            BOSP_CUDA(cudaStreamEndCapture(rt.stream(), &body));
            }
            rt.set_capture_sink(nullptr);
            rt.set_capture_prof(nullptr);
            BOSP_CUDA(cudaGraphInstantiate(&g->exec, g->graph, 0));
            } catch (const std::exception& e) {
                // end the (invalidated) capture, drop the half-built graph; one rank re-throws,
                // several ranks run the host loop from now on
                cudaGraph_t tmp = nullptr;
                cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                if (cudaStreamIsCapturing(rt.stream(), &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone)
                    cudaStreamEndCapture(rt.stream(), &tmp);
                if (tmp) cudaGraphDestroy(tmp);
                cudaGetLastError();
                rt.set_capture_sink(nullptr);
                rt.set_capture_prof(nullptr);
                rt.timer_reserve(0);
                if (g->graph) cudaGraphDestroy(g->graph);
                ws.graphs.pop_back();
                g = nullptr;
                if (!multi) throw;
                multi_capture_failed.store(true);
                std::fprintf(stderr, "[bosp] cg graph capture over %d ranks failed (%s): host loop\n", rt.nranks(), e.what());
            }
            if (g) {
            rt.graph_builds_ += 1;
            rt.graph_build_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - tb).count();
            if (std::getenv("BOSP_SYNC_STATS"))
                std::fprintf(stderr, "[bosp] cg graph: op %p rhs %p x %p m %lld tol %g max_iter %lld (cache %zu)\n",
                             (const void*)a.impl(), (const void*)rhs.p, (const void*)x.p, (long long)m, tol,
                             (long long)max_iter, ws.graphs.size());
            }
        }
    }
    if (g) {
        if (unrolled) set_device_int(ws.m_live, static_cast<int>(m));
        BOSP_CUDA(cudaGraphLaunch(g->exec, rt.stream()));
        if (defer_sweeps && g->body_launches.empty() && g->prof_pairs.empty() && !want_stats) {
            // unrolled graph: every launch is known, the sweep count lands in ws.s.total
            rt.add_launches(g->start_launches, 1);
            out.sweeps = -1;
            return out;
        }
        BOSP_CUDA(cudaMemcpyAsync(&ws.host_active[2], ws.s.loops, sizeof(int), cudaMemcpyDeviceToHost, rt.stream()));
        rt.sync();
        out.sweeps = ws.host_active[2];
        // timer slots recorded in the graph: every launch of an unrolled graph, the last
        // iteration of a while body
        if (!g->prof_pairs.empty() && out.sweeps > 0) rt.add_prof_samples(g->prof_pairs);
        rt.add_launches(g->start_launches, 1);
        rt.add_launches(g->body_launches, out.sweeps);
    } else {
        // ---- host-driven loop (host callbacks, x0 != 0, or per-kernel profiling) ----
        if (x0) {
            a.apply_device(*x0, ap);
            cg_start_x0(rhs, *x0, ap, x, r, p, ws.s, tol, mi);
        } else {
            cg_start(rhs, x, r, p, ws.s, tol, mi);
        }
        // State s (s = 0 after start, s = it+1 after iteration it) publishes its active-column
        // count to pinned slot s % 2.  Before issuing iteration it the host looks at state it-1,
        // which the device has finished while it works on iteration it-1: no stall, and at most
        // one fully masked iteration is ever issued.
        auto publish = [&](int64_t state) {
            const int slot = static_cast<int>(state & 1);
            BOSP_CUDA(cudaMemcpyAsync(&ws.host_active[slot], ws.s.any_active, sizeof(int),
                                      cudaMemcpyDeviceToHost, rt.stream()));
            BOSP_CUDA(cudaEventRecord(ws.ev[slot], rt.stream()));
        };
        publish(0);
        int64_t it = 0;
        for (; it < max_iter; ++it) {
            if (it >= 1) {
                const int slot = static_cast<int>((it - 1) & 1);
                BOSP_CUDA(cudaEventSynchronize(ws.ev[slot]));
                if (ws.host_active[slot] == 0) break;
            }
            cg_iteration(a, x, r, p, ap, ws.s, ws, tol, mi);
            publish(it + 1);
        }
        out.sweeps = it;
    }
    if (want_stats) {
        std::vector<int> broken(static_cast<size_t>(m)), iters(static_cast<size_t>(m));
        BOSP_CUDA(cudaMemcpyAsync(broken.data(), ws.s.broken, sizeof(int) * m, cudaMemcpyDeviceToHost, rt.stream()));
        BOSP_CUDA(cudaMemcpyAsync(iters.data(), ws.s.iters, sizeof(int) * m, cudaMemcpyDeviceToHost, rt.stream()));
        rt.sync();
        for (int64_t j = 0; j < m; ++j) {
            out.breakdown |= broken[j] != 0;
            out.max_iterations_used = std::max<int64_t>(out.max_iterations_used, iters[j]);
        }
    }
    return out;
}

}  // namespace b200
}  // namespace bosp
