// Host small dense algebra for the projected LREP and the coefficient-space MGS-Biorth.
#include "small_dense.hpp"

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <numeric>
#include <thread>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace bosp {
inline namespace b200 {

DenseMatrix DenseMatrix::identity(int64_t n) {
    DenseMatrix a(n, n);
    for (int64_t i = 0; i < n; ++i) a(i, i) = 1.0;
    return a;
}

DenseMatrix DenseMatrix::diagonal(const std::vector<double>& d) {
    DenseMatrix a(static_cast<int64_t>(d.size()), static_cast<int64_t>(d.size()));
    for (size_t i = 0; i < d.size(); ++i) a(i, i) = d[i];
    return a;
}

DenseMatrix DenseMatrix::transposed() const {
    DenseMatrix t(cols_, rows_);
    for (int64_t j = 0; j < cols_; ++j)
        for (int64_t i = 0; i < rows_; ++i) t(j, i) = (*this)(i, j);
    return t;
}

DenseMatrix DenseMatrix::symmetrized() const {
    require(rows_ == cols_, "symmetrized: matrix is not square");
    DenseMatrix s(rows_, cols_);
    for (int64_t j = 0; j < cols_; ++j)
        for (int64_t i = 0; i < rows_; ++i) s(i, j) = 0.5 * ((*this)(i, j) + (*this)(j, i));
    return s;
}

void DenseMatrix::mirror_lower() {
    require(rows_ == cols_, "mirror_lower: matrix is not square");
    for (int64_t j = 0; j < cols_; ++j)
        for (int64_t i = j + 1; i < rows_; ++i) (*this)(j, i) = (*this)(i, j);
}

double DenseMatrix::max_abs() const {
    double m = 0.0;
    for (double v : data_) m = std::max(m, std::fabs(v));
    return m;
}

double DenseMatrix::frobenius_norm() const {
    double s = 0.0;
    for (double v : data_) s += v * v;
    return std::sqrt(s);
}

bool DenseMatrix::is_symmetric(double tol_rel) const {
    if (rows_ != cols_) return false;
    const double scale = max_abs();
    for (int64_t j = 0; j < cols_; ++j)
        for (int64_t i = j + 1; i < rows_; ++i)
            if (std::fabs((*this)(i, j) - (*this)(j, i)) > tol_rel * scale) return false;
    return true;
}

namespace {
// AVX2 helpers for the rotation kernels (x86-64-v3 build).
// i0 (a multiple of 8) skips leading products known to be exactly zero without changing the
// lane assignment: bitwise the full-range sum (up to the sign of an exact-zero result).
inline double dot_avx(const double* a, const double* b, int64_t m, int64_t i0 = 0) {
    __m256d s0 = _mm256_setzero_pd(), s1 = _mm256_setzero_pd();
    int64_t i = i0;
    for (; i + 8 <= m; i += 8) {
        s0 = _mm256_fmadd_pd(_mm256_loadu_pd(a + i), _mm256_loadu_pd(b + i), s0);
        s1 = _mm256_fmadd_pd(_mm256_loadu_pd(a + i + 4), _mm256_loadu_pd(b + i + 4), s1);
    }
    for (; i + 4 <= m; i += 4) s0 = _mm256_fmadd_pd(_mm256_loadu_pd(a + i), _mm256_loadu_pd(b + i), s0);
    s0 = _mm256_add_pd(s0, s1);
    alignas(32) double t[4];
    _mm256_store_pd(t, s0);
    double r = (t[0] + t[1]) + (t[2] + t[3]);
    for (; i < m; ++i) r += a[i] * b[i];
    return r;
}

inline void rotate_avx(double* x, double* y, int64_t m, double c, double s) {
    const __m256d vc = _mm256_set1_pd(c), vs = _mm256_set1_pd(s);
    int64_t i = 0;
    for (; i + 4 <= m; i += 4) {
        const __m256d a = _mm256_loadu_pd(x + i), b = _mm256_loadu_pd(y + i);
        _mm256_storeu_pd(x + i, _mm256_fmsub_pd(vc, a, _mm256_mul_pd(vs, b)));
        _mm256_storeu_pd(y + i, _mm256_fmadd_pd(vs, a, _mm256_mul_pd(vc, b)));
    }
    for (; i < m; ++i) {
        const double a = x[i], b = y[i];
        x[i] = c * a - s * b;
        y[i] = s * a + c * b;
    }
}

}  // namespace

DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b, bool a_lower) {
    require(a.cols() == b.rows(), "matmul: inner dimensions disagree");
    DenseMatrix c(a.rows(), b.cols());
    const int64_t m = a.rows(), k = a.cols();
#pragma omp parallel for schedule(static) if (m * k * b.cols() > (int64_t(1) << 21))
    for (int64_t j = 0; j < b.cols(); ++j) {
        double* cj = c.col(j);
        for (int64_t p = 0; p < k; ++p) {
            const double bpj = b(p, j);
            if (bpj == 0.0) continue;
            const double* ap = a.col(p);
            for (int64_t i = a_lower ? p : 0; i < m; ++i) cj[i] += ap[i] * bpj;
        }
    }
    return c;
}

DenseMatrix matmul_tn_lower(const DenseMatrix& l, const DenseMatrix& r) {
    require(l.rows() == r.rows() && l.rows() == l.cols() && r.rows() == r.cols(), "matmul_tn_lower: square factors");
    const int64_t n = l.rows();
    DenseMatrix c(n, n);
    // (L^T R)(i, j) = sum_{p >= max(i, j)} L(p, i) R(p, j): the structural zeros are skipped
    // (bitwise matmul_tn: same lanes, only exact-zero products left out)
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t j = 0; j < n; ++j) {
        const double* rj = r.col(j);
        for (int64_t i = 0; i < n; ++i) {
            const int64_t p0 = std::max(i, j) & ~int64_t(7);
            c(i, j) = dot_avx(l.col(i), rj, n, p0);
        }
    }
    return c;
}

DenseMatrix matmul_tn(const DenseMatrix& a, const DenseMatrix& b) {
    require(a.rows() == b.rows(), "matmul_tn: row dimensions disagree");
    DenseMatrix c(a.cols(), b.cols());
    const int64_t m = a.rows();
#pragma omp parallel for schedule(static) if (m * a.cols() * b.cols() > (int64_t(1) << 21))
    for (int64_t j = 0; j < b.cols(); ++j) {
        const double* bj = b.col(j);
        for (int64_t i = 0; i < a.cols(); ++i) c(i, j) = dot_avx(a.col(i), bj, m);
    }
    return c;
}

std::optional<DenseMatrix> cholesky_lower(const DenseMatrix& a) {
    if (a.rows() != a.cols()) return std::nullopt;
    const int64_t n = a.rows();
    DenseMatrix l(n, n);
    // Left-looking, column-oriented: column j = (a(:, j) - sum_k l(j,k) l(:, k)) / l_jj with the
    // k-sum accumulated in the reference's order (dense_kernels.cpp:11-28) but as unit-stride
    // axpys; the diagonal pivot test (d > 0, finite) is the contract.
    std::vector<double> s(static_cast<size_t>(n));
    for (int64_t j = 0; j < n; ++j) {
        for (int64_t i = j; i < n; ++i) s[i] = a(i, j);
        // four k at a time with each element's subtractions still in ascending k (bitwise the
        // one-k-at-a-time loop; s is loaded and stored once per four columns of L)
        int64_t k = 0;
        for (; k + 4 <= j; k += 4) {
            const double c0 = l(j, k), c1 = l(j, k + 1), c2 = l(j, k + 2), c3 = l(j, k + 3);
            const double *l0 = l.col(k), *l1 = l.col(k + 1), *l2 = l.col(k + 2), *l3 = l.col(k + 3);
            for (int64_t i = j; i < n; ++i) {
                double v = s[i];
                v -= l0[i] * c0;
                v -= l1[i] * c1;
                v -= l2[i] * c2;
                v -= l3[i] * c3;
                s[i] = v;
            }
        }
        for (; k < j; ++k) {
            const double ljk = l(j, k);
            const double* lk = l.col(k);
            for (int64_t i = j; i < n; ++i) s[i] -= lk[i] * ljk;
        }
        const double d = s[j];
        if (!(d > 0.0) || !std::isfinite(d)) return std::nullopt;
        const double ljj = std::sqrt(d);
        double* lj = l.col(j);
        lj[j] = ljj;
        for (int64_t i = j + 1; i < n; ++i) lj[i] = s[i] / ljj;
    }
    return l;
}

void cholesky_lower_pair(const DenseMatrix& a, const DenseMatrix& b, std::optional<DenseMatrix>& la,
                         std::optional<DenseMatrix>& lb) {
    // the two factorizations on two threads (a barrier-per-column parallel factorization lost
    // to barrier latency at d = 320)
#pragma omp parallel sections num_threads(2) if (a.rows() >= 64)
    {
#pragma omp section
        la = cholesky_lower(a);
#pragma omp section
        lb = cholesky_lower(b);
    }
}

namespace {

// Rotate columns p, q of a (m rows) and v (k rows) if they are not yet orthogonal; returns
// whether a rotation happened.  Rotation formula and test of dense_kernels.cpp:47-79.  The
// squared column norms are carried in `nrm` (recomputed at every sweep start): after the
// rotation that annihilates gamma they are exactly alpha - t*gamma and beta + t*gamma, so a pair
// costs one dot product instead of three.
inline bool jacobi_pair(DenseMatrix& a, DenseMatrix* v, double* nrm, int64_t p, int64_t q, double tol = 1e-15) {
    const int64_t m = a.rows();
    double* ap = a.col(p);
    double* aq = a.col(q);
    double& np = nrm[p];
    double& nq = nrm[q];
    const double alpha = np, beta = nq;
    if (alpha == 0.0 || beta == 0.0) return false;
    const double gamma = dot_avx(ap, aq, m);
    if (std::fabs(gamma) <= tol * std::sqrt(alpha * beta)) return false;
    const double zeta = (beta - alpha) / (2.0 * gamma);
    const double t = ((zeta >= 0.0) ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
    const double c = 1.0 / std::sqrt(1.0 + t * t);
    const double s = c * t;
    rotate_avx(ap, aq, m, c, s);
    if (v) rotate_avx(v->col(p), v->col(q), v->rows(), c, s);
    np = alpha - t * gamma;
    nq = beta + t * gamma;
    return true;
}

void column_norms(const DenseMatrix& a, double* nrm) {
    for (int64_t j = 0; j < a.cols(); ++j) nrm[j] = dot_avx(a.col(j), a.col(j), a.rows());
}

}  // namespace

JacobiSvdResult jacobi_svd(DenseMatrix a, int64_t max_sweeps) { return jacobi_svd_tol(std::move(a), max_sweeps, 1e-15); }

JacobiSvdResult jacobi_svd_tol(DenseMatrix a, int64_t max_sweeps, double tol, bool accumulate) {
    const int64_t m = a.rows(), k = a.cols();
    require(m >= k, "jacobi_svd: requires rows >= cols");
    JacobiSvdResult res;
    if (accumulate) res.v = DenseMatrix::identity(k);
    DenseMatrix* vp = accumulate ? &res.v : nullptr;
    bool rotated = true;
    int64_t sweep = 0;
    if (k < 96) {
        // cyclic-by-row order, exactly the reference's sweep
        std::vector<double> nrm(static_cast<size_t>(k));
        while (rotated && sweep < max_sweeps) {
            rotated = false;
            ++sweep;
            column_norms(a, nrm.data());
            for (int64_t p = 0; p + 1 < k; ++p)
                for (int64_t q = p + 1; q < k; ++q) rotated |= jacobi_pair(a, vp, nrm.data(), p, q, tol);
        }
    } else {
        // Block round-robin: the columns are cut into nblk blocks (2 per thread) and every round
        // of a block tournament gives each thread one disjoint block pair (I, J), whose column
        // pairs it rotates in cyclic order (cross pairs p in I, q in J; in a sweep's first round
        // also the pairs inside I and inside J), so every column pair is visited once per sweep
        // as in the cyclic sweep.  nblk - 1 barriers per sweep instead of k - 1 (the per-column
        // tournament spent as long in barriers as in rotations at d = 320).
        const int nthr = std::max(1, omp_get_max_threads());
        int64_t nblk = std::min<int64_t>(2 * nthr, k / 4);
        nblk += nblk & 1;
        const int64_t bs = (k + nblk - 1) / nblk;
        nblk = (k + bs - 1) / bs;
        nblk += nblk & 1;  // a trailing empty block when odd (a bye in the tournament)
        auto blk_lo = [&](int64_t b) { return std::min(k, b * bs); };
        auto blk_hi = [&](int64_t b) { return std::min(k, (b + 1) * bs); };
        std::vector<int64_t> pos(static_cast<size_t>(nblk));
        std::iota(pos.begin(), pos.end(), 0);
        std::vector<double> nrm(static_cast<size_t>(k));
        // Pairs whose columns are unchanged since they last passed the orthogonality test are
        // skipped: the test would recompute the same dot product from the same data (and the
        // same norms: nrm is recomputed from the columns every sweep) and reach the same "no
        // rotation" -- decision-exact, and most of the late sweeps' dot products disappear.
        std::vector<uint32_t> ver(static_cast<size_t>(k), 0u);
        std::vector<uint64_t> seen(static_cast<size_t>(k * k), ~uint64_t(0));
        auto pair = [&](int64_t p, int64_t q) -> int {
            const uint64_t key = (static_cast<uint64_t>(ver[p]) << 32) | ver[q];
            uint64_t& sk = seen[p * k + q];
            if (sk == key) return 0;
            if (jacobi_pair(a, vp, nrm.data(), p, q, tol)) {
                ++ver[p];
                ++ver[q];
                return 1;
            }
            sk = key;
            return 0;
        };
        // Rounds are ordered per block, not by a barrier: a block pair of round r starts as soon
        // as both of its blocks have finished round r - 1 (acquire/release round counters), so a
        // thread whose pairs were skipped (late sweeps) runs ahead instead of waiting for the
        // slowest thread of every round.  Pair i of every round belongs to thread i mod T.
        // (config 3 on one box: host small solve 0.727 s with an omp-for barrier per round,
        // 0.656 s with the counters; 0.765 s before this round's Cholesky / back-transform work.)
        std::unique_ptr<std::atomic<int64_t>[]> done(new std::atomic<int64_t>[static_cast<size_t>(nblk)]);
        while (rotated && sweep < max_sweeps) {
            ++sweep;
            int any = 0;
            column_norms(a, nrm.data());
            for (int64_t b = 0; b < nblk; ++b) done[b].store(0, std::memory_order_relaxed);
#pragma omp parallel reduction(+ : any)
            {
                const int nt = omp_get_num_threads(), t = omp_get_thread_num();
                std::vector<int64_t> lp(pos);
                for (int64_t round = 0; round < nblk - 1; ++round) {
                    for (int64_t i = t; i < nblk / 2; i += nt) {
                        int64_t bi = lp[i], bj = lp[nblk - 1 - i];
                        if (bi > bj) std::swap(bi, bj);
                        // spin, yielding now and then (ranks as host threads can oversubscribe)
                        for (int spin = 1; done[bi].load(std::memory_order_acquire) < round ||
                                           done[bj].load(std::memory_order_acquire) < round;
                             ++spin)
                            if (spin % 1024 == 0) std::this_thread::yield(); else _mm_pause();
                        const int64_t i0 = blk_lo(bi), i1 = blk_hi(bi), j0 = blk_lo(bj), j1 = blk_hi(bj);
                        if (round == 0) {
                            for (int64_t p = i0; p + 1 < i1; ++p)
                                for (int64_t q = p + 1; q < i1; ++q) any += pair(p, q);
                            for (int64_t p = j0; p + 1 < j1; ++p)
                                for (int64_t q = p + 1; q < j1; ++q) any += pair(p, q);
                        }
                        for (int64_t p = i0; p < i1; ++p)
                            for (int64_t q = j0; q < j1; ++q) any += pair(p, q);
                        done[bi].store(round + 1, std::memory_order_release);
                        done[bj].store(round + 1, std::memory_order_release);
                    }
                    const int64_t last = lp[nblk - 1];
                    for (int64_t i = nblk - 1; i > 1; --i) lp[i] = lp[i - 1];
                    lp[1] = last;
                }
#pragma omp barrier
#pragma omp single
                pos = lp;
            }
            rotated = (any != 0);
            if (std::getenv("BOSP_DEBUG_SWEEPS")) std::fprintf(stderr, "[bosp] jacobi sweep %lld rotations %d\n", (long long)sweep, any);
        }
    }
    res.converged = !rotated;
    res.sweeps = sweep;
    std::vector<double> sig(static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j) {
        double s = 0.0;
        const double* aj = a.col(j);
        for (int64_t i = 0; i < m; ++i) s += aj[i] * aj[i];
        sig[j] = std::sqrt(s);
    }
    std::vector<int64_t> order(static_cast<size_t>(k));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t i, int64_t j) { return sig[i] < sig[j]; });
    res.u = DenseMatrix(m, k);
    res.sigma.resize(static_cast<size_t>(k));
    DenseMatrix vs(accumulate ? k : 0, accumulate ? k : 0);
    for (int64_t j = 0; j < k; ++j) {
        const int64_t src = order[j];
        res.sigma[j] = sig[src];
        const double inv = sig[src] > 0.0 ? 1.0 / sig[src] : 0.0;
        for (int64_t i = 0; i < m; ++i) res.u(i, j) = a(i, src) * inv;
        if (accumulate)
            for (int64_t i = 0; i < k; ++i) vs(i, j) = res.v(i, src);
    }
    res.v = std::move(vs);
    return res;
}

namespace {

// Householder QR with column pivoting, W P = Q R (LAPACK dgeqp2 semantics: largest remaining
// column norm first, norms downdated with the cancellation guard of dlaqp2).  On return `a`
// holds R on and above the diagonal and the reflectors' tails below; tau / perm as in dgeqp2.
void householder_qrcp(DenseMatrix& a, std::vector<double>& tau, std::vector<int64_t>& perm, bool pivot = true) {
    const int64_t m = a.rows(), k = a.cols();
    tau.assign(static_cast<size_t>(k), 0.0);
    perm.resize(static_cast<size_t>(k));
    std::iota(perm.begin(), perm.end(), 0);
    std::vector<double> vn1(static_cast<size_t>(k)), vn2(static_cast<size_t>(k));
    for (int64_t j = 0; j < k; ++j) vn1[j] = vn2[j] = std::sqrt(dot_avx(a.col(j), a.col(j), m));
    const double tol3z = std::sqrt(std::numeric_limits<double>::epsilon());
    for (int64_t j = 0; j < k && j < m; ++j) {
        const int64_t pvt = pivot ? j + (std::max_element(vn1.begin() + j, vn1.end()) - (vn1.begin() + j)) : j;
        if (pvt != j) {
            std::swap_ranges(a.col(pvt), a.col(pvt) + m, a.col(j));
            std::swap(perm[pvt], perm[j]);
            vn1[pvt] = vn1[j];
            vn2[pvt] = vn2[j];
        }
        double* v = a.col(j) + j;  // v = [1; a(j+1:m, j)] after scaling
        const int64_t len = m - j;
        const double alpha = v[0];
        const double xnorm = len > 1 ? std::sqrt(dot_avx(v + 1, v + 1, len - 1)) : 0.0;
        double t = 0.0;
        if (xnorm != 0.0) {
            const double beta = -std::copysign(std::hypot(alpha, xnorm), alpha);
            t = (beta - alpha) / beta;
            const double sc = 1.0 / (alpha - beta);
            for (int64_t i = 1; i < len; ++i) v[i] *= sc;
            v[0] = beta;
        }
        tau[j] = t;
        if (t != 0.0) {
#pragma omp parallel for schedule(static) if ((k - j) * len > 16384)
            for (int64_t c = j + 1; c < k; ++c) {
                double* ac = a.col(c) + j;
                const double w = t * (ac[0] + (len > 1 ? dot_avx(v + 1, ac + 1, len - 1) : 0.0));
                ac[0] -= w;
                for (int64_t i = 1; i < len; ++i) ac[i] -= w * v[i];
            }
        }
        for (int64_t c = j + 1; c < k; ++c) {
            if (vn1[c] == 0.0) continue;
            double temp = std::fabs(a(j, c)) / vn1[c];
            temp = std::max(0.0, 1.0 - temp * temp);
            const double r = vn1[c] / vn2[c];
            if (temp * r * r <= tol3z) {
                const int64_t rest = m - j - 1;
                vn1[c] = rest > 0 ? std::sqrt(dot_avx(a.col(c) + j + 1, a.col(c) + j + 1, rest)) : 0.0;
                vn2[c] = vn1[c];
            } else {
                vn1[c] *= std::sqrt(temp);
            }
        }
    }
}

// b <- Q b for Q = H_0 H_1 ... H_{k-1} (reflectors below the diagonal of `a`, dgeqp2 layout);
// the columns of b are independent.
void apply_q(const DenseMatrix& a, const std::vector<double>& tau, DenseMatrix& b) {
    const int64_t m = a.rows(), k = static_cast<int64_t>(tau.size());
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < b.cols(); ++c) {
        double* bc = b.col(c);
        for (int64_t j = k - 1; j >= 0; --j) {
            if (tau[j] == 0.0) continue;
            const double* v = a.col(j) + j;
            const int64_t len = m - j;
            double s = bc[j];
            for (int64_t i = 1; i < len; ++i) s += v[i] * bc[j + i];
            s *= tau[j];
            bc[j] -= s;
            for (int64_t i = 1; i < len; ++i) bc[j + i] -= s * v[i];
        }
    }
}

}  // namespace

// One-sided Jacobi SVD with QR preconditioning (Drmac & Veselic): W P = Q R, then the same
// one-sided Jacobi (rotation formula, 1e-15 test, sweep cap) on X = R^T, whose columns are
// graded and nearly orthogonal -- a few sweeps instead of ~15 at d = 320.  X V_x = U_x S gives
// W = (Q V_x) S (P U_x)^T.  Same outputs as jacobi_svd (sigma ascending, u, v), restricted to the
// first `nvec` (smallest) singular vectors when 0 <= nvec < k (Q applied to those only).
//
// Measured and not kept: skipping the accumulation of V_x (half the work per rotation) and
// solving R^T v_j = sigma_j u_j for the wanted columns instead -- accurate to ~kappa(R~) eps
// (max |V_x^T V_x - I| = 1.5e-13 at d = 320, vs ~1e-15 accumulated) and 2.5 ms faster per call,
// but that perturbation moved the SPEC-6 moving-off solve (n = 1000, d = 420, stopped at
// max_outer_iter) from 299 to 297 converged pairs.
JacobiSvdResult jacobi_svd_qr(const DenseMatrix& w, int64_t max_sweeps, int64_t nvec) {
    const int64_t m = w.rows(), k = w.cols();
    require(m == k, "jacobi_svd_qr: square input expected");
    if (nvec < 0 || nvec > k) nvec = k;
    static const bool dbg = std::getenv("BOSP_DEBUG") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    DenseMatrix a = w;
    std::vector<double> tau;
    std::vector<int64_t> perm;
    householder_qrcp(a, tau, perm);
    const auto t1 = std::chrono::steady_clock::now();
    DenseMatrix x(k, k);  // X = R^T (lower triangular)
    for (int64_t j = 0; j < k; ++j)
        for (int64_t i = j; i < k; ++i) x(i, j) = a(j, i);
    JacobiSvdResult jx = jacobi_svd_tol(std::move(x), max_sweeps, 1e-15);
    const auto t2 = std::chrono::steady_clock::now();
    // left vectors of W: Q V_x, Q = H_0 H_1 ... H_{k-1} applied to V_x's wanted columns
    DenseMatrix u(k, nvec);
    for (int64_t c = 0; c < nvec; ++c) std::copy(jx.v.col(c), jx.v.col(c) + k, u.col(c));
    apply_q(a, tau, u);
    if (dbg) {
        auto ms = [](auto x0, auto x1) { return std::chrono::duration<double>(x1 - x0).count() * 1e3; };
        std::fprintf(stderr, "[bosp] svd_qr d=%lld nvec=%lld qrcp %.2f ms jacobi %.2f ms (%lld sweeps) apply_q %.2f ms\n",
                     (long long)k, (long long)nvec, ms(t0, t1), ms(t1, t2), (long long)jx.sweeps,
                     ms(t2, std::chrono::steady_clock::now()));
    }
    // right vectors of W: P U_x (row perm[i] of the result is row i of U_x)
    JacobiSvdResult res;
    res.sigma = std::move(jx.sigma);
    res.converged = jx.converged;
    res.sweeps = jx.sweeps;
    res.v = DenseMatrix(k, nvec);
    for (int64_t j = 0; j < nvec; ++j)
        for (int64_t i = 0; i < k; ++i) res.v(perm[i], j) = jx.u(i, j);
    res.u = std::move(u);
    return res;
}

double spectral_norm(const DenseMatrix& a) {
    if (a.rows() == 0 || a.cols() == 0) return 0.0;
    auto svd = a.rows() >= a.cols() ? jacobi_svd(a) : jacobi_svd(a.transposed());
    return svd.sigma.back();
}

DenseMatrix lu_inverse(const DenseMatrix& a0) {
    require(a0.rows() == a0.cols(), "lu_inverse: matrix not square");
    const int64_t n = a0.rows();
    DenseMatrix a = a0;
    std::vector<int64_t> perm(static_cast<size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    for (int64_t k = 0; k < n; ++k) {
        int64_t piv = k;
        for (int64_t i = k + 1; i < n; ++i)
            if (std::fabs(a(i, k)) > std::fabs(a(piv, k))) piv = i;
        if (a(piv, k) == 0.0) throw ContractViolation("lu_factor: singular matrix");
        if (piv != k) {
            for (int64_t j = 0; j < n; ++j) std::swap(a(k, j), a(piv, j));
            std::swap(perm[k], perm[piv]);
        }
        for (int64_t i = k + 1; i < n; ++i) {
            const double l = a(i, k) / a(k, k);
            a(i, k) = l;
            for (int64_t j = k + 1; j < n; ++j) a(i, j) -= l * a(k, j);
        }
    }
    DenseMatrix inv(n, n);
    std::vector<double> x(static_cast<size_t>(n));
    for (int64_t c = 0; c < n; ++c) {
        for (int64_t i = 0; i < n; ++i) x[i] = (perm[i] == c) ? 1.0 : 0.0;
        for (int64_t i = 1; i < n; ++i)
            for (int64_t j = 0; j < i; ++j) x[i] -= a(i, j) * x[j];
        for (int64_t i = n - 1; i >= 0; --i) {
            for (int64_t j = i + 1; j < n; ++j) x[i] -= a(i, j) * x[j];
            x[i] /= a(i, i);
        }
        for (int64_t i = 0; i < n; ++i) inv(i, c) = x[i];
    }
    return inv;
}

ProjectedLrep finish_assembly(const DenseMatrix& khat, const DenseMatrix& mhat) {
    static const bool dbg = std::getenv("BOSP_DEBUG") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    ProjectedLrep p;
    p.d = khat.rows();
    p.khat = khat.symmetrized();
    p.mhat = mhat.symmetrized();
    std::optional<DenseMatrix> lk, lm;
    cholesky_lower_pair(p.khat, p.mhat, lk, lm);
    if (!lk) throw NullspaceLeak("assemble_projected: U^T K U is not SPD");
    if (!lm) throw NullspaceLeak("assemble_projected: V^T M V is not SPD");
    p.chol_k = std::move(*lk);
    p.chol_m = std::move(*lm);
    if (dbg)
        std::fprintf(stderr, "[bosp] finish_assembly d=%lld %.2f ms\n", (long long)p.d,
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3);
    return p;
}

SmallEigenSolution solve_small_lrep(const ProjectedLrep& p, int64_t k) {
    require(k <= p.d, "solve_small_lrep: k exceeds d");
    require(p.chol_k.rows() == p.d && p.chol_m.rows() == p.d, "solve_small_lrep: missing Cholesky factors");
    const DenseMatrix& l = p.chol_k;
    const DenseMatrix& r = p.chol_m;
    // d >= 96 (configs 3/5: d = 320): QR-preconditioned Jacobi, a few sweeps instead of ~15
    static const bool dbg = std::getenv("BOSP_DEBUG") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    JacobiSvdResult svd = p.d >= 96 ? jacobi_svd_qr(matmul_tn_lower(l, r), 40, k) : jacobi_svd(matmul_tn(l, r));
    if (dbg)
        std::fprintf(stderr, "[bosp] small svd d=%lld sweeps=%lld %.2f ms\n", (long long)p.d, (long long)svd.sweeps,
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() * 1e3);
    const double smax = svd.sigma.empty() ? 0.0 : svd.sigma.back();
    for (double s : svd.sigma)
        if (s < 1e-14 * smax)
            throw DegenerateSpectrum("solve_small_lrep: singular value at round-off scale, "
                                     "a near-zero eigenvalue escaped deflation");
    const auto t1 = std::chrono::steady_clock::now();
    SmallEigenSolution sol;
    sol.lambdas.assign(svd.sigma.begin(), svd.sigma.begin() + k);
    DenseMatrix phi(p.d, k), psi(p.d, k);
    for (int64_t j = 0; j < k; ++j) {
        const double w = 1.0 / std::sqrt(svd.sigma[j]);
        for (int64_t i = 0; i < p.d; ++i) {
            phi(i, j) = svd.u(i, j) * w;
            psi(i, j) = svd.v(i, j) * w;
        }
    }
    sol.yhat = matmul(l, phi, true);  // L, R lower triangular
    sol.xhat = matmul(r, psi, true);
    if (dbg)
        std::fprintf(stderr, "[bosp] small back-transform %.2f ms\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count() * 1e3);
    return sol;
}

namespace {

inline double dotn(const double* a, const double* b, int64_t n) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}
inline void axpyn(double alpha, const double* x, double* y, int64_t n) {
    for (int64_t i = 0; i < n; ++i) y[i] += alpha * x[i];
}
inline double sign_or_plus(double v) { return v < 0.0 ? -1.0 : 1.0; }

HostBiorth host_gs(const DenseMatrix& x, const DenseMatrix& y, double drop_tol, bool classical) {
    require(x.rows() == y.rows() && x.cols() == y.cols(), "biorth: X and Y must have equal shape");
    const int64_t n = x.rows(), m = x.cols();
    DenseMatrix p(n, m), q(n, m);
    HostBiorth out;
    std::vector<double> pl(static_cast<size_t>(n)), ql(static_cast<size_t>(n));
    for (int64_t l = 0; l < m; ++l) {
        std::copy(x.col(l), x.col(l) + n, pl.begin());
        std::copy(y.col(l), y.col(l) + n, ql.begin());
        for (size_t t = 0; t < out.kept.size(); ++t) {
            const double r = classical ? dotn(q.col(t), x.col(l), n) : dotn(q.col(t), pl.data(), n);
            axpyn(-r, p.col(t), pl.data(), n);
            const double s = classical ? dotn(p.col(t), y.col(l), n) : dotn(p.col(t), ql.data(), n);
            axpyn(-s, q.col(t), ql.data(), n);
        }
        const double pn = std::sqrt(std::max(0.0, dotn(pl.data(), pl.data(), n)));
        const double qn = std::sqrt(std::max(0.0, dotn(ql.data(), ql.data(), n)));
        const double eta = dotn(pl.data(), ql.data(), n);
        if (pn == 0.0 || qn == 0.0 || std::fabs(eta) < drop_tol * pn * qn) {
            out.dropped.push_back(l);
            continue;
        }
        const double sc = 1.0 / std::sqrt(std::fabs(eta)), sg = sign_or_plus(eta);
        const int64_t kc = static_cast<int64_t>(out.kept.size());
        for (int64_t i = 0; i < n; ++i) {
            p(i, kc) = sg * pl[i] * sc;
            q(i, kc) = ql[i] * sc;
        }
        out.kept.push_back(l);
    }
    const int64_t k = static_cast<int64_t>(out.kept.size());
    out.p = DenseMatrix(n, k);
    out.q = DenseMatrix(n, k);
    std::copy(p.data(), p.data() + n * k, out.p.data());
    std::copy(q.data(), q.data() + n * k, out.q.data());
    return out;
}

}  // namespace

double biorth_loss(const DenseMatrix& g) {
    DenseMatrix d = g;
    for (int64_t i = 0; i < d.rows(); ++i) d(i, i) -= 1.0;
    return spectral_norm(d);
}

bool biorth_loss_exceeds(const DenseMatrix& g, double thr) {
    DenseMatrix d = g;
    const int64_t m = d.rows(), k = d.cols();
    for (int64_t i = 0; i < std::min(m, k); ++i) d(i, i) -= 1.0;
    if (d.frobenius_norm() <= thr) return false;  // ||.||_2 <= ||.||_F settles it exactly
    // ||D||_2 <= sqrt(||D||_1 ||D||_inf) settles "no" as exactly
    double n1 = 0.0, ninf = 0.0;
    std::vector<double> rows(static_cast<size_t>(m), 0.0);
    for (int64_t j = 0; j < k; ++j) {
        double c = 0.0;
        for (int64_t i = 0; i < m; ++i) {
            c += std::fabs(d(i, j));
            rows[i] += std::fabs(d(i, j));
        }
        n1 = std::max(n1, c);
    }
    for (double r : rows) ninf = std::max(ninf, r);
    if (std::sqrt(n1 * ninf) <= thr) return false;
    // power iteration on D^T D: every ||D v|| / ||v|| is a lower bound of ||D||_2, so crossing
    // thr proves "yes" (the common case: a clearly needed second pass) without the O(d^3) SVD
    std::vector<double> v(static_cast<size_t>(k), 1.0), w(static_cast<size_t>(m));
    for (int it = 0; it < 30; ++it) {
        double vv = 0.0;
        for (double x : v) vv += x * x;
        if (vv == 0.0) break;
        std::fill(w.begin(), w.end(), 0.0);
        for (int64_t j = 0; j < k; ++j) {
            const double vj = v[j];
            for (int64_t i = 0; i < m; ++i) w[i] += d(i, j) * vj;
        }
        double ww = 0.0;
        for (double x : w) ww += x * x;
        if (std::sqrt(ww / vv) > thr) return true;
        for (int64_t j = 0; j < k; ++j) {
            double s = 0.0;
            for (int64_t i = 0; i < m; ++i) s += d(i, j) * w[i];
            v[j] = s;
        }
        double nv = 0.0;
        for (double x : v) nv = std::max(nv, std::fabs(x));
        if (nv == 0.0) break;
        for (double& x : v) x /= nv;
    }
    return spectral_norm(d) > thr;  // undecided by the bounds: the exact Jacobi spectral norm
}

HostBiorth host_mgs_biorth(const DenseMatrix& x, const DenseMatrix& y, double drop_tol) {
    HostBiorth out = host_gs(x, y, drop_tol, false);
    const int64_t k = out.p.cols(), n = out.p.rows();
    if (k > 1 && biorth_loss_exceeds(matmul_tn(out.p, out.q), 1e-10)) {
        // rebiorth_pass (biorth.cpp:72-98)
        std::vector<double> pl(static_cast<size_t>(n)), ql(static_cast<size_t>(n));
        for (int64_t l = 0; l < k; ++l) {
            std::copy(out.p.col(l), out.p.col(l) + n, pl.begin());
            std::copy(out.q.col(l), out.q.col(l) + n, ql.begin());
            for (int64_t j = 0; j < l; ++j) {
                const double r = dotn(out.q.col(j), pl.data(), n);
                axpyn(-r, out.p.col(j), pl.data(), n);
                const double s = dotn(out.p.col(j), ql.data(), n);
                axpyn(-s, out.q.col(j), ql.data(), n);
            }
            const double eta = dotn(pl.data(), ql.data(), n);
            if (eta == 0.0) continue;
            const double sc = 1.0 / std::sqrt(std::fabs(eta)), sg = sign_or_plus(eta);
            for (int64_t i = 0; i < n; ++i) {
                out.p(i, l) = sg * pl[i] * sc;
                out.q(i, l) = ql[i] * sc;
            }
        }
    }
    return out;
}

HostBiorth host_cgs_biorth(const DenseMatrix& x, const DenseMatrix& y, double drop_tol) {
    return host_gs(x, y, drop_tol, true);
}

namespace {

// Fast path of the coefficient recurrence for m >= 64: in exact arithmetic MGS-Biorth of (X, Y)
// is the unpivoted LDU factorisation Gxy = L D U with P = X L^-T, Q = Y U^-1 (then the
// sign/sqrt|eta| split of D).  Computed with vectorised/threaded loops; returns false -- and the
// caller runs the column-sequential recurrence instead -- whenever a pivot would be dropped or a
// column cancels (the rare cases where the order of operations matters).
bool coef_mgs_ldu(const DenseMatrix& gxx, const DenseMatrix& gxy, const DenseMatrix& gyy,
                  double drop_tol, double cancel_tol, CoefBiorth& out) {
    const int64_t m = gxy.rows();
    DenseMatrix g = gxy;
    std::vector<double> dpiv(static_cast<size_t>(m));
    for (int64_t l = 0; l < m; ++l) {
        const double d = g(l, l);
        if (!(std::fabs(d) > 0.0) || !std::isfinite(d)) return false;
        dpiv[l] = d;
        const double inv = 1.0 / d;
        for (int64_t i = l + 1; i < m; ++i) g(i, l) *= inv;  // L below the diagonal
        // trailing update G_ij -= L_il * G_lj (G_lj still unscaled = D_l U_lj)
#pragma omp parallel for schedule(static) if (m - l > 96)
        for (int64_t j = l + 1; j < m; ++j) {
            const double glj = g(l, j);
            if (glj == 0.0) continue;
            double* gj = g.col(j);
            const double* gl = g.col(l);
            for (int64_t i = l + 1; i < m; ++i) gj[i] -= gl[i] * glj;
        }
        for (int64_t j = l + 1; j < m; ++j) g(l, j) *= inv;  // U right of the diagonal
    }
    // Ahat = L^-T (unit upper): column c of L^-T = row c of L^-1.  Solve L^T Ahat = I.
    DenseMatrix ah(m, m), bh(m, m);
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t c = 0; c < m; ++c) {
        // L^T a = e_c, L^T upper unit: back substitution; a supported on [0, c]
        double* a = ah.col(c);
        a[c] = 1.0;
        for (int64_t i = c - 1; i >= 0; --i) {
            double s = 0.0;
            for (int64_t k = i + 1; k <= c; ++k) s += g(k, i) * a[k];
            a[i] = -s;
        }
        // U b = e_c, U upper unit: back substitution
        double* b = bh.col(c);
        b[c] = 1.0;
        for (int64_t i = c - 1; i >= 0; --i) {
            double s = 0.0;
            for (int64_t k = i + 1; k <= c; ++k) s += g(i, k) * b[k];
            b[i] = -s;
        }
    }
    // norms of the unscaled residuals: diag(Ah^T Gxx Ah), diag(Bh^T Gyy Bh); naive magnitudes
    std::vector<double> pn2(static_cast<size_t>(m)), qn2(static_cast<size_t>(m));
    bool ok = true;
#pragma omp parallel for schedule(dynamic, 8) reduction(&& : ok)
    for (int64_t c = 0; c < m; ++c) {
        const double* a = ah.col(c);
        const double* b = bh.col(c);
        double sp = 0.0, sq = 0.0, pnaive = 0.0, qnaive = 0.0;
        for (int64_t j = 0; j <= c; ++j) {
            const double* gx = gxx.col(j);
            const double* gy = gyy.col(j);
            double tx = 0.0, ty = 0.0;
            for (int64_t i = 0; i <= c; ++i) {
                tx += gx[i] * a[i];
                ty += gy[i] * b[i];
            }
            sp += a[j] * tx;
            sq += b[j] * ty;
            pnaive += std::fabs(a[j]) * std::sqrt(std::max(0.0, gxx(j, j)));
            qnaive += std::fabs(b[j]) * std::sqrt(std::max(0.0, gyy(j, j)));
        }
        pn2[c] = sp;
        qn2[c] = sq;
        const double pn = std::sqrt(std::max(0.0, sp)), qn = std::sqrt(std::max(0.0, sq));
        if (cancel_tol > 0.0 && ((pnaive > 0.0 && sp < cancel_tol * pnaive * pnaive) ||
                                 (qnaive > 0.0 && sq < cancel_tol * qnaive * qnaive)))
            ok = false;
        if (pn == 0.0 || qn == 0.0 || std::fabs(dpiv[c]) < drop_tol * pn * qn) ok = false;
    }
    if (!ok) return false;
    out.a = DenseMatrix(m, m);
    out.b = DenseMatrix(m, m);
    for (int64_t c = 0; c < m; ++c) {
        const double sc = 1.0 / std::sqrt(std::fabs(dpiv[c])), sg = sign_or_plus(dpiv[c]);
        for (int64_t i = 0; i <= c; ++i) {
            out.a(i, c) = sg * sc * ah(i, c);
            out.b(i, c) = sc * bh(i, c);
        }
        out.kept.push_back(c);
    }
    return true;
}

}  // namespace

CoefBiorth coef_mgs(const DenseMatrix& gxx, const DenseMatrix& gxy, const DenseMatrix& gyy,
                    double drop_tol, bool classical, double cancel_tol, int64_t* stop) {
    const int64_t m = gxy.rows();
    if (stop) *stop = m;
    if (!classical && m >= 64) {
        CoefBiorth fast;
        if (coef_mgs_ldu(gxx, gxy, gyy, drop_tol, cancel_tol, fast)) return fast;
    }
    // coefficient columns of the kept pairs, plus their images ua = Gyx a, ub = Gxy b
    std::vector<std::vector<double>> av, bv, ua, ub;
    CoefBiorth out;
    std::vector<double> al, be, ta, tb;
    for (int64_t l = 0; l < m; ++l) {
        const int64_t len = l + 1;  // supports are within [0, l]
        al.assign(static_cast<size_t>(len), 0.0);
        be.assign(static_cast<size_t>(len), 0.0);
        al[l] = be[l] = 1.0;
        // ta = Gyx e_l = row l of Gxy ;  tb = Gxy e_l = column l of Gxy  (first len entries)
        ta.resize(static_cast<size_t>(len));
        tb.resize(static_cast<size_t>(len));
        for (int64_t i = 0; i < len; ++i) {
            ta[i] = gxy(l, i);
            tb[i] = gxy(i, l);
        }
        const std::vector<double> ta0 = ta, tb0 = tb;
        for (size_t t = 0; t < av.size(); ++t) {
            const int64_t lt = static_cast<int64_t>(av[t].size());  // support of pair t
            // r = <q_t, p~> = b_t^T Gyx alpha  (classical: <q_t, x_l> = b_t^T Gyx e_l)
            const double r = dotn(bv[t].data(), classical ? ta0.data() : ta.data(), lt);
            axpyn(-r, av[t].data(), al.data(), lt);
            axpyn(-r, ua[t].data(), ta.data(), len);
            const double s = dotn(av[t].data(), classical ? tb0.data() : tb.data(), lt);
            axpyn(-s, bv[t].data(), be.data(), lt);
            axpyn(-s, ub[t].data(), tb.data(), len);
        }
        double pn2 = 0.0, qn2 = 0.0, pnaive = 0.0, qnaive = 0.0;
        for (int64_t j = 0; j < len; ++j) {
            if (al[j] != 0.0) pn2 += al[j] * dotn(gxx.col(j), al.data(), len);
            if (be[j] != 0.0) qn2 += be[j] * dotn(gyy.col(j), be.data(), len);
            pnaive += std::fabs(al[j]) * std::sqrt(std::max(0.0, gxx(j, j)));
            qnaive += std::fabs(be[j]) * std::sqrt(std::max(0.0, gyy(j, j)));
        }
        if (cancel_tol > 0.0 && ((pnaive > 0.0 && pn2 < cancel_tol * pnaive * pnaive) ||
                                 (qnaive > 0.0 && qn2 < cancel_tol * qnaive * qnaive))) {
            if (stop) *stop = l;  // caller materialises column l in n-space
            break;
        }
        const double pn = std::sqrt(std::max(0.0, pn2)), qn = std::sqrt(std::max(0.0, qn2));
        const double eta = dotn(al.data(), tb.data(), len);
        if (pn == 0.0 || qn == 0.0 || std::fabs(eta) < drop_tol * pn * qn) {
            if (std::getenv("BOSP_DEBUG"))
                std::fprintf(stderr, "[bosp] coef_mgs drop col %lld/%lld: pn2=%.3e qn2=%.3e eta=%.3e gxx=%.3e gyy=%.3e\n",
                             (long long)l, (long long)m, pn2, qn2, eta, gxx(l, l), gyy(l, l));
            out.dropped.push_back(l);
            continue;
        }
        const double sc = 1.0 / std::sqrt(std::fabs(eta)), sg = sign_or_plus(eta);
        std::vector<double> a_new(al), b_new(be), ua_new(static_cast<size_t>(m)), ub_new(static_cast<size_t>(m));
        for (auto& v : a_new) v *= sg * sc;
        for (auto& v : b_new) v *= sc;
        // full-length images for later columns: ua = Gyx a_new, ub = Gxy b_new
        for (int64_t i = 0; i < m; ++i) {
            double sa = 0.0, sb = 0.0;
            for (int64_t j = 0; j < len; ++j) {
                sa += gxy(j, i) * a_new[j];
                sb += gxy(i, j) * b_new[j];
            }
            ua_new[i] = sa;
            ub_new[i] = sb;
        }
        av.push_back(std::move(a_new));
        bv.push_back(std::move(b_new));
        ua.push_back(std::move(ua_new));
        ub.push_back(std::move(ub_new));
        out.kept.push_back(l);
    }
    const int64_t k = static_cast<int64_t>(out.kept.size());
    out.a = DenseMatrix(m, k);
    out.b = DenseMatrix(m, k);
    for (int64_t t = 0; t < k; ++t)
        for (size_t i = 0; i < av[t].size(); ++i) {
            out.a(static_cast<int64_t>(i), t) = av[t][i];
            out.b(static_cast<int64_t>(i), t) = bv[t][i];
        }
    return out;
}

namespace {
// rebiorth_pass (biorth.cpp:72-98) for k >= 64 as the unpivoted LDU of Gpq -- the same
// recurrence in exact arithmetic (the first pass's coef_mgs_ldu, without drop tests, which the
// second pass does not apply): O(k^3) in threaded level-2/3 loops instead of ~50 ms of scalar
// recurrence at k = 320.  Falls back (false) on a zero or non-finite pivot, whose column the
// sequential form leaves unchanged (biorth.cpp:90).
bool coef_rebiorth_ldu(const DenseMatrix& gpq, CoefBiorth& out) {
    const int64_t m = gpq.rows();
    DenseMatrix g = gpq;
    std::vector<double> dpiv(static_cast<size_t>(m));
    for (int64_t l = 0; l < m; ++l) {
        const double d = g(l, l);
        if (!(std::fabs(d) > 0.0) || !std::isfinite(d)) return false;
        dpiv[l] = d;
        const double inv = 1.0 / d;
        for (int64_t i = l + 1; i < m; ++i) g(i, l) *= inv;
#pragma omp parallel for schedule(static) if (m - l > 96)
        for (int64_t j = l + 1; j < m; ++j) {
            const double glj = g(l, j);
            if (glj == 0.0) continue;
            double* gj = g.col(j);
            const double* gl = g.col(l);
            for (int64_t i = l + 1; i < m; ++i) gj[i] -= gl[i] * glj;
        }
        for (int64_t j = l + 1; j < m; ++j) g(l, j) *= inv;
    }
    out.a = DenseMatrix(m, m);
    out.b = DenseMatrix(m, m);
#pragma omp parallel for schedule(dynamic, 8)
    for (int64_t c = 0; c < m; ++c) {
        double* a = out.a.col(c);  // L^T a = e_c
        a[c] = 1.0;
        for (int64_t i = c - 1; i >= 0; --i) {
            double s = 0.0;
            for (int64_t k = i + 1; k <= c; ++k) s += g(k, i) * a[k];
            a[i] = -s;
        }
        double* b = out.b.col(c);  // U b = e_c
        b[c] = 1.0;
        for (int64_t i = c - 1; i >= 0; --i) {
            double s = 0.0;
            for (int64_t k = i + 1; k <= c; ++k) s += g(i, k) * b[k];
            b[i] = -s;
        }
        const double sc = 1.0 / std::sqrt(std::fabs(dpiv[c])), sg = sign_or_plus(dpiv[c]);
        for (int64_t i = 0; i <= c; ++i) {
            a[i] *= sg * sc;
            b[i] *= sc;
        }
    }
    for (int64_t c = 0; c < m; ++c) out.kept.push_back(c);
    return true;
}
}  // namespace

CoefBiorth coef_rebiorth(const DenseMatrix& gpq) {
    const int64_t k = gpq.rows();
    if (k >= 64) {
        CoefBiorth fast;
        if (coef_rebiorth_ldu(gpq, fast)) return fast;
    }
    std::vector<std::vector<double>> av, bv, ua, ub;
    std::vector<double> al, be, ta, tb;
    for (int64_t l = 0; l < k; ++l) {
        const int64_t len = l + 1;
        al.assign(static_cast<size_t>(len), 0.0);
        be.assign(static_cast<size_t>(len), 0.0);
        al[l] = be[l] = 1.0;
        ta.resize(static_cast<size_t>(len));
        tb.resize(static_cast<size_t>(len));
        for (int64_t i = 0; i < len; ++i) {
            ta[i] = gpq(l, i);
            tb[i] = gpq(i, l);
        }
        for (int64_t t = 0; t < l; ++t) {
            const int64_t lt = static_cast<int64_t>(av[t].size());
            const double r = dotn(bv[t].data(), ta.data(), lt);
            axpyn(-r, av[t].data(), al.data(), lt);
            axpyn(-r, ua[t].data(), ta.data(), len);
            const double s = dotn(av[t].data(), tb.data(), lt);
            axpyn(-s, bv[t].data(), be.data(), lt);
            axpyn(-s, ub[t].data(), tb.data(), len);
        }
        const double eta = dotn(al.data(), tb.data(), len);
        std::vector<double> a_new, b_new;
        if (eta == 0.0) {  // biorth.cpp:90: column left as it was
            a_new.assign(static_cast<size_t>(len), 0.0);
            b_new.assign(static_cast<size_t>(len), 0.0);
            a_new[l] = b_new[l] = 1.0;
        } else {
            const double sc = 1.0 / std::sqrt(std::fabs(eta)), sg = sign_or_plus(eta);
            a_new = al;
            b_new = be;
            for (auto& v : a_new) v *= sg * sc;
            for (auto& v : b_new) v *= sc;
        }
        std::vector<double> ua_new(static_cast<size_t>(k)), ub_new(static_cast<size_t>(k));
        for (int64_t i = 0; i < k; ++i) {
            double sa = 0.0, sb = 0.0;
            for (int64_t j = 0; j < len; ++j) {
                sa += gpq(j, i) * a_new[j];
                sb += gpq(i, j) * b_new[j];
            }
            ua_new[i] = sa;
            ub_new[i] = sb;
        }
        av.push_back(std::move(a_new));
        bv.push_back(std::move(b_new));
        ua.push_back(std::move(ua_new));
        ub.push_back(std::move(ub_new));
    }
    CoefBiorth out;
    out.a = DenseMatrix(k, k);
    out.b = DenseMatrix(k, k);
    for (int64_t t = 0; t < k; ++t) {
        out.kept.push_back(t);
        for (size_t i = 0; i < av[t].size(); ++i) {
            out.a(static_cast<int64_t>(i), t) = av[t][i];
            out.b(static_cast<int64_t>(i), t) = bv[t][i];
        }
    }
    return out;
}

}  // namespace b200
}  // namespace bosp
