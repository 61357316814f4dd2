// MGS-Biorth coefficient recurrence for a block of m <= 32 columns, run by a 1024-thread CTA
// (device function shared by the standalone kernel, coef_dev.cu, and the fused
// Gram-reduction epilogue, dmma_gemm.cu).
//
// In exact arithmetic the column-sequential recurrence of gs_biorth (biorth.cpp:19-69) applied
// to (X, Y) is the unpivoted LDU factorisation Gxy = L D U of the cross Gram: P = X L^-T,
// Q = Y U^-1, then the sign / sqrt|eta| split of D -- the host's coef_mgs_ldu (small_dense.cpp).
// One thread per element: the LDU, the two unit-triangular inverses (L^-T, U^-1) and the
// residual norms |p_c|^2 = a_c^T Gxx a_c, |q_c|^2 = b_c^T Gyy b_c each step a CTA barrier.  Exactly as on
// the host, a column that would be dropped (|eta| < drop_tol |p| |q|), whose residual cancels
// (< cancel_tol of its naive magnitude squared) or whose pivot is zero / not finite sets
// *status = 1: the caller redoes the block with the column-sequential host recurrence, whose
// order of operations those cases depend on.
#pragma once

#include <cstdio>

namespace bosp {
inline namespace b200 {

constexpr int kCoefM = 32, kCoefL = 33;  // max columns, shared stride
constexpr int kCoefThreads = kCoefM * kCoefM;  // one thread per element
// shared doubles coef_ldu_cta needs
constexpr int kCoefSmem = 3 * kCoefM * kCoefL + 4 * 2 * kCoefM + 5 * kCoefM + 2;

// z: the pair Gram Z^T Z (2m x 2m, column-major, leading dimension ldz; shared or global);
// c: A | B (m x 2m, ldc).  Called by every thread of a kCoefThreads-thread CTA (thread t owns
// element (t % 32, t / 32)); it synchronises the CTA.
//
// Element-parallel: every thread keeps its element in registers and each elimination / back-
// substitution step publishes one row and one column through a double-buffered shared strip,
// so a step costs one CTA barrier.  (Warp-per-column forms of the same loops took 25-45 us:
// every pivot step was a chain of dependent shared-memory round trips.)
__device__ __forceinline__ void coef_ldu_cta(const double* z, int64_t ldz, int m, double* c, int64_t ldc,
                                             int* status, double drop_tol, double cancel_tol, double* work) {
    double* gx = work;                     // X^T X (column-major, stride kCoefL)
    double* gy = gx + kCoefM * kCoefL;     // Y^T Y
    double* ab = gy + kCoefM * kCoefL;     // A^ then (scratch) rows of the inverses
    double* colb = ab + kCoefM * kCoefL;   // [2][kCoefM] published column
    double* rowb = colb + 2 * kCoefM;      // [2][kCoefM] published row
    double* ra = rowb + 2 * kCoefM;        // [2][kCoefM] published row of A^
    double* rb = ra + 2 * kCoefM;          // [2][kCoefM] published row of B^
    double* pn2 = rb + 2 * kCoefM;
    double* qn2 = pn2 + kCoefM;
    double* pnv = qn2 + kCoefM;
    double* qnv = pnv + kCoefM;
    double* dpiv = qnv + kCoefM;
    int* flag = reinterpret_cast<int*>(dpiv + kCoefM);
    const int t = threadIdx.x, i = t % kCoefM, j = t / kCoefM;
    const bool in = i < m && j < m;
    double v = in ? z[i + static_cast<int64_t>(m + j) * ldz] : 0.0;  // Gxy(i, j)
    if (in) {
        gx[j * kCoefL + i] = z[i + static_cast<int64_t>(j) * ldz];             // X^T X
        gy[j * kCoefL + i] = z[(m + i) + static_cast<int64_t>(m + j) * ldz];   // Y^T Y
    }
    if (t == 0) *flag = 0;
    // unpivoted LDU of Gxy (the host's coef_mgs_ldu operation by operation: L = A(i,l) * inv,
    // trailing update fma(-L, A(l,j) unscaled, A(i,j)), U = A(l,j) * inv)
    bool ok = true;
    for (int l = 0; l < m; ++l) {
        const int b = l & 1;
        if (in && j == l) colb[b * kCoefM + i] = v;
        if (in && i == l) rowb[b * kCoefM + j] = v;
        __syncthreads();
        const double d = colb[b * kCoefM + l];
        ok = fabs(d) > 0.0 && isfinite(d);  // uniform
        if (!ok) break;
        const double inv = 1.0 / d;
        if (in) {
            if (j == l && i > l) v *= inv;                                           // L(i, l)
            else if (i == l && j > l) v *= inv;                                      // U(l, j)
            else if (i > l && j > l) v = fma(-(colb[b * kCoefM + i] * inv), rowb[b * kCoefM + j], v);
        }
        if (t == 0) dpiv[l] = d;
    }
    if (!ok) {
        if (t == 0) *status = 1;
        return;
    }
    __syncthreads();  // the last elimination step's reads of the strips are done
    // element (i, j) of L \ U now in v.  A^ = L^-T and B^ = U^-1 (unit upper) by back
    // substitution, column-oriented: step k publishes row k of A^, B^ (final) and column k of
    // L (row k of L^T) / U; entries r < k subtract.  Thread (i, j) owns A^(i, j), B^(i, j).
    double a_ = (i == j) ? 1.0 : 0.0, b_ = a_;
    // factors needed at step k by thread (i, j): L(k, i) and U(i, k) -> publish column/row k
    for (int k = m - 1; k >= 1; --k) {
        const int bb = k & 1;
        if (in && i == k) {
            ra[bb * kCoefM + j] = a_;
            rb[bb * kCoefM + j] = b_;
        }
        if (in && i == k) colb[bb * kCoefM + j] = v;  // L(k, j) for j < k  (row k of L)
        if (in && j == k) rowb[bb * kCoefM + i] = v;  // U(i, k) for i < k  (column k of U)
        __syncthreads();
        if (in && i < k && j >= k) {
            a_ = fma(-colb[bb * kCoefM + i], ra[bb * kCoefM + j], a_);
            b_ = fma(-rowb[bb * kCoefM + i], rb[bb * kCoefM + j], b_);
        }
    }
    if (in) ab[j * kCoefL + i] = a_;
    __syncthreads();
    // residual norms: pn2_c = a_c^T Gxx a_c, qn2_c = b_c^T Gyy b_c; thread (i, j) forms row i of
    // Gxx A^ (resp. Gyy B^) for column j, the columns are folded in shared memory below
    {
        double tx = 0.0, ty = 0.0;
        if (in && i <= j) {
            for (int r = 0; r <= j; ++r) tx = fma(gx[i * kCoefL + r], ab[j * kCoefL + r], tx);
        }
        __syncthreads();
        if (in) ab[j * kCoefL + i] = b_;  // B^ replaces A^ in the scratch
        __syncthreads();
        if (in && i <= j) {
            for (int r = 0; r <= j; ++r) ty = fma(gy[i * kCoefL + r], ab[j * kCoefL + r], ty);
        }
        const double px = (in && i <= j) ? a_ * tx : 0.0, py = (in && i <= j) ? b_ * ty : 0.0;
        const double nx = (in && i <= j) ? fabs(a_) * sqrt(fmax(0.0, gx[i * kCoefL + i])) : 0.0;
        const double ny = (in && i <= j) ? fabs(b_) * sqrt(fmax(0.0, gy[i * kCoefL + i])) : 0.0;
        // warp j holds column j (lanes = rows i): fold with shuffles
        double s0 = px, s1 = py, s2 = nx, s3 = ny;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            s0 += __shfl_xor_sync(0xffffffffu, s0, o);
            s1 += __shfl_xor_sync(0xffffffffu, s1, o);
            s2 += __shfl_xor_sync(0xffffffffu, s2, o);
            s3 += __shfl_xor_sync(0xffffffffu, s3, o);
        }
        if (i == 0 && j < m) {
            pn2[j] = s0;
            qn2[j] = s1;
            pnv[j] = s2;
            qnv[j] = s3;
        }
    }
    __syncthreads();
    if (t < m) {
        const double sp = pn2[t], sq = qn2[t], pv = pnv[t], qv = qnv[t];
        const double pn = sqrt(fmax(0.0, sp)), qn = sqrt(fmax(0.0, sq));
        bool bad = cancel_tol > 0.0 && ((pv > 0.0 && sp < cancel_tol * pv * pv) || (qv > 0.0 && sq < cancel_tol * qv * qv));
        bad = bad || pn == 0.0 || qn == 0.0 || fabs(dpiv[t]) < drop_tol * pn * qn;
        if (bad) atomicOr(flag, 1);
    }
    __syncthreads();
    const int fail = *flag;
    if (t == 0) *status = fail;
    if (fail) return;
    // A = sign(d) A^ / sqrt|d|, B = B^ / sqrt|d| (upper triangular, zeros below)
    if (in) {
        const double d = dpiv[j];
        const double sc = 1.0 / sqrt(fabs(d)), sg = d < 0.0 ? -1.0 : 1.0;
        c[i + static_cast<int64_t>(j) * ldc] = i <= j ? sg * sc * a_ : 0.0;
        c[i + static_cast<int64_t>(m + j) * ldc] = i <= j ? sc * b_ : 0.0;
    }
}

}  // namespace b200
}  // namespace bosp
