// MGS-Biorth coefficient recurrence for a block of m <= 32 columns, run by a CTA of >= 64 threads
// (device function shared by the standalone kernel, coef_dev.cu, and the fused
// Gram-reduction epilogue, dmma_gemm.cu).
//
// In exact arithmetic the column-sequential recurrence of gs_biorth (biorth.cpp:19-69) applied
// to (X, Y) is the unpivoted LDU factorisation Gxy = L D U of the cross Gram: P = X L^-T,
// Q = Y U^-1, then the sign / sqrt|eta| split of D -- the host's coef_mgs_ldu (small_dense.cpp).
// Warp 0 factors Gxy in registers (lane j owns column j; the L column of each pivot is
// broadcast by shuffles); then the warps invert L^T and U column by column (lane = row) and
// compute |p_c|^2 = a_c^T Gxx a_c, |q_c|^2 = b_c^T Gyy b_c.  (A shared-memory form of the same
// loops took ~18 us: every update waited on the previous store.)  Exactly as on
// the host, a column that would be dropped (|eta| < drop_tol |p| |q|), whose residual cancels
// (< cancel_tol of its naive magnitude squared) or whose pivot is zero / not finite sets
// *status = 1: the caller redoes the block with the column-sequential host recurrence, whose
// order of operations those cases depend on.
#pragma once

namespace bosp {
inline namespace b200 {

constexpr int kCoefM = 32, kCoefL = 33;  // max columns, shared stride
// shared doubles coef_ldu_cta needs
constexpr int kCoefSmem = 3 * kCoefM * kCoefL + 5 * kCoefM + 2;

// z: the pair Gram Z^T Z (2m x 2m, column-major, leading dimension ldz; shared or global);
// c: A | B (m x 2m, ldc); every thread of the CTA calls it (it synchronises the CTA).
__device__ __forceinline__ void coef_ldu_cta(const double* z, int64_t ldz, int m, double* c, int64_t ldc,
                                             int* status, double drop_tol, double cancel_tol, double* work) {
    double* g = work;                    // L \ U (column-major, stride kCoefL)
    double* gx = g + kCoefM * kCoefL;    // X^T X
    double* gy = gx + kCoefM * kCoefL;   // Y^T Y
    double* pn2 = gy + kCoefM * kCoefL;
    double* qn2 = pn2 + kCoefM;
    double* pnv = qn2 + kCoefM;
    double* qnv = pnv + kCoefM;
    double* dpiv = qnv + kCoefM;
    int* flag = reinterpret_cast<int*>(dpiv + kCoefM);
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    constexpr unsigned kAll = 0xffffffffu;
    for (int e = t; e < m * m; e += blockDim.x) {
        const int i = e % m, j = e / m;
        gx[j * kCoefL + i] = z[i + static_cast<int64_t>(j) * ldz];             // X^T X
        gy[j * kCoefL + i] = z[(m + i) + static_cast<int64_t>(m + j) * ldz];   // Y^T Y
    }
    for (int e = t; e < m * m; e += blockDim.x) {
        const int i = e % m, j = e / m;
        g[j * kCoefL + i] = z[i + static_cast<int64_t>(m + j) * ldz];          // Gxy = X^T Y
    }
    __syncthreads();
    if (warp == 0) {
        // unpivoted LDU of Gxy in place (L below the diagonal, U right of it), same operation
        // order as the host's coef_mgs_ldu: lane j owns column j; per pivot the L column is read by
        // broadcast.  Restrict-qualified pointers let the update loop batch its loads (written
        // through plain pointers, every update waited on the previous store: ~18 us).
        bool ok = true;
        for (int l = 0; l < m; ++l) {
            const double d = g[l * kCoefL + l];
            ok = fabs(d) > 0.0 && isfinite(d);  // uniform: every lane read the same pivot
            if (!ok) break;
            const double inv = 1.0 / d;
            if (lane > l && lane < m) g[l * kCoefL + lane] *= inv;  // L(lane, l)
            __syncwarp();
            if (lane > l && lane < m) {
                const double* __restrict__ gl = g + l * kCoefL;
                double* __restrict__ gj = g + lane * kCoefL;
                const double glj = gj[l];  // U(l, lane), unscaled
#pragma unroll 4
                for (int i = l + 1; i < m; ++i) gj[i] = fma(-gl[i], glj, gj[i]);
                gj[l] = glj * inv;
            }
            if (lane == 0) dpiv[l] = d;
            __syncwarp();
        }
        if (lane == 0) *flag = ok ? 0 : 1;
    }
    __syncthreads();
    if (*flag) {
        if (t == 0) *status = 1;
        return;
    }
    // A^ = L^-T and B^ = U^-1 (unit upper) column by column: half of the warps take the columns of
    // A^, half those of B^; lane r holds entry r of the column, the substitution runs from the
    // diagonal up (the newest entry broadcast by a shuffle, an axpy with the factor's column /
    // row).  Then the column's residual norm a^T Gxx a (b^T Gyy b) and its naive magnitude; the
    // finished column goes straight to A | B (scaled once the pivots are checked, below).
    const int nw = static_cast<int>(blockDim.x >> 5), half = nw >= 2 ? nw / 2 : 1;
    if (warp < 2 * half) {
        const bool is_b = warp >= half;
        const double* gg = is_b ? gy : gx;
        for (int cc = is_b ? warp - half : warp; cc < m; cc += half) {
            double v = lane == cc ? 1.0 : 0.0;
            for (int k = cc; k > 0; --k) {
                const double vk = __shfl_sync(kAll, v, k);
                // L^T a = e_c: a_r -= L(k, r) a_k;  U b = e_c: b_r -= U(r, k) b_k   (r < k)
                if (lane < k) v = fma(-(is_b ? g[k * kCoefL + lane] : g[lane * kCoefL + k]), vk, v);
            }
            double tx = 0.0;  // lane j: (G v)_j over the support [0, cc]
            for (int i = 0; i <= cc; ++i) {
                const double vi = __shfl_sync(kAll, v, i);
                if (lane <= cc) tx = fma(gg[lane * kCoefL + i], vi, tx);
            }
            double sp = lane <= cc ? v * tx : 0.0;
            double nv = lane <= cc ? fabs(v) * sqrt(fmax(0.0, gg[lane * kCoefL + lane])) : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                sp += __shfl_xor_sync(kAll, sp, o);
                nv += __shfl_xor_sync(kAll, nv, o);
            }
            if (lane == 0) {
                (is_b ? qn2 : pn2)[cc] = sp;
                (is_b ? qnv : pnv)[cc] = nv;
            }
            if (lane < m) c[lane + static_cast<int64_t>((is_b ? m : 0) + cc) * ldc] = lane <= cc ? v : 0.0;
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
    for (int e = t; e < 2 * m * m; e += blockDim.x) {
        const int i = e % m, j = e / m, jj = j % m;
        const double d = dpiv[jj];
        const double sc = 1.0 / sqrt(fabs(d)), sg = (d < 0.0 && j < m) ? -1.0 : 1.0;
        c[i + static_cast<int64_t>(j) * ldc] *= sg * sc;
    }
}

}  // namespace b200
}  // namespace bosp
