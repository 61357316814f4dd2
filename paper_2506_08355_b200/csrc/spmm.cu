// SELL-32 CSR SpMM and matrix-free 5/7-point stencil SpMM (fp64).
//
// Both kernels map one thread to one row and CB right-hand-side columns (registers), grid.y
// walks the column groups.  HBM traffic is ideally 16 B per row per column (x read once, y
// written once); neighbour re-reads of x are L1/L2 hits.  The SELL matrix (12 B/nnz + padding)
// is read once per column group and stays L2-resident across groups.  Reference:
// SparseMatrixCSR::apply (sparse_csr.cpp:29-36) via from_csr (linear_operator.cpp:33-43), and
// the matrix-free from_callback path (linear_operator.cpp:45-47) for the stencils.
#include <algorithm>

#include "runtime.hpp"
#include "sparse_ops.hpp"

namespace bosp {
inline namespace b200 {

namespace {

constexpr int kRows = 256;  // threads per block = rows per block (8 SELL slices)

template <int CB>
__global__ void __launch_bounds__(kRows) k_sell(SellDev a, const double* __restrict__ x, int64_t ldx,
                                                 double* __restrict__ y, int64_t ldy, int ncols) {
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRows + threadIdx.x;
    if (row >= a.n) return;
    const int j0 = blockIdx.y * CB;
    const int64_t s = row >> 5;
    const int lane = static_cast<int>(row & 31);
    const int64_t base = a.slice_ptr[s] + lane;
    const int w = a.slice_w[s];
    double acc[CB];
#pragma unroll
    for (int c = 0; c < CB; ++c) acc[c] = 0.0;
    const double* xb = x + static_cast<int64_t>(j0) * ldx;
    for (int k = 0; k < w; ++k) {
        const int col = __ldg(a.col + base + 32 * k);
        const double v = __ldg(a.val + base + 32 * k);
#pragma unroll
        for (int c = 0; c < CB; ++c)
            if (j0 + c < ncols) acc[c] += v * __ldg(xb + c * ldx + col);
    }
#pragma unroll
    for (int c = 0; c < CB; ++c)
        if (j0 + c < ncols) y[(j0 + c) * ldy + row] = acc[c];
}

template <int CB>
__global__ void __launch_bounds__(kRows) k_stencil(StencilDev st, const double* __restrict__ x,
                                                    int64_t ldx, double* __restrict__ y,
                                                    int64_t ldy, int ncols) {
    const int64_t n = st.nx * st.ny * st.nz;
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * kRows + threadIdx.x;
    if (idx >= n) return;
    const int j0 = blockIdx.y * CB;
    const int64_t nxy = st.nx * st.ny;
    const int64_t i = idx % st.nx;
    const int64_t jy = (idx / st.nx) % st.ny;
    const int64_t kz = idx / nxy;
    const bool xm = i > 0, xp = i + 1 < st.nx;
    const bool ym = jy > 0, yp = jy + 1 < st.ny;
    const bool zm = kz > 0, zp = kz + 1 < st.nz;
    const int dims = st.nz > 1 ? 3 : 2;
    double diag;
    if (st.bc == 0)
        diag = static_cast<double>(xm + xp + ym + yp + (dims == 3 ? (zm + zp) : 0));
    else
        diag = 2.0 * dims;
    diag *= st.scale;
    double pot = 0.0;
    if (st.potential == 1) {
        const double cx = st.origin + (i + 1) * st.h;
        const double cy = st.origin + (jy + 1) * st.h;
        const double cz = dims == 3 ? st.origin + (kz + 1) * st.h : 0.0;
        pot = 0.5 * (cx * cx + cy * cy + cz * cz);
    } else if (st.potential == 2) {
        pot = __ldg(st.v + idx);
    }
    const double dg = diag + pot;
#pragma unroll
    for (int c = 0; c < CB; ++c) {
        if (j0 + c >= ncols) break;
        const double* xc = x + static_cast<int64_t>(j0 + c) * ldx + idx;
        double nb = 0.0;
        if (xm) nb += __ldg(xc - 1);
        if (xp) nb += __ldg(xc + 1);
        if (ym) nb += __ldg(xc - st.nx);
        if (yp) nb += __ldg(xc + st.nx);
        if (dims == 3) {
            if (zm) nb += __ldg(xc - nxy);
            if (zp) nb += __ldg(xc + nxy);
        }
        y[(j0 + c) * ldy + idx] = dg * __ldg(xc) - st.scale * nb;
    }
}

}  // namespace

void sell_spmm(const SellDev& a, const DMat& x, const DMat& y) {
    if (a.n == 0 || x.cols == 0) return;
    Runtime& rt = Runtime::get();
    constexpr int CB = 4;
    const int ncols = static_cast<int>(x.cols);
    dim3 grid(static_cast<unsigned>((a.n + kRows - 1) / kRows), (ncols + CB - 1) / CB);
    // algorithmic (minimum) traffic: CSR once (8 B value + 4 B int32 index per nnz,
    // 4 B per row pointer) + x read once + y written once
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 16.0 * a.n * ncols;
    LaunchScope ls("spmm", bytes, 2.0 * a.nnz * ncols);
    k_sell<CB><<<grid, kRows, 0, rt.stream()>>>(a, x.p, x.ld, y.p, y.ld, ncols);
    BOSP_LAUNCH_CHECK();
}

void stencil_spmm(const StencilDev& s, const DMat& x, const DMat& y) {
    const int64_t n = s.nx * s.ny * s.nz;
    if (n == 0 || x.cols == 0) return;
    Runtime& rt = Runtime::get();
    constexpr int CB = 4;
    const int ncols = static_cast<int>(x.cols);
    dim3 grid(static_cast<unsigned>((n + kRows - 1) / kRows), (ncols + CB - 1) / CB);
    const double pts = s.nz > 1 ? 7.0 : 5.0;
    LaunchScope ls("spmm", 16.0 * n * ncols, 2.0 * pts * n * ncols);
    k_stencil<CB><<<grid, kRows, 0, rt.stream()>>>(s, x.p, x.ld, y.p, y.ld, ncols);
    BOSP_LAUNCH_CHECK();
}

}  // namespace b200
}  // namespace bosp
