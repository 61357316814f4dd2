// SELL-32 CSR SpMM and matrix-free 5/7-point stencil SpMM (fp64).
//
// One thread per row.  The SELL kernel loads its row's (column, value) pairs once into registers
// (coalesced: entry k of the 32 rows of a slice is contiguous) and then sweeps all right-hand-
// side columns four at a time, so the matrix crosses HBM once per apply and x/y are streamed
// once per column (16 B per row per column).  Neighbour re-reads of x hit L1/L2.  Reference:
// SparseMatrixCSR::apply (sparse_csr.cpp:29-36) via from_csr (linear_operator.cpp:33-43), and
// the matrix-free from_callback path (linear_operator.cpp:45-47) for the stencils.
#include <algorithm>
#include <cstdlib>

#include "runtime.hpp"
#include "sparse_ops.hpp"

namespace bosp {
inline namespace b200 {

namespace {

constexpr int kRows = 256;  // threads per block = rows per block (8 SELL slices)

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Device-clock timing of one launch (Runtime::timer_begin): slot[0] = max(~start) -> earliest
// start, slot[1] = max(end) -> latest end.
struct KTimer {
    unsigned long long* slot;
    __device__ __forceinline__ void start() const {
        if (slot && threadIdx.x == 0) atomicMax(&slot[0], ~gtimer());
    }
    __device__ __forceinline__ void stop() const {
        if (slot) {
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                atomicMax(&slot[1], gtimer());
            }
        }
    }
};

// Rows whose slice is wider than kWMax fall back to the streaming loop below.
constexpr int kWMax = 16;

__global__ void __launch_bounds__(kRows) k_sell(SellDev a, const double* __restrict__ x, int64_t ldx,
                                                 double* __restrict__ y, int64_t ldy, int ncols,
                                                 KTimer tm) {
    tm.start();
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRows + threadIdx.x;
    if (row < a.n) {
        const int64_t s = row >> 5;
        const int64_t base = a.slice_ptr[s] + (row & 31);
        const int w = a.slice_w[s];
        if (w <= kWMax) {
            int col[kWMax];
            double val[kWMax];
#pragma unroll
            for (int k = 0; k < kWMax; ++k) {
                col[k] = k < w ? __ldg(a.col + base + 32 * k) : 0;
                val[k] = k < w ? __ldg(a.val + base + 32 * k) : 0.0;
            }
            int j = 0;
            for (; j + 4 <= ncols; j += 4) {
                const double* x0 = x + static_cast<int64_t>(j) * ldx;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
                for (int k = 0; k < kWMax; ++k) {
                    if (k < w) {
                        const double* xc = x0 + col[k];
                        s0 += val[k] * __ldg(xc);
                        s1 += val[k] * __ldg(xc + ldx);
                        s2 += val[k] * __ldg(xc + 2 * ldx);
                        s3 += val[k] * __ldg(xc + 3 * ldx);
                    }
                }
                double* yo = y + static_cast<int64_t>(j) * ldy + row;
                yo[0] = s0;
                yo[ldy] = s1;
                yo[2 * ldy] = s2;
                yo[3 * ldy] = s3;
            }
            for (; j < ncols; ++j) {
                const double* x0 = x + static_cast<int64_t>(j) * ldx;
                double s0 = 0.0;
#pragma unroll
                for (int k = 0; k < kWMax; ++k)
                    if (k < w) s0 += val[k] * __ldg(x0 + col[k]);
                y[static_cast<int64_t>(j) * ldy + row] = s0;
            }
        } else {
            for (int j = 0; j < ncols; ++j) {
                const double* x0 = x + static_cast<int64_t>(j) * ldx;
                double s0 = 0.0;
                for (int k = 0; k < w; ++k)
                    s0 += __ldg(a.val + base + 32 * k) * __ldg(x0 + __ldg(a.col + base + 32 * k));
                y[static_cast<int64_t>(j) * ldy + row] = s0;
            }
        }
    }
    tm.stop();
}

// Column-group variant: grid.y walks groups of CB columns, the row's entries are re-read per
// group (from L2).  More independent blocks; kept for shapes where it wins.
template <int CB>
__global__ void __launch_bounds__(kRows) k_sell_cb(SellDev a, const double* __restrict__ x, int64_t ldx,
                                                    double* __restrict__ y, int64_t ldy, int ncols,
                                                    KTimer tm) {
    tm.start();
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kRows + threadIdx.x;
    if (row < a.n) {
        const int j0 = blockIdx.y * CB;
        const int64_t s = row >> 5;
        const int64_t base = a.slice_ptr[s] + (row & 31);
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
    tm.stop();
}

template <int CB>
__global__ void __launch_bounds__(kRows) k_stencil(StencilDev st, const double* __restrict__ x,
                                                    int64_t ldx, double* __restrict__ y,
                                                    int64_t ldy, int ncols, KTimer tm) {
    tm.start();
    const int64_t n = st.nx * st.ny * st.nz;
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * kRows + threadIdx.x;
    if (idx < n) {
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
    tm.stop();
}

}  // namespace

void sell_spmm(const SellDev& a, const DMat& x, const DMat& y) {
    if (a.n == 0 || x.cols == 0) return;
    Runtime& rt = Runtime::get();
    const int ncols = static_cast<int>(x.cols);
    // algorithmic (minimum) traffic: CSR once (8 B value + 4 B int32 index per nnz,
    // 4 B per row pointer) + x read once + y written once
    const double bytes = 12.0 * a.nnz + 4.0 * (a.n + 1) + 16.0 * a.n * ncols;
    const double flops = 2.0 * a.nnz * ncols;
    KTimer tm{rt.timer_begin("spmm", bytes, flops)};
    LaunchScope ls("spmm", bytes, flops, false);
    // Column groups of CB (grid.y) keep many independent blocks in flight; measured 2x the
    // bandwidth of the all-columns-per-thread variant (k_sell) on config 2 (B200).
    static const int variant = std::getenv("BOSP_SPMM_CB") ? std::atoi(std::getenv("BOSP_SPMM_CB")) : 4;
    const unsigned gx = static_cast<unsigned>((a.n + kRows - 1) / kRows);
    switch (variant) {
        case 0: k_sell<<<gx, kRows, 0, rt.stream()>>>(a, x.p, x.ld, y.p, y.ld, ncols, tm); break;
        case 1: k_sell_cb<1><<<dim3(gx, ncols), kRows, 0, rt.stream()>>>(a, x.p, x.ld, y.p, y.ld, ncols, tm); break;
        case 2: k_sell_cb<2><<<dim3(gx, (ncols + 1) / 2), kRows, 0, rt.stream()>>>(a, x.p, x.ld, y.p, y.ld, ncols, tm); break;
        case 8: k_sell_cb<8><<<dim3(gx, (ncols + 7) / 8), kRows, 0, rt.stream()>>>(a, x.p, x.ld, y.p, y.ld, ncols, tm); break;
        default: k_sell_cb<4><<<dim3(gx, (ncols + 3) / 4), kRows, 0, rt.stream()>>>(a, x.p, x.ld, y.p, y.ld, ncols, tm); break;
    }
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
    const double bytes = 16.0 * n * ncols, flops = 2.0 * pts * n * ncols;
    KTimer tm{rt.timer_begin("spmm", bytes, flops)};
    LaunchScope ls("spmm", bytes, flops, false);
    k_stencil<CB><<<grid, kRows, 0, rt.stream()>>>(s, x.p, x.ld, y.p, y.ld, ncols, tm);
    BOSP_LAUNCH_CHECK();
}

}  // namespace b200
}  // namespace bosp
