// Block sparse-matrix x multi-vector on sm_100a: SELL-32 CSR and matrix-free 5/7-point stencils.
#pragma once

#include <functional>

#include "common.hpp"

namespace bosp {
inline namespace b200 {

// SELL-C-sigma with C = 32, sigma = 1 (no row sorting): rows in slices of 32; within a slice the
// k-th entry of every row is stored contiguously (entry k of lane l at ptr[s] + 32*k + l), so a
// warp's matrix loads are fully coalesced.  Padding entries point at the row itself with value 0.
struct SellDev {
    int64_t n = 0;
    int64_t nslices = 0;
    const int64_t* slice_ptr = nullptr;  // nslices + 1
    const int32_t* slice_w = nullptr;    // nslices
    const int32_t* col = nullptr;
    const double* val = nullptr;
    int64_t nnz = 0;                     // true nonzeros (for algorithmic byte counts)
    // row-partitioned: column indices >= n refer to halo row (c - n) of `halo` (ld `ldh`)
    const double* halo = nullptr;
    int64_t ldh = 0;
};

// DIA (diagonal) storage for banded / stencil-structured CSR matrices: ndiag offsets (ascending,
// the CSR column order within a row), a per-row presence mask (bit d: A(i, i+off[d]) stored in
// the CSR) and, per diagonal, either one constant value (every stored entry equal -- the
// off-diagonals of a constant-coefficient stencil) or an n-vector of values.  Row i's products
// are summed over the present entries in CSR order, so the sums equal the CSR row sums.
constexpr int kDiaMax = 16;
struct DiaDev {
    int64_t n = 0;
    int32_t ndiag = 0;
    int64_t off[kDiaMax] = {};
    double cval[kDiaMax] = {};   // constant diagonals
    int32_t vidx[kDiaMax] = {};  // -1: constant, else row of `val`
    const double* val = nullptr; // nvar x n
    const uint16_t* mask = nullptr;
    uint32_t full_pair = 0;  // mask word of a row pair with every diagonal present
    uint32_t even = 0;       // bit d: off[d] even (16-byte x pairs)
    int64_t nnz = 0;  // CSR nonzeros (algorithmic byte counts)
};

// Fused x(:,j)^T y(:,j) (the CG's p^T A p): per-block partials in `parts` (<= 256 x ncols),
// folded in fixed order by the last block into out[j]; `ticket` must be zero and stays zero.
struct SpmmDot {
    double* parts;              // per-block partials, parts_cap doubles
    unsigned* ticket;           // nullptr: leave the partials unfolded (the consumer folds them)
    double* out;
    const int* active = nullptr;  // optional column mask: inactive columns are neither applied nor dotted
    int64_t parts_cap = 0;
};

// Device CSR -> SELL-32 conversion (rp/ci/vv device copies of the CSR arrays; rp may carry a
// base offset rp[0]).  sell_layout writes the slice widths and offsets (nslices + 1) and returns
// the padded entry count; sell_fill scatters columns/values (padding -> the row itself, 0.0).
int64_t sell_layout(int64_t n, const int64_t* rp, int64_t* slice_ptr, int32_t* slice_w);
void sell_fill(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv, const int64_t* slice_ptr,
               const int32_t* slice_w, int32_t* col, double* val);

// y(:, j) = A x(:, j) for all columns of x (optionally with the fused dots); returns the number
// of row blocks.
int sell_spmm(const SellDev& a, const DMat& x, const DMat& y, const SpmmDot* dot = nullptr);
// Device DIA construction from device CSR arrays (rp may carry a base offset):
//   dia_offsets: distinct column offsets into table[kDiaMax] (unsorted, INT64_MIN = empty);
//                returns the count, or -1 when there are more than kDiaMax;
//   dia_scan:    presence masks + per-diagonal min/max of the raw value bits (constant test);
//   dia_fill:    values of the non-constant diagonals.
int dia_offsets(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* table);
void dia_scan(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv, const DiaDev& layout,
              uint16_t* mask, unsigned long long* vmin, unsigned long long* vmax);
void dia_fill(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv, const DiaDev& layout, double* val);
// y = A x for a DIA matrix (n even), optionally with the fused dots; returns the row blocks.
int dia_spmm(const DiaDev& a, const DMat& x, const DMat& y, const SpmmDot* dot = nullptr);
// Blocks a dot-fused apply of n rows x ncols uses (partials per column).
unsigned spmm_dot_blocks(int64_t n, const SpmmDot& dot, int ncols);

// Structured-grid Laplacian family: y = scale * (L_bc x) + v .* x on nx*ny*nz nodes (nz = 1 ->
// 5-point).  bc: 0 = Neumann graph Laplacian (diag = #in-grid neighbours), 1 = Dirichlet
// (diag = 2*dims).  potential: 0 none, 1 harmonic 0.5|x|^2 with x_i = origin + (i+1)*h,
// 2 explicit per-node array v.
struct StencilDev {
    int64_t nx = 0, ny = 0, nz = 1;  // local grid (partitioned along the slowest axis)
    int32_t dims = 3;                // 3 = 7-point (global nz > 1), 2 = 5-point
    int32_t bc = 0;
    double scale = 1.0;
    int32_t potential = 0;
    double origin = 0.0, h = 1.0;
    const double* v = nullptr;       // local rows of the explicit potential
    // row partition along the slowest axis (z for 3-D, y for 2-D): this rank holds slow-axis
    // planes [s0, s0 + local) of s_global; halo_lo/halo_hi hold the neighbouring planes
    // (plane = nx*ny (3-D) or nx (2-D) values per column, ld = plane) or are null.
    int64_t s0 = 0, s_global = 0;
    const double* halo_lo = nullptr;
    const double* halo_hi = nullptr;
};
// Halo overlap of a slab-partitioned stencil: `exchange` posts the halo exchange (on its own
// stream) and makes the apply stream wait for it; stencil_spmm calls it after launching the
// interior planes, then applies the boundary plane(s) (plane values each, below / above).
struct StencilOverlap {
    int64_t plane = 0;
    bool has_lo = false, has_hi = false;
    std::function<void()> exchange;
};
int stencil_spmm(const StencilDev& s, const DMat& x, const DMat& y, const SpmmDot* dot = nullptr,
                 const StencilOverlap* ov = nullptr);

}  // namespace b200
}  // namespace bosp
