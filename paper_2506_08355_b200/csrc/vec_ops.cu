// Column-wise reductions, the batched-CG vector kernels and element-wise helpers.
//
// Reductions are deterministic: grid (chunks x columns), every block writes its partial sums,
// the last block to finish (one ticket per launch) folds the partials in fixed chunk order and
// runs the per-column epilogue.  HBM traffic is one streaming pass over the operands.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "dense_ops.hpp"
#include "ktimer.cuh"
#include "runtime.hpp"

namespace bosp {
inline namespace b200 {

namespace {

constexpr int kThreads = 256;

template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* sh) {
#pragma unroll
    for (int k = 0; k < K; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) sh[warp * K + k] = v[k];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) s += sh[w * K + k];
            v[k] = s;
        }
    }
}

// Generic column reduction: F::row(i, j, acc) accumulates K sums over rows of column j;
// F::skip(j) lets a block skip a masked column; F::fin(j, sums) is the epilogue (last block).
template <int K, class F>
__global__ void __launch_bounds__(kThreads) k_colred(int64_t n, int ncols, int nchunks,
                                                      int64_t chunk, F f, double* partial,
                                                      unsigned* ticket, double* defer, KTimer tm) {
    __shared__ double sh[(kThreads / 32) * K];
    __shared__ bool last;
    const int j = blockIdx.y;
    const int c = blockIdx.x;
    tm.start();
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.0;
    f.prologue(j);
    if (!f.skip(j)) {
        if (c == 0 && threadIdx.x == 0) tm.add_column();
        // 16-byte accesses: rows in pairs (chunk is even, columns are 256-byte aligned)
        const int64_t r0 = c * chunk;
        const int64_t r1 = min(n, r0 + chunk);
        const int64_t pend = r0 + ((r1 - r0) & ~int64_t(1));
        int64_t i = r0 + 2 * threadIdx.x;
        for (; i + 2 * kThreads < pend; i += 4 * kThreads) {
            f.row2(i, j, acc);
            f.row2(i + 2 * kThreads, j, acc);
        }
        for (; i < pend; i += 2 * kThreads) f.row2(i, j, acc);
        if (pend < r1 && threadIdx.x == 0) f.row(pend, j, acc);
    }
    block_sum<K>(acc, sh);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) partial[(static_cast<int64_t>(j) * nchunks + c) * K + k] = acc[k];
        __threadfence();
        const unsigned total = static_cast<unsigned>(nchunks) * ncols;
        last = (atomicAdd(ticket, 1u) == total - 1);
    }
    __syncthreads();
    if (!last) {
        tm.stop();
        return;
    }
    __threadfence();
    // fold: one warp per column, lanes strided over the chunks (all loads independent), then a
    // fixed shuffle tree -- the tail block finishes in a few L2 round trips, not nchunks
    {
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int jj = warp; jj < ncols; jj += kThreads / 32) {
            double s[K];
#pragma unroll
            for (int k = 0; k < K; ++k) s[k] = 0.0;
            for (int cc = lane; cc < nchunks; cc += 32)
#pragma unroll
                for (int k = 0; k < K; ++k) s[k] += __ldcg(&partial[(static_cast<int64_t>(jj) * nchunks + cc) * K + k]);
#pragma unroll
            for (int k = 0; k < K; ++k)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], o);
            if (lane != 0) continue;
            if (defer) {  // row-partitioned: the epilogue runs after the cross-rank allreduce
#pragma unroll
                for (int k = 0; k < K; ++k) defer[k * ncols + jj] = s[k];
            } else {
                f.fin(jj, s);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (!defer) f.fin_all(ncols);
        *ticket = 0u;
    }
    tm.stop();
}

// Epilogue of k_colred on cross-rank sums (one block).
template <int K, class F>
__global__ void k_colred_finish(F f, const double* sums, int ncols) {
    for (int jj = threadIdx.x; jj < ncols; jj += blockDim.x) {
        double s[K];
#pragma unroll
        for (int k = 0; k < K; ++k) s[k] = sums[k * ncols + jj];
        f.fin(jj, s);
    }
    __syncthreads();
    if (threadIdx.x == 0) f.fin_all(ncols);
}

struct NoFinAll {
    __device__ void fin_all(int) const {}
    __device__ void prologue(int) const {}
};

__device__ __forceinline__ double2 ldg2(const double* p) { return __ldg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }
__device__ __forceinline__ void st2(double* p, double a, double b) {
    *reinterpret_cast<double2*>(p) = make_double2(a, b);
}

template <int K, class F>
void launch_colred(const char* family, int64_t n, int ncols, const F& f, double bytes) {
    if (ncols <= 0) return;
    Runtime& rt = Runtime::get();
    const int64_t target = 4 * rt.sm_count();  // 4 waves: 2..32 within 3% on configs 2 and 3
    // >= 1024 rows per chunk: narrow solves (1-8 live columns) still fill the machine
    int nchunks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 1023) / 1024,
                                                                            (target + ncols - 1) / ncols)));
    const int64_t chunk = ((n + nchunks - 1) / nchunks + 1) & ~int64_t(1);  // even: pairs stay aligned
    double* partial = rt.scratch(static_cast<size_t>(nchunks) * ncols * K + static_cast<size_t>(K) * ncols);
    unsigned* ticket = rt.tickets(1);
    // several ranks: park the column sums after the partials, allreduce them, then run the
    // epilogue on the global sums so every rank sets identical scalars
    double* defer = rt.nranks() > 1 ? partial + static_cast<size_t>(nchunks) * ncols * K : nullptr;
    {
        // device-clock timed (works inside the CG graphs); bytes credited per applied column
        KTimer tm{rt.timer_begin(family, bytes, 0.0, 0.0, ncols)};
        LaunchScope ls(family, bytes, 0.0, false);
        dim3 grid(nchunks, ncols);
        k_colred<K, F><<<grid, kThreads, 0, rt.stream()>>>(n, ncols, nchunks, chunk, f, partial, ticket, defer, tm);
        BOSP_LAUNCH_CHECK();
    }
    if (defer) {
        rt.allreduce(defer, static_cast<int64_t>(K) * ncols);
        LaunchScope ls(family, 0.0, 0.0);
        k_colred_finish<K, F><<<1, kThreads, 0, rt.stream()>>>(f, defer, ncols);
        BOSP_LAUNCH_CHECK();
    }
}

// ---- functors -------------------------------------------------------------------------------
// row(i, j, acc) handles one row; row2(i, j, acc) rows i, i+1 (i even) with 16-byte accesses.
struct DotF : NoFinAll {
    const double* x; int64_t ldx;
    const double* y; int64_t ldy;
    double* out;
    __device__ bool skip(int) const { return false; }
    __device__ void row(int64_t i, int j, double (&a)[1]) const {
        a[0] += x[i + j * ldx] * y[i + j * ldy];
    }
    __device__ void row2(int64_t i, int j, double (&a)[1]) const {
        const double2 u = ldg2(x + i + j * ldx), v = ldg2(y + i + j * ldy);
        a[0] += u.x * v.x + u.y * v.y;
    }
    __device__ void fin(int j, const double (&s)[1]) const { out[j] = s[0]; }
};

struct ResidF : NoFinAll {
    const double *kx, *my, *xb, *yb, *x, *y;
    int64_t lkx, lmy, lxb, lyb, lx, ly;
    const double* lam;
    double *num, *den;
    __device__ bool skip(int) const { return false; }
    __device__ void row(int64_t i, int j, double (&a)[2]) const {
        const double l = lam[j];
        const double r1 = kx[i + j * lkx] - l * yb[i + j * lyb];
        const double r2 = my[i + j * lmy] - l * xb[i + j * lxb];
        const double xv = x[i + j * lx], yv = y[i + j * ly];
        a[0] += r1 * r1 + r2 * r2;
        a[1] += xv * xv + yv * yv;
    }
    __device__ void row2(int64_t i, int j, double (&a)[2]) const {
        const double l = lam[j];
        const double2 k2 = ldg2(kx + i + j * lkx), y2 = ldg2(yb + i + j * lyb);
        const double2 m2 = ldg2(my + i + j * lmy), x2 = ldg2(xb + i + j * lxb);
        const double2 xv = ldg2(x + i + j * lx), yv = ldg2(y + i + j * ly);
        const double r1a = k2.x - l * y2.x, r1b = k2.y - l * y2.y;
        const double r2a = m2.x - l * x2.x, r2b = m2.y - l * x2.y;
        a[0] += (r1a * r1a + r2a * r2a) + (r1b * r1b + r2b * r2b);
        a[1] += (xv.x * xv.x + yv.x * yv.x) + (xv.y * xv.y + yv.y * yv.y);
    }
    __device__ void fin(int j, const double (&s)[2]) const {
        num[j] = s[0];
        den[j] = s[1];
    }
};

__device__ __forceinline__ void cg_publish(const CgScalars& s, int ncols, bool reset_loops) {
    int c = 0;
    for (int j = 0; j < ncols; ++j) c += s.active[j];
    // an iteration counts when some column entered it active (unrolled graphs launch idle ones)
    if (reset_loops) {
        *s.loops = 0;
    } else if (*s.any_active > 0) {
        *s.loops += 1;
        if (s.total) *s.total += 1;
    }
    *s.any_active = c;
    if (s.has_cond) cudaGraphSetConditional(s.cond, c > 0 ? 1u : 0u);
}

// CG start: x = 0, r = b, p = b and ||b||^2 in one pass.
struct CgStartF {
    const double* b; int64_t lb;
    double *x, *r, *p; int64_t lx, lr, lp;
    CgScalars s;
    double tol; int max_iter;
    __device__ void prologue(int) const {}
    __device__ bool dead(int j) const { return s.m_live && j >= *s.m_live; }
    __device__ bool skip(int j) const { return dead(j); }
    __device__ void row(int64_t i, int j, double (&a)[1]) const {
        const double v = b[i + j * lb];
        x[i + j * lx] = 0.0;
        r[i + j * lr] = v;
        p[i + j * lp] = v;
        a[0] += v * v;
    }
    __device__ void row2(int64_t i, int j, double (&a)[1]) const {
        const double2 v = ldg2(b + i + j * lb);
        st2(x + i + j * lx, 0.0, 0.0);
        st2(r + i + j * lr, v.x, v.y);
        st2(p + i + j * lp, v.x, v.y);
        a[0] += v.x * v.x + v.y * v.y;
    }
    __device__ void fin(int j, const double (&sm)[1]) const {
        if (dead(j)) {
            s.rr[j] = s.bnorm[j] = 0.0;
            s.iters[j] = s.broken[j] = s.active[j] = 0;
            return;
        }
        const double bn = sqrt(sm[0]);
        s.rr[j] = sm[0];
        s.bnorm[j] = bn;
        s.iters[j] = 0;
        s.broken[j] = 0;
        // cg.cpp:22 (bnorm == 0 -> column skipped) and the loop test at :33
        s.active[j] = (bn != 0.0 && sqrt(sm[0]) > tol * bn && max_iter > 0) ? 1 : 0;
    }
    __device__ void fin_all(int ncols) const { cg_publish(s, ncols, true); }
};

struct CgStartX0F {
    const double *b, *x0, *ax0; int64_t lb, lx0, lax0;
    double *x, *r, *p; int64_t lx, lr, lp;
    CgScalars s;
    double tol; int max_iter;
    __device__ void prologue(int) const {}
    __device__ bool skip(int) const { return false; }
    __device__ void row(int64_t i, int j, double (&a)[2]) const {
        const double bv = b[i + j * lb];
        const double rv = bv - ax0[i + j * lax0];
        x[i + j * lx] = x0[i + j * lx0];
        r[i + j * lr] = rv;
        p[i + j * lp] = rv;
        a[0] += rv * rv;
        a[1] += bv * bv;
    }
    __device__ void row2(int64_t i, int j, double (&a)[2]) const {
        row(i, j, a);
        row(i + 1, j, a);
    }
    __device__ void fin(int j, const double (&sm)[2]) const {
        const double bn = sqrt(sm[1]);
        s.rr[j] = sm[0];
        s.bnorm[j] = bn;
        s.iters[j] = 0;
        s.broken[j] = 0;
        s.active[j] = (bn != 0.0 && sqrt(sm[0]) > tol * bn && max_iter > 0) ? 1 : 0;
    }
    __device__ void fin_all(int ncols) const { cg_publish(s, ncols, true); }
};

struct CgPapF : NoFinAll {
    const double *p, *ap; int64_t lp, lap;
    CgScalars s;
    __device__ bool skip(int j) const { return s.active[j] == 0; }
    __device__ void row(int64_t i, int j, double (&a)[1]) const { a[0] += p[i + j * lp] * ap[i + j * lap]; }
    __device__ void row2(int64_t i, int j, double (&a)[1]) const {
        const double2 u = ldg2(p + i + j * lp), v = ldg2(ap + i + j * lap);
        a[0] += u.x * v.x + u.y * v.y;
    }
    __device__ void fin(int j, const double (&sm)[1]) const {
        if (s.active[j]) s.pap[j] = sm[0];
    }
};

// x += alpha p, r -= alpha ap, accumulate r^T r (cg.cpp:37-48); epilogue decides the masks.
// With pap_parts set, every block first folds the SpMM's per-block p^T A p partials of its own
// column (fixed order, all blocks in parallel) instead of the SpMM's last block doing it
// serially; block 0 of the column publishes the value to s.pap for the epilogue.
__device__ __forceinline__ double& xr_pap_slot() {
    __shared__ double v;
    return v;
}

struct CgXrF {
    double *x, *r; const double *p, *ap; int64_t lx, lr, lp, lap;
    CgScalars s;
    double* beta;
    double tol; int max_iter;
    const double* pap_parts = nullptr;
    int nparts = 0;
    __device__ void prologue(int j) const {
        if (!pap_parts) return;
        __shared__ double red[kThreads / 32];
        double t = 0.0;
        for (int q = threadIdx.x; q < nparts; q += kThreads)
            t += __ldcg(pap_parts + static_cast<int64_t>(j) * nparts + q);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double v = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) v += red[w];
            xr_pap_slot() = v;
            if (blockIdx.x == 0) s.pap[j] = v;
        }
        __syncthreads();
    }
    __device__ double pap(int j) const { return pap_parts ? xr_pap_slot() : s.pap[j]; }
    __device__ bool skip(int j) const { return s.active[j] == 0 || !(pap(j) > 0.0); }
    // x += alpha p happens here (the host loop and the separate-update path) or, with defer_x,
    // in the direction kernel (CgDirXF), which reads p anyway: 3 instead of 6 passes here
    bool defer_x = false;
    __device__ void row(int64_t i, int j, double (&a)[1]) const {
        const double alpha = s.rr[j] / pap(j);
        if (!defer_x) x[i + j * lx] = x[i + j * lx] + alpha * p[i + j * lp];
        const double rv = r[i + j * lr] - alpha * ap[i + j * lap];
        r[i + j * lr] = rv;
        a[0] += rv * rv;
    }
    __device__ void row2(int64_t i, int j, double (&a)[1]) const {
        const double alpha = s.rr[j] / pap(j);
        if (!defer_x) {
            const double2 xv = ld2(x + i + j * lx), pv = ldg2(p + i + j * lp);
            st2(x + i + j * lx, xv.x + alpha * pv.x, xv.y + alpha * pv.y);
        }
        const double2 rv = ld2(r + i + j * lr), av = ldg2(ap + i + j * lap);
        const double r0 = rv.x - alpha * av.x, r1 = rv.y - alpha * av.y;
        st2(r + i + j * lr, r0, r1);
        a[0] += r0 * r0 + r1 * r1;
    }
    __device__ void fin(int j, const double (&sm)[1]) const {
        if (!s.active[j]) {
            beta[j] = 0.0;
            s.alpha[j] = 0.0;
            return;
        }
        if (!(s.pap[j] > 0.0)) {  // cg.cpp:40-44: breakdown keeps the current iterate
            s.broken[j] = 1;
            s.active[j] = 0;
            beta[j] = 0.0;
            s.alpha[j] = 0.0;
            return;
        }
        const double rr_new = sm[0];
        s.alpha[j] = s.rr[j] / s.pap[j];  // the alpha the rows applied
        beta[j] = rr_new / s.rr[j];
        s.rr[j] = rr_new;
        s.iters[j] += 1;
        s.active[j] = (sqrt(rr_new) > tol * s.bnorm[j] && s.iters[j] < max_iter) ? 1 : 0;
    }
    __device__ void fin_all(int ncols) const { cg_publish(s, ncols, false); }
};

// ---- element-wise kernels ----------------------------------------------------------------
// f(i, j) one row, f.pair(i, j) rows i, i+1 (i even, 16-byte accesses).
template <class F>
__global__ void __launch_bounds__(kThreads) k_cols(int64_t n, F f, KTimer tm) {
    const int j = blockIdx.y;
    if (f.skip(j)) return;
    tm.start();
    if (blockIdx.x == 0 && threadIdx.x == 0) tm.add_column();
    const int64_t npair = n >> 1;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(kThreads) + threadIdx.x; q < npair; q += stride)
        f.pair(2 * q, j);
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) f(n - 1, j);
    tm.stop();
}

template <class F>
void launch_cols(const char* family, int64_t n, int ncols, const F& f, double bytes) {
    if (ncols <= 0 || n <= 0) return;
    Runtime& rt = Runtime::get();
    // 32 waves of blocks over all columns: the CG direction/x update (5 streams) went 1.08 ->
    // ~0.9 ms per 64-column launch at 128^3 (8 waves: the grid-stride loop left HBM idle)
    const int64_t target = 32LL * rt.sm_count();
    const unsigned gx = static_cast<unsigned>(std::max<int64_t>(
        1, std::min<int64_t>((n / 2 + kThreads - 1) / kThreads, (target + ncols - 1) / ncols)));
    KTimer tm{rt.timer_begin(family, bytes, 0.0, 0.0, ncols)};
    LaunchScope ls(family, bytes, 0.0, false);
    k_cols<F><<<dim3(gx, ncols), kThreads, 0, rt.stream()>>>(n, f, tm);
    BOSP_LAUNCH_CHECK();
}

struct LamAxmyF {
    const double *a, *b; double* o; int64_t la, lb, lo; const double* lam;
    __device__ bool skip(int) const { return false; }
    __device__ void operator()(int64_t i, int j) const { o[i + j * lo] = lam[j] * a[i + j * la] - b[i + j * lb]; }
    __device__ void pair(int64_t i, int j) const {
        const double l = lam[j];
        const double2 u = ldg2(a + i + j * la), v = ldg2(b + i + j * lb);
        st2(o + i + j * lo, l * u.x - v.x, l * u.y - v.y);
    }
};
struct LamAxpyF {
    const double* x; double* y; int64_t lx, ly; const double* lam;
    __device__ bool skip(int) const { return false; }
    __device__ void operator()(int64_t i, int j) const { y[i + j * ly] += lam[j] * x[i + j * lx]; }
    __device__ void pair(int64_t i, int j) const {
        const double l = lam[j];
        const double2 u = ldg2(x + i + j * lx), v = ld2(y + i + j * ly);
        st2(y + i + j * ly, v.x + l * u.x, v.y + l * u.y);
    }
};
struct SubScaledF {  // y -= s[0] x (device scalar)
    const double* x; double* y; int64_t lx, ly; const double* s;
    __device__ bool skip(int) const { return false; }
    __device__ void operator()(int64_t i, int j) const { y[i + j * ly] -= s[0] * x[i + j * lx]; }
    __device__ void pair(int64_t i, int j) const {
        const double a = s[0];
        const double2 u = ldg2(x + i + j * lx), v = ld2(y + i + j * ly);
        st2(y + i + j * ly, v.x - a * u.x, v.y - a * u.y);
    }
};
struct AxpbyF {
    double a, b; const double* x; double* y; int64_t lx, ly;
    __device__ bool skip(int) const { return false; }
    __device__ void operator()(int64_t i, int j) const {
        const double xv = x[i + j * lx];
        y[i + j * ly] = (b == 0.0) ? a * xv : a * xv + b * y[i + j * ly];
    }
    __device__ void pair(int64_t i, int j) const {
        const double2 u = ld2(x + i + j * lx);
        if (b == 0.0) {
            st2(y + i + j * ly, a * u.x, a * u.y);
        } else {
            const double2 v = ld2(y + i + j * ly);
            st2(y + i + j * ly, a * u.x + b * v.x, a * u.y + b * v.y);
        }
    }
};
struct DiagF {
    const double* d; const double* x; double* y; int64_t lx, ly;
    __device__ bool skip(int) const { return false; }
    __device__ void operator()(int64_t i, int j) const { y[i + j * ly] = d[i] * x[i + j * lx]; }
    __device__ void pair(int64_t i, int j) const {
        (*this)(i, j);
        (*this)(i + 1, j);
    }
};
// x += alpha p (the iteration's update, deferred from CgXrF) and p = r + beta p for columns still
// active (cg.cpp:37, 49): x, p read once for both.  alpha == 0: the column did not move.
struct CgDirXF {
    double* x; const double* r; double* p; int64_t lx, lr, lp; const double* alpha; const double* beta;
    const int* active;
    __device__ bool skip(int j) const { return alpha[j] == 0.0; }
    __device__ void operator()(int64_t i, int j) const {
        const double pv = p[i + j * lp];
        x[i + j * lx] = x[i + j * lx] + alpha[j] * pv;
        if (active[j]) p[i + j * lp] = r[i + j * lr] + beta[j] * pv;
    }
    __device__ void pair(int64_t i, int j) const {
        const double aj = alpha[j];
        const double2 pv = ld2(p + i + j * lp), xv = ld2(x + i + j * lx);
        st2(x + i + j * lx, xv.x + aj * pv.x, xv.y + aj * pv.y);
        if (active[j]) {
            const double bj = beta[j];
            const double2 u = ldg2(r + i + j * lr);
            st2(p + i + j * lp, u.x + bj * pv.x, u.y + bj * pv.y);
        }
    }
};


__global__ void k_transpose(const double* __restrict__ a, int64_t lda, int64_t rows, int64_t cols,
                            double* __restrict__ t, int64_t ldt) {
    __shared__ double tile[32][33];
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32, c0 = static_cast<int64_t>(blockIdx.y) * 32;
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int64_t r = r0 + threadIdx.x, c = c0 + j;
        if (r < rows && c < cols) tile[j][threadIdx.x] = a[c * lda + r];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += 8) {
        const int64_t c = c0 + threadIdx.x, r = r0 + j;  // t(c, r) = a(r, c)
        if (r < rows && c < cols) t[r * ldt + c] = tile[threadIdx.x][j];
    }
}

}  // namespace

void transpose(const DMat& a, const DMat& t) {
    if (a.rows == 0 || a.cols == 0) return;
    Runtime& rt = Runtime::get();
    LaunchScope ls("transpose", 16.0 * a.rows * a.cols, 0.0);
    dim3 grid(static_cast<unsigned>((a.rows + 31) / 32), static_cast<unsigned>((a.cols + 31) / 32));
    k_transpose<<<grid, dim3(32, 8), 0, rt.stream()>>>(a.p, a.ld, a.rows, a.cols, t.p, t.ld);
    BOSP_LAUNCH_CHECK();
}

void col_dots(const DMat& x, const DMat& y, double* out) {
    DotF f;
    f.x = x.p; f.ldx = x.ld; f.y = y.p; f.ldy = y.ld; f.out = out;
    launch_colred<1>("coldot", x.rows, static_cast<int>(x.cols), f, 16.0 * x.rows * x.cols);
}

void residual_sums(const DMat& kx, const DMat& my, const DMat& xb, const DMat& yb, const DMat& x,
                   const DMat& y, const double* lam, double* num, double* den) {
    ResidF f;
    f.kx = kx.p; f.my = my.p; f.xb = xb.p; f.yb = yb.p; f.x = x.p; f.y = y.p;
    f.lkx = kx.ld; f.lmy = my.ld; f.lxb = xb.ld; f.lyb = yb.ld; f.lx = x.ld; f.ly = y.ld;
    f.lam = lam; f.num = num; f.den = den;
    launch_colred<2>("residual", x.rows, static_cast<int>(x.cols), f, 8.0 * 4 * x.rows * x.cols);
}

void lam_axmy(const DMat& a, const DMat& b, const double* lam, const DMat& out) {
    LamAxmyF f{a.p, b.p, out.p, a.ld, b.ld, out.ld, lam};
    launch_cols("elementwise", a.rows, static_cast<int>(a.cols), f, 24.0 * a.rows * a.cols);
}

void lam_axpy(const DMat& x, const double* lam, const DMat& y) {
    LamAxpyF f{x.p, y.p, x.ld, y.ld, lam};
    launch_cols("elementwise", x.rows, static_cast<int>(x.cols), f, 24.0 * x.rows * x.cols);
}

void sub_scaled(const DMat& x, const double* s_dev, const DMat& y) {
    SubScaledF f{x.p, y.p, x.ld, y.ld, s_dev};
    launch_cols("elementwise", x.rows, static_cast<int>(x.cols), f, 24.0 * x.rows * x.cols);
}

void axpby(double a, const DMat& x, double b, const DMat& y) {
    AxpbyF f{a, b, x.p, y.p, x.ld, y.ld};
    launch_cols("elementwise", x.rows, static_cast<int>(x.cols), f, 24.0 * x.rows * x.cols);
}

void diag_scale(const double* d, const DMat& x, const DMat& y) {
    DiagF f{d, x.p, y.p, x.ld, y.ld};
    launch_cols("elementwise", x.rows, static_cast<int>(x.cols), f, 24.0 * x.rows * x.cols);
}

namespace {
__global__ void k_set_int(int* p, int v) { *p = v; }
}  // namespace

void set_device_int(int* p, int v) {
    LaunchScope ls("cg_vec");
    k_set_int<<<1, 1, 0, Runtime::get().stream()>>>(p, v);
    BOSP_LAUNCH_CHECK();
}

void cg_start(const DMat& b, const DMat& x, const DMat& r, const DMat& p, const CgScalars& s,
              double tol, int max_iter) {
    CgStartF f;
    f.b = b.p; f.lb = b.ld; f.x = x.p; f.r = r.p; f.p = p.p; f.lx = x.ld; f.lr = r.ld; f.lp = p.ld;
    f.s = s; f.tol = tol; f.max_iter = max_iter;
    launch_colred<1>("cg_vec", b.rows, static_cast<int>(b.cols), f, 32.0 * b.rows * b.cols);
}

void cg_start_x0(const DMat& b, const DMat& x0, const DMat& ax0, const DMat& x, const DMat& r,
                 const DMat& p, const CgScalars& s, double tol, int max_iter) {
    CgStartX0F f;
    f.b = b.p; f.x0 = x0.p; f.ax0 = ax0.p; f.lb = b.ld; f.lx0 = x0.ld; f.lax0 = ax0.ld;
    f.x = x.p; f.r = r.p; f.p = p.p; f.lx = x.ld; f.lr = r.ld; f.lp = p.ld;
    f.s = s; f.tol = tol; f.max_iter = max_iter;
    launch_colred<2>("cg_vec", b.rows, static_cast<int>(b.cols), f, 48.0 * b.rows * b.cols);
}

void cg_pap(const DMat& p, const DMat& ap, const CgScalars& s) {
    CgPapF f;
    f.p = p.p; f.ap = ap.p; f.lp = p.ld; f.lap = ap.ld; f.s = s;
    launch_colred<1>("cg_vec", p.rows, static_cast<int>(p.cols), f, 16.0 * p.rows * p.cols);
}

void cg_update(const DMat& x, const DMat& r, const DMat& p, const DMat& ap, const CgScalars& s,
               double tol, int max_iter, const double* pap_parts, int nparts) {
    CgXrF f;
    f.x = x.p; f.r = r.p; f.p = p.p; f.ap = ap.p; f.lx = x.ld; f.lr = r.ld; f.lp = p.ld; f.lap = ap.ld;
    f.s = s; f.beta = s.beta;
    f.tol = tol; f.max_iter = max_iter;
    f.pap_parts = pap_parts;
    f.nparts = nparts;
    f.defer_x = true;
    launch_colred<1>("cg_vec", x.rows, static_cast<int>(x.cols), f, 24.0 * x.rows * x.cols);
    CgDirXF d{x.p, r.p, p.p, x.ld, r.ld, p.ld, s.alpha, s.beta, s.active};
    launch_cols("cg_vec", r.rows, static_cast<int>(r.cols), d, 40.0 * r.rows * r.cols);
}

}  // namespace b200
}  // namespace bosp
