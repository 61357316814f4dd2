// fp64 tall-skinny GEMMs on the DMMA pipe for sm_100a.
//
//  * gram()    G = A^T B   (A: n x a, B: n x b, a,b <= a few hundred, n up to millions)
//              -> split-K over n: every CTA owns one (BM x BN) output tile and a contiguous
//                 row range; partial tiles go to scratch and a deterministic two-level
//                 reduction (fixed split order) produces G.  Reference: block_inner
//                 (kernels.cpp:47-68), assemble_projected_applied (projected_lrep.cpp:40-46).
//  * product() Out = alpha A C + beta Out  (A: n x k, C: k x b small or, for the dense
//              operator, k = n) -> one CTA per (BM x BN) output tile, K loop over k.
//              Reference: block_product / block_axpy (kernels.cpp:70-104) and the dense
//              operator (linear_operator.cpp:12-31).
//
// Operands are staged global->shared with 16-byte cp.async (LDGSTS) in a 3-stage ring, fed to
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  Shared layouts are padded (+4 doubles) so the
// fragment loads of a half-warp hit 16 distinct 8-byte bank pairs.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "coef_ldu.cuh"
#include "dense_ops.hpp"
#include "runtime.hpp"

namespace bosp {
inline namespace b200 {

namespace {

#ifndef BOSP_KSTAGES
#define BOSP_KSTAGES 3
#endif
constexpr int kStages = BOSP_KSTAGES;
#ifndef BOSP_KBK
#define BOSP_KBK 32
#endif
constexpr int kBK = BOSP_KBK;      // k-depth of one pipeline stage

__device__ __forceinline__ const double* colptr(const ColList& cl, int c) {
    int s = 0;
#pragma unroll
    for (int i = 1; i < kMaxSeg; ++i)
        if (i < cl.nseg && c >= cl.start[i]) s = i;
    return cl.p[s] + static_cast<int64_t>(c - cl.start[s]) * cl.ld[s];
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
                 "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Load a "k-contiguous" tile: R columns (from ColList starting at col0, total ncols), rows
// [k0, k0+kBK) clipped to kmax, into smem[c * (BK + 4) + k].  Missing data is zero-filled.
template <int R, int NT, int BK = kBK>
__device__ __forceinline__ void load_kcontig(double* smem, const ColList& cl, int col0, int ncols,
                                             int64_t k0, int64_t kmax) {
    constexpr int kChunks = R * (BK / 2);
    for (int ch = threadIdx.x; ch < kChunks; ch += NT) {
        const int c = ch / (BK / 2);
        const int kp = ch % (BK / 2);
        const int64_t k = k0 + 2 * kp;
        const int gc = col0 + c;
        int bytes = 0;
        const double* src = cl.p[0];
        if (gc < ncols && k < kmax) {
            const int64_t rem = kmax - k;
            bytes = rem >= 2 ? 16 : 8;
            src = colptr(cl, gc) + k;
        }
        cp_async16(smem + c * (BK + 4) + 2 * kp, src, bytes);
    }
}

// The same k-contiguous tile load with every per-thread address computed once per CTA.  A thread
// always copies the same row pair (2 kp) of the same kPer columns of every stage (NT is a
// multiple of BK / 2), so the column pointers (ColList segment lookup) and shared offsets are
// fixed; a stage only adds its first row k0.  (ncu on the per-chunk form: ~60 % of the Gram
// kernel's issued instructions were this address arithmetic, DMMA only 10 %.)
template <int R, int NT, int BK>
struct KcontigLoader {
    static_assert(NT % (BK / 2) == 0, "a thread keeps one row pair across stages");
    static constexpr int kChunks = R * (BK / 2);
    static constexpr int kPer = (kChunks + NT - 1) / NT;
    const double* src[kPer];  // column base + this thread's row pair offset; nullptr: zero fill
    int off[kPer];            // shared offset (c * (BK + 4) + 2 kp), -1: no chunk
    int kp2;
    const double* dummy;      // a valid address for zero-fill copies

    __device__ __forceinline__ void init(const ColList& cl, int col0, int ncols) {
        kp2 = 2 * (static_cast<int>(threadIdx.x) % (BK / 2));
        dummy = cl.p[0];
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int ch = static_cast<int>(threadIdx.x) + i * NT;
            const int c = ch / (BK / 2);
            const bool have = (kChunks % NT == 0) || ch < kChunks;
            off[i] = have ? c * (BK + 4) + kp2 : -1;
            src[i] = (have && col0 + c < ncols) ? colptr(cl, col0 + c) + kp2 : nullptr;
        }
    }
    // rows [k0, k0 + BK) of the tile, rows >= kmax zero-filled
    __device__ __forceinline__ void load(double* smem, int64_t k0, int64_t kmax) const {
        const int64_t k = k0 + kp2;
        const int bytes = k + 2 <= kmax ? 16 : (k < kmax ? 8 : 0);
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            if ((kChunks % NT) != 0 && off[i] < 0) continue;
            const bool v = src[i] != nullptr;
            cp_async16(smem + off[i], v ? src[i] + k0 : dummy, v ? bytes : 0);
        }
    }
};

// m-contiguous tile load (BK columns x BM rows into smem[k * (BM + 4) + m]) for the product's A
// operand with fixed per-thread rows: a thread always copies rows m0 + 2 mp of columns
// k0 + kk0 + i * (NT / (BM / 2)); the column base pointers come from a shared table filled once
// per CTA (no ColList segment search per chunk and stage).
template <int BM, int NT, int BK>
struct McontigLoader {
    static_assert(NT % (BM / 2) == 0, "a thread keeps one row pair across stages");
    static constexpr int kRowsPer = NT / (BM / 2);  // column stride between a thread's chunks
    static constexpr int kPer = (BK * (BM / 2) + NT - 1) / NT;
    int kk0, soff;
    int64_t m;   // first row of this thread's pair
    int bytes;   // rows of the pair inside the matrix (16, 8 or 0 bytes)
    const double* dummy;
    __device__ __forceinline__ void init(const double* any, int64_t m0, int64_t mmax) {
        const int mp = static_cast<int>(threadIdx.x) % (BM / 2);
        kk0 = static_cast<int>(threadIdx.x) / (BM / 2);
        m = m0 + 2 * mp;
        const int64_t rem = mmax - m;
        bytes = rem >= 2 ? 16 : (rem == 1 ? 8 : 0);
        soff = kk0 * (BM + 4) + 2 * mp;
        dummy = any;
    }
    __device__ __forceinline__ void load(double* smem, const double* const* coltab, int k0, int kcols) const {
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int kk = kk0 + i * kRowsPer;
            if ((BK * (BM / 2)) % NT != 0 && kk >= BK) continue;
            const int gk = k0 + kk;
            const bool v = gk < kcols && bytes > 0;
            cp_async16(smem + soff + i * kRowsPer * (BM + 4), v ? coltab[gk] + m : dummy, v ? bytes : 0);
        }
    }
};

// Load an "m-contiguous" tile for the NN product: kBK columns (k0..k0+kBK of A, clipped to
// kcols) x BM rows (m0.., clipped to mmax) into smem[k * (BM+4) + m].
template <int BM, int NT, int BK = kBK>
__device__ __forceinline__ void load_mcontig(double* smem, const ColList& cl, int k0, int kcols,
                                             int64_t m0, int64_t mmax) {
    constexpr int kChunks = BK * (BM / 2);
    for (int ch = threadIdx.x; ch < kChunks; ch += NT) {
        const int kk = ch / (BM / 2);
        const int mp = ch % (BM / 2);
        const int gk = k0 + kk;
        const int64_t m = m0 + 2 * mp;
        int bytes = 0;
        const double* src = cl.p[0];
        if (gk < kcols && m < mmax) {
            const int64_t rem = mmax - m;
            bytes = rem >= 2 ? 16 : 8;
            src = colptr(cl, gk) + m;
        }
        cp_async16(smem + kk * (BM + 4) + 2 * mp, src, bytes);
    }
}

// ------------------------------------------------------------------------------------------
// Gram kernel
// ------------------------------------------------------------------------------------------
struct GramParams {
    GramJob job[4];
    int64_t n;
    int tiles_n[4];      // column tiles per job
    int tiles[4];        // tiles per job (sym: upper-triangular tiles only)
    int sym[4];          // G symmetric: tile t -> upper pair, mirrored stores
    int same[4];         // and A, B are the same columns (B fragments = A fragments)
    int splits;
    int64_t chunk;       // rows per split (multiple of kBK)
    double* partial;     // [job][split][tile][BM*BN]
    int64_t job_stride;  // doubles per job in partial
};

// BOSP_PROF_SHAPES=1 (measurement): profile families split by launch shape, e.g.
// "gram_wide:320x320s/2" (a x b, symmetric, jobs) -- interned, the profiler keeps the pointer.
const char* shape_family(const char* fam, int a, int b, bool sym, int njobs) {
    static const bool on = std::getenv("BOSP_PROF_SHAPES") != nullptr;
    if (!on) return fam;
    static std::mutex mu;
    static std::set<std::string> names;
    std::lock_guard<std::mutex> lk(mu);
    return names.insert(std::string(fam) + ":" + std::to_string(a) + "x" + std::to_string(b) + (sym ? "s" : "") + "/" +
                        std::to_string(njobs)).first->c_str();
}

bool same_columns(const ColList& a, const ColList& b) {
    if (a.nseg != b.nseg) return false;
    for (int s = 0; s < a.nseg; ++s)
        if (a.p[s] != b.p[s] || a.ld[s] != b.ld[s] || a.start[s + 1] != b.start[s + 1]) return false;
    return true;
}

// Tile index -> (tm, tn).  Symmetric jobs enumerate the upper triangle row by row
// (tm <= tn, T tiles per side).
__device__ __forceinline__ void gram_tile(const GramParams& prm, int jb, int tile, int& tm, int& tn) {
    const int T = prm.tiles_n[jb];
    if (!prm.sym[jb]) {
        tm = tile / T;
        tn = tile % T;
        return;
    }
    int r = 0, t = tile;
    while (t >= T - r) {
        t -= T - r;
        ++r;
    }
    tm = r;
    tn = r + t;
}

// Store one reduced Gram element; symmetric jobs store (m, n) for m <= n and mirror it.
__device__ __forceinline__ void gram_store(const GramJob& job, bool sym, int m, int nn, double v) {
    if (!sym) {
        job.g[m + static_cast<int64_t>(nn) * job.ldg] = v;
    } else if (m <= nn) {
        job.g[m + static_cast<int64_t>(nn) * job.ldg] = v;
        job.g[nn + static_cast<int64_t>(m) * job.ldg] = v;
    }
}

template <int BM, int BN, int WM, int WN, int GBK = kBK, int GST = kStages>
__global__ void __launch_bounds__(WM * WN * 32)
k_gram(GramParams prm) {
    constexpr int kBK = GBK, kStages = GST, kLdK = GBK + 4;
    constexpr int NT = WM * WN * 32;
    constexpr int WTM = BM / WM, WTN = BN / WN;
    constexpr int MT = WTM / 8, NTL = WTN / 8;
    extern __shared__ __align__(16) double smem[];
    double* sa = smem;                           // [kStages][BM][kLdK]
    double* sb = smem + kStages * BM * kLdK;     // [kStages][BN][kLdK]

    const int jb = blockIdx.z;
    const GramJob& job = prm.job[jb];
    const int tile = blockIdx.x;
    if (tile >= prm.tiles[jb]) return;
    int tm, tn;
    gram_tile(prm, jb, tile, tm, tn);
    const int m0 = tm * BM, n0 = tn * BN;
    const int acols = job.a.cols(), bcols = job.b.cols();
    const int64_t kb = static_cast<int64_t>(blockIdx.y) * prm.chunk;
    const int64_t ke = min(prm.n, kb + prm.chunk);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm0 = (warp / WN) * WTM, wn0 = (warp % WN) * WTN;

    double acc[MT][NTL][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int nk = ke > kb ? static_cast<int>((ke - kb + kBK - 1) / kBK) : 0;
    KcontigLoader<BM, NT, kBK> lda;
    KcontigLoader<BN, NT, kBK> ldb;
    lda.init(job.a, m0, acols);
    ldb.init(job.b, n0, bcols);
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) {
            lda.load(sa + s * BM * kLdK, kb + s * kBK, ke);
            ldb.load(sb + s * BN * kLdK, kb + s * kBK, ke);
        }
        cp_async_commit();
    }
    // symmetric job, diagonal tile: a warp tile strictly below the diagonal only produces
    // mirrored entries (never stored) -- it keeps the pipeline but leaves the DMMA pipe to the
    // other warps (a quarter of a 2 x 2 diagonal tile's work)
    const bool idle = prm.sym[jb] && tm == tn && wm0 >= wn0 + WTN;
    for (int it = 0; it < nk; ++it) {
        cp_async_wait<kStages - 2>();
        __syncthreads();
        const int st = it % kStages;
        const double* a = sa + st * BM * kLdK;
        const double* b = sb + st * BN * kLdK;
        if (!idle) {
#pragma unroll
            for (int kk = 0; kk < kBK; kk += 4) {
                double af[MT], bf[NTL];
#pragma unroll
                for (int i = 0; i < MT; ++i) af[i] = a[(wm0 + i * 8 + gid) * kLdK + kk + tig];
#pragma unroll
                for (int j = 0; j < NTL; ++j) bf[j] = b[(wn0 + j * 8 + gid) * kLdK + kk + tig];
#pragma unroll
                for (int i = 0; i < MT; ++i)
#pragma unroll
                    for (int j = 0; j < NTL; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
            }
        }
        const int nxt = it + kStages - 1;
        if (nxt < nk) {
            const int sn = nxt % kStages;
            lda.load(sa + sn * BM * kLdK, kb + nxt * kBK, ke);
            ldb.load(sb + sn * BN * kLdK, kb + nxt * kBK, ke);
        }
        cp_async_commit();
    }
    cp_async_wait<0>();

    if (prm.splits == 1) {  // whole K range in this CTA: write G directly
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
            for (int j = 0; j < NTL; ++j) {
                const int m = m0 + wm0 + i * 8 + gid;
                const int nn = n0 + wn0 + j * 8 + 2 * tig;
                if (m < acols) {
                    if (nn < bcols) gram_store(job, prm.sym[jb], m, nn, acc[i][j][0]);
                    if (nn + 1 < bcols) gram_store(job, prm.sym[jb], m, nn + 1, acc[i][j][1]);
                }
            }
        return;
    }
    // partial tile -> scratch (element (m, n) of the tile at m + n*BM)
    double* part = prm.partial + jb * prm.job_stride +
                   (static_cast<int64_t>(blockIdx.y) * prm.tiles[jb] + tile) * (BM * BN);
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j) {
            const int m = wm0 + i * 8 + gid;
            const int nn = wn0 + j * 8 + 2 * tig;
            part[m + nn * BM] = acc[i][j][0];
            part[m + (nn + 1) * BM] = acc[i][j][1];
        }
}

// Sum split partials in a fixed order.  A block owns 32 consecutive output elements; its 8
// warps each fold a strided eighth of the splits (two accumulators, loads independent across
// the unrolled loop), then warp 0 folds the 8 group sums in order.  grid.z = job.
constexpr int kRedElems = 8, kRedGroups = 32;  // 8 outputs x 32 split groups per block: ~4x the blocks of 32 x 8

template <int BM, int BN>
__global__ void __launch_bounds__(kRedElems * kRedGroups) k_gram_reduce(GramParams prm) {
    __shared__ double part_sum[kRedGroups][kRedElems];
    const int jb = blockIdx.z;
    const GramJob& job = prm.job[jb];
    const int el = threadIdx.x % kRedElems, grp = threadIdx.x / kRedElems;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * kRedElems + el;
    const int64_t total = static_cast<int64_t>(prm.tiles[jb]) * BM * BN;
    double s0 = 0.0, s1 = 0.0;
    if (e < total) {
        const double* part = prm.partial + jb * prm.job_stride + e;
        int sp = grp;
#pragma unroll 4
        for (; sp + kRedGroups < prm.splits; sp += 2 * kRedGroups) {
            s0 += __ldcg(part + sp * total);
            s1 += __ldcg(part + (sp + kRedGroups) * total);
        }
        if (sp < prm.splits) s0 += __ldcg(part + sp * total);
    }
    part_sum[grp][el] = s0 + s1;
    __syncthreads();
    if (grp != 0 || e >= total) return;
    double s = 0.0;
#pragma unroll
    for (int g = 0; g < kRedGroups; ++g) s += part_sum[g][el];
    const int tile = static_cast<int>(e / (BM * BN));
    const int r = static_cast<int>(e % (BM * BN));
    int tm, tn;
    gram_tile(prm, jb, tile, tm, tn);
    const int m = tm * BM + r % BM;
    const int nn = tn * BN + r / BM;
    if (m >= job.a.cols() || nn >= job.b.cols()) return;
    gram_store(job, prm.sym[jb], m, nn, s);
}

// The split reduction of a single-job symmetric Gram (k_gram_reduce) fused with the MGS-Biorth
// coefficients of the reduced pair Gram: the last block to finish (ticket) runs coef_ldu_cta on
// G -- one launch less per MGS-Biorth call, and no Gram round trip through the host.
struct CoefParams {
    double* c;          // A | B (m x 2m)
    int64_t ldc;
    int* status;
    unsigned* ticket;   // zero on entry, left zero
    int m;
    double drop_tol, cancel_tol;
};

template <int LDP>
__global__ void __launch_bounds__(kCoefThreads) k_gram_reduce_coef(GramParams prm, CoefParams cp) {
    constexpr int kE = 32, kG = kCoefThreads / kE;  // 32 outputs x 32 split groups per block
    __shared__ double part_sum[kG][kE];
    __shared__ double work[kCoefSmem];
    __shared__ bool last;
    const GramJob& job = prm.job[0];
    const int el = threadIdx.x % kE, grp = threadIdx.x / kE;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * kE + el;
    const int64_t total = static_cast<int64_t>(LDP) * LDP;
    double s0 = 0.0, s1 = 0.0;
    // symmetric: only the upper triangle of the real columns is stored (and mirrored) -- the
    // rest of the LDP x LDP partial (padding, the uncomputed lower tiles) is not even read
    // (m = 20: 820 of 4096 elements)
    const int em = static_cast<int>(e % LDP), en = static_cast<int>(e / LDP);
    const bool need = e < total && em <= en && en < job.b.cols();
    if (need) {
        const double* part = prm.partial + e;
        int sp = grp;
#pragma unroll 4
        for (; sp + kG < prm.splits; sp += 2 * kG) {
            s0 += __ldcg(part + sp * total);
            s1 += __ldcg(part + (sp + kG) * total);
        }
        if (sp < prm.splits) s0 += __ldcg(part + sp * total);
    }
    part_sum[grp][el] = s0 + s1;
    __syncthreads();
    if (grp == 0 && need) {
        double s = 0.0;
#pragma unroll
        for (int g = 0; g < kG; ++g) s += part_sum[g][el];
        gram_store(job, true, em, en, s);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(cp.ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    coef_ldu_cta(job.g, job.ldg, cp.m, cp.c, cp.ldc, cp.status, cp.drop_tol, cp.cancel_tol, work);
    if (threadIdx.x == 0) *cp.ticket = 0u;
}

template <int BM, int BN, int WM, int WN, int GBK = kBK, int GST = kStages>
void launch_gram(const GramJob* jobs, int njobs, int64_t n) {
    constexpr int kBK = GBK, kStages = GST, kLdK = GBK + 4;
    Runtime& rt = Runtime::get();
    GramParams prm{};
    int max_tiles = 0;
    for (int j = 0; j < njobs; ++j) {
        prm.job[j] = jobs[j];
        prm.tiles_n[j] = (jobs[j].b.cols() + BN - 1) / BN;
        prm.sym[j] = jobs[j].sym && BM == BN;
        const int tm = (jobs[j].a.cols() + BM - 1) / BM;
        prm.tiles[j] = prm.sym[j] ? tm * (tm + 1) / 2 : tm * prm.tiles_n[j];
        max_tiles = std::max(max_tiles, prm.tiles[j]);
    }
    prm.n = n;
    constexpr int NTh = WM * WN * 32;
    constexpr size_t smem_b = sizeof(double) * kStages * (BM + BN) * kLdK;
    static int resident[64] = {0};  // CTAs per SM, per device
    if (resident[rt.device() & 63] == 0) {
        int r = 0;
        BOSP_CUDA(cudaFuncSetAttribute(k_gram<BM, BN, WM, WN, GBK, GST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_b)));
        BOSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_gram<BM, BN, WM, WN, GBK, GST>, NTh, smem_b));
        resident[rt.device() & 63] = std::max(1, r);
    }
    const int kblocks = static_cast<int>((n + kBK - 1) / kBK);
    // Split count by wave efficiency: tiles x splits CTAs over `slots` resident CTA slots run in
    // ceil(total / slots) waves.  Among split counts giving at least ~2 waves of CTAs (more CTAs
    // amortise the tail) with >= 4 stages of work per CTA, <= 16 waves and split partials <= 3 %
    // of the operand bytes (>= 32 MB), take the one whose last wave is fullest (ties within 0.5 %: fewer
    // splits).  (The previous rule, ~2 waves rounded down, gave the dense operator's 128 tiles
    // 4 splits = 1.73 waves: 774 -> 687 us per apply; a 320 x 320 Gram 4 instead of 2 waves: +3 %.)
    const int slots = resident[rt.device() & 63] * rt.sm_count();
    const int per_split = max_tiles * njobs;
    double opnd = 0.0;
    for (int j = 0; j < njobs; ++j) opnd += 8.0 * n * (jobs[j].a.cols() + jobs[j].b.cols());
    // (small problems: a 32 MB floor, or config 1's n = 2000 dense apply would get one split)
    const int pcap = static_cast<int>(std::max(1.0, std::max(0.03 * opnd, 32.0 * (1 << 20)) / (8.0 * BM * BN * per_split)));
    const int smax = std::max(1, std::min({kblocks / 4, 512, std::max(1, 16 * slots / per_split), pcap}));
    const int smin = std::min(smax, std::max(1, (19 * slots / 10 + per_split - 1) / per_split));
    int splits = smin;
    double best = -1.0;
    for (int sp = smin; sp <= smax; ++sp) {
        const int64_t total = static_cast<int64_t>(sp) * per_split;
        const int64_t waves = (total + slots - 1) / slots;
        const double eff = static_cast<double>(total) / static_cast<double>(waves * slots);
        if (eff > best + 0.005) {
            best = eff;
            splits = sp;
        }
    }
    const int kb_per = (kblocks + splits - 1) / splits;
    prm.chunk = static_cast<int64_t>(kb_per) * kBK;
    splits = static_cast<int>((n + prm.chunk - 1) / prm.chunk);
    prm.splits = std::max(1, splits);
    prm.job_stride = static_cast<int64_t>(prm.splits) * max_tiles * BM * BN;
    prm.partial = rt.scratch(static_cast<size_t>(prm.job_stride) * njobs);

    constexpr int NT = WM * WN * 32;
    constexpr size_t smem = sizeof(double) * kStages * (BM + BN) * kLdK;
    static unsigned attr_mask = 0;
    rt.once_per_device(attr_mask, [&] { BOSP_CUDA(cudaFuncSetAttribute(k_gram<BM, BN, WM, WN, GBK, GST>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); });
    double flops = 0.0, bytes = 0.0;
    for (int j = 0; j < njobs; ++j) {
        flops += 2.0 * n * (double)jobs[j].a.cols() * jobs[j].b.cols() * (prm.sym[j] ? 0.5 : 1.0);
        bytes += 8.0 * n * (double)(same_columns(jobs[j].a, jobs[j].b) ? jobs[j].a.cols() : jobs[j].a.cols() + jobs[j].b.cols());
    }
    {
        // families: the wide Rayleigh-Ritz / repair Grams (64 x 64 tiles), the dense operator's
        // A x (128 x 32 tiles over the stored A^T), and the small tiled Grams
        int amx = 0, bmx = 0;
        for (int j = 0; j < njobs; ++j) {
            amx = std::max(amx, jobs[j].a.cols());
            bmx = std::max(bmx, jobs[j].b.cols());
        }
        const char* fam = shape_family((BM == 64 && BN == 64) ? "gram_wide" : "gram", amx, bmx, prm.sym[0] != 0, njobs);
        LaunchScope ls(fam, bytes, flops);
        dim3 grid(max_tiles, prm.splits, njobs);
        k_gram<BM, BN, WM, WN, GBK, GST><<<grid, NT, smem, rt.stream()>>>(prm);
        BOSP_LAUNCH_CHECK();
    }
    if (prm.splits > 1) {
        LaunchScope ls("gram_reduce");
        const int64_t total = static_cast<int64_t>(max_tiles) * BM * BN;
        dim3 grid(static_cast<unsigned>((total + kRedElems - 1) / kRedElems), 1, njobs);
        k_gram_reduce<BM, BN><<<grid, kRedElems * kRedGroups, 0, rt.stream()>>>(prm);
        BOSP_LAUNCH_CHECK();
    }
}

// ------------------------------------------------------------------------------------------
// Skinny Gram (a, b <= 32): DMMA fragments straight from global memory
// ------------------------------------------------------------------------------------------
// For G = A^T B the n rows are the MMA's k dimension: the A fragment of m8n8k4 (8 x 4, row i =
// column m0+i of A, entry kk = row k0+kk) is one double per lane, A[k0 + (lane&3), m0 + lane/4]
// -- a warp reads 8 columns x 4 consecutive rows, eight full 32-byte sectors.  No shared-memory
// staging and tiles padded to 8 (not 32) columns: a 20 x 20 Gram issues 9 DMMAs per 4 rows
// instead of 16.  Each warp walks its own 4-row steps; warps fold through shared memory in a
// fixed order, blocks through the split-K partial buffer (k_gram_reduce, 32 x 32 layout).
constexpr int kRegWarps = 8;
// k-steps per iteration of the register Gram: ~16 independent fragments in flight per lane,
// even (k-steps come in pairs from one 16-byte load)
// single-group layouts wider than 4 x 4 fragment tiles fold the warps sequentially
template <int G, int MS, int NS>
constexpr bool kGramSeqFold = G == 1 && MS * NS > 16;
template <int F>
constexpr int kGramU = (16 / F) < 2 ? 2 : (16 / F) > 8 ? 8 : ((16 / F) & ~1);

template <int MT, int NTL, int GM, int GN>
__global__ void __launch_bounds__(kRegWarps * 32) k_gram_regs(GramParams prm) {
    // GM x GN warp groups split the MT x NTL fragment tiles (each warp holds MS x NS of them);
    // the warps of a group walk alternate 4-row steps.  GM = GN = 1: every warp the whole tile.
    constexpr int G = GM * GN, WPG = kRegWarps / G;
    constexpr int MS = (MT + GM - 1) / GM, NS = (NTL + GN - 1) / GN;
    constexpr int TM = MT * 8, TN = NTL * 8, SM = MS * 8, SN = NS * 8;
    constexpr int LDP = (TM <= 32 && TN <= 32) ? 32 : 64;  // k_gram_reduce<LDP, LDP> layout
    extern __shared__ __align__(16) double red[];  // [warp][SM x SN]
    const int jb = blockIdx.y;
    const GramJob& job = prm.job[jb];
    const int acols = job.a.cols(), bcols = job.b.cols();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int grp = warp / WPG, wig = warp - grp * WPG;
    const int gm = grp / GN, gn = grp - gm * GN;
    const double* pa[MS];
    const double* pb[NS];
#pragma unroll
    for (int i = 0; i < MS; ++i) {
        const int c = (gm * MS + i) * 8 + gid;
        pa[i] = c < acols ? colptr(job.a, c) : nullptr;
    }
#pragma unroll
    for (int j = 0; j < NS; ++j) {
        const int c = (gn * NS + j) * 8 + gid;
        pb[j] = c < bcols ? colptr(job.b, c) : nullptr;
    }
    double acc[MS][NS][2];
#pragma unroll
    for (int i = 0; i < MS; ++i)
#pragma unroll
        for (int j = 0; j < NS; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int64_t kb = static_cast<int64_t>(blockIdx.x) * prm.chunk;
    const bool sym = prm.sym[jb] != 0;
    // symmetric job: a warp group wholly below the diagonal has nothing to compute
    const int64_t ke = (sym && gm > gn) ? kb : min(prm.n, kb + prm.chunk);
    const bool same_ab = sym && prm.same[jb] && gm == gn;
    // U 4-row k-steps per iteration (U even), every load issued before the first DMMA.  The
    // Gram sums over rows in any order, so a k-step need not be 4 consecutive rows: lane tig
    // loads rows (2 tig, 2 tig + 1) of each 8-row block as one 16-byte load and feeds .x to
    // k-step u, .y to k-step u + 1 (A and B paired identically) -- half the load instructions,
    // and each warp load covers 64 contiguous bytes of 8 columns.
    constexpr int U = kGramU<MS + NS>;
    for (int64_t k0 = kb + 4 * U * wig; k0 < ke; k0 += 4 * U * WPG) {
        double af[U][MS], bf[U][NS];
#pragma unroll
        for (int u = 0; u < U; u += 2) {
            const int64_t r = k0 + 4 * u + 2 * tig;
            const bool v2 = r + 1 < ke, v1 = r < ke;
#pragma unroll
            for (int i = 0; i < MS; ++i) {
                double2 t = make_double2(0.0, 0.0);
                if (pa[i] && v2) t = __ldg(reinterpret_cast<const double2*>(pa[i] + r));
                else if (pa[i] && v1) t.x = __ldg(pa[i] + r);
                af[u][i] = t.x;
                af[u + 1][i] = t.y;
            }
            if constexpr (MS == NS) {
                if (same_ab) {  // G = A^T A on the diagonal group: B fragments are the A fragments
#pragma unroll
                    for (int j = 0; j < NS; ++j) {
                        bf[u][j] = af[u][j];
                        bf[u + 1][j] = af[u + 1][j];
                    }
                    continue;
                }
            }
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                double2 t = make_double2(0.0, 0.0);
                if (pb[j] && v2) t = __ldg(reinterpret_cast<const double2*>(pb[j] + r));
                else if (pb[j] && v1) t.x = __ldg(pb[j] + r);
                bf[u][j] = t.x;
                bf[u + 1][j] = t.y;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < MS; ++i)
#pragma unroll
                for (int j = 0; j < NS; ++j)
                    if ((!sym || gm * MS + i <= gn * NS + j) && (gm * MS + i) * 8 < acols &&
                        (gn * NS + j) * 8 < bcols)  // skip pairs of all-padding fragment tiles
                        dmma(acc[i][j][0], acc[i][j][1], af[u][i], bf[u][j]);
    }
    if constexpr (kGramSeqFold<G, MS, NS>) {
        // wide single-group tiles: warps add into one tile in warp order (same fixed order as
        // the per-warp buffers, 1/8 of the shared memory)
        for (int w = 0; w < kRegWarps; ++w) {
            if (warp == w) {
#pragma unroll
                for (int i = 0; i < MS; ++i)
#pragma unroll
                    for (int j = 0; j < NS; ++j) {
                        const int m = i * 8 + gid, nn = j * 8 + 2 * tig;
                        red[m + nn * SM] = (w == 0 ? 0.0 : red[m + nn * SM]) + acc[i][j][0];
                        red[m + (nn + 1) * SM] = (w == 0 ? 0.0 : red[m + (nn + 1) * SM]) + acc[i][j][1];
                    }
            }
            __syncthreads();
        }
    } else {
        double* mine = red + warp * (SM * SN);
#pragma unroll
        for (int i = 0; i < MS; ++i)
#pragma unroll
            for (int j = 0; j < NS; ++j) {
                const int m = i * 8 + gid, nn = j * 8 + 2 * tig;
                mine[m + nn * SM] = acc[i][j][0];
                mine[m + (nn + 1) * SM] = acc[i][j][1];
            }
        __syncthreads();
    }
    double* part = prm.partial + jb * prm.job_stride + static_cast<int64_t>(blockIdx.x) * (LDP * LDP);
    for (int e = threadIdx.x; e < TM * TN; e += kRegWarps * 32) {
        const int m = e % TM, nn = e / TM;
        const int om = m / SM, on = nn / SN;  // owning group
        double v = 0.0;
        if constexpr (kGramSeqFold<G, MS, NS>) {
            v = red[m + nn * SM];
        } else if (om < GM && on < GN) {
            const int g = om * GN + on, loc = (m - om * SM) + (nn - on * SN) * SM;
#pragma unroll
            for (int w = 0; w < WPG; ++w) v += red[(g * WPG + w) * (SM * SN) + loc];
        }
        if (prm.splits == 1) {
            if (m < acols && nn < bcols) gram_store(job, sym, m, nn, v);
        } else {
            part[m + nn * LDP] = v;
        }
    }
}

template <int MT, int NTL, int GM = 1, int GN = 1>
void launch_gram_regs(const GramJob* jobs, int njobs, int64_t n) {
    constexpr int LDP = (MT * 8 <= 32 && NTL * 8 <= 32) ? 32 : 64;
    constexpr int MS = (MT + GM - 1) / GM, NS = (NTL + GN - 1) / GN;
    constexpr int WPG = kRegWarps / (GM * GN);
    Runtime& rt = Runtime::get();
    GramParams prm{};
    for (int j = 0; j < njobs; ++j) {
        prm.job[j] = jobs[j];
        prm.tiles_n[j] = 1;
        prm.tiles[j] = 1;
        prm.sym[j] = jobs[j].sym && MT == NTL && GM == GN;
        prm.same[j] = prm.sym[j] && same_columns(jobs[j].a, jobs[j].b);
    }
    prm.n = n;
    constexpr int U = kGramU<MS + NS>;
    constexpr int64_t kStep = 4 * U * WPG;  // rows per warp-group iteration
    const int64_t steps = (n + 4 * kRegWarps - 1) / (4 * kRegWarps);
    // one full wave of resident blocks (2 per SM at ~100 registers, 1 for the wide symmetric
    // layouts); 3-8 waves measured 30-100 % slower on config 2's 20-column Grams (more partials,
    // tail).  BOSP_GRAM_WAVES overrides the blocks per SM.
    constexpr size_t smem_need = sizeof(double) * (kGramSeqFold<GM * GN, MS, NS> ? 1 : kRegWarps) * MS * 8 * NS * 8;
    static int resident[64] = {0};
    if (resident[rt.device() & 63] == 0) {
        int r = 0;
        BOSP_CUDA(cudaFuncSetAttribute(k_gram_regs<MT, NTL, GM, GN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_need)));
        BOSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_gram_regs<MT, NTL, GM, GN>, kRegWarps * 32,
                                                                smem_need));
        resident[rt.device() & 63] = std::max(1, std::min(r, 2));
    }
    const int64_t waves = resident[rt.device() & 63];
    int splits = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(
        (waves * rt.sm_count() + njobs - 1) / njobs, steps / 8)));  // >= 8 steps of work per block
    const int64_t per = ((n + splits - 1) / splits + kStep - 1) / kStep;
    prm.chunk = per * kStep;
    splits = static_cast<int>((n + prm.chunk - 1) / prm.chunk);
    prm.splits = std::max(1, splits);
    prm.job_stride = static_cast<int64_t>(prm.splits) * LDP * LDP;
    prm.partial = rt.scratch(static_cast<size_t>(prm.job_stride) * njobs);
    constexpr size_t smem = sizeof(double) * (kGramSeqFold<GM * GN, MS, NS> ? 1 : kRegWarps) * MS * 8 * NS * 8;
    static unsigned attr_mask = 0;
    rt.once_per_device(attr_mask, [&] { BOSP_CUDA(cudaFuncSetAttribute(k_gram_regs<MT, NTL, GM, GN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem))); });
    double flops = 0.0, bytes = 0.0;
    for (int j = 0; j < njobs; ++j) {
        flops += 2.0 * n * jobs[j].a.cols() * jobs[j].b.cols() * (prm.sym[j] ? 0.5 : 1.0);
        bytes += 8.0 * n * (same_columns(jobs[j].a, jobs[j].b) ? jobs[j].a.cols() : jobs[j].a.cols() + jobs[j].b.cols());
    }
    {
        LaunchScope ls("gram", bytes, flops);
        k_gram_regs<MT, NTL, GM, GN><<<dim3(prm.splits, njobs), kRegWarps * 32, smem, rt.stream()>>>(prm);
        BOSP_LAUNCH_CHECK();
    }
    if (prm.splits > 1) {
        LaunchScope ls("gram_reduce");
        dim3 grid(static_cast<unsigned>(LDP * LDP / kRedElems), 1, njobs);
        k_gram_reduce<LDP, LDP><<<grid, kRedElems * kRedGroups, 0, rt.stream()>>>(prm);
        BOSP_LAUNCH_CHECK();
    }
}


// ------------------------------------------------------------------------------------------
// Product kernel
// ------------------------------------------------------------------------------------------
// The product streams A from L2 (every column tile of Out re-reads the same row tile), so a
// shallower stage (16 k) with 3 stages keeps 3 blocks per SM instead of 2: measured 24.6 ->
// 29.0 TF/s at n = 2^21, k = b = 320 (the Gram, streaming fresh rows from HBM, keeps 3 x 32).
#ifndef BOSP_PSTAGES
#define BOSP_PSTAGES 3
#endif
#ifndef BOSP_PBK
#define BOSP_PBK 16
#endif
constexpr int kPStages = BOSP_PSTAGES;
constexpr int kPBK = BOSP_PBK;
constexpr int kProdTab = 1024;  // A column pointers kept in shared memory (wider K: per-stage lookup)

struct ProductParams {
    ProductJob job[4];
    int64_t n;
    int tiles_n[4];
    int64_t tiles[4];
    int16_t kend[4][16];  // per column tile: K rows of C that can be nonzero (0 = all)
};

template <int BM, int BN, int WM, int WN, int PBK = kPBK, int PST = kPStages>
__global__ void __launch_bounds__(WM * WN * 32)
k_product(ProductParams prm) {
    constexpr int kPBK = PBK, kPStages = PST, kPLdK = PBK + 4;
    constexpr int NT = WM * WN * 32;
    constexpr int WTM = BM / WM, WTN = BN / WN;
    constexpr int MT = WTM / 8, NTL = WTN / 8;
    constexpr int LdM = BM + 4;
    extern __shared__ __align__(16) double smem[];
    double* sa = smem;                        // [kPStages][kPBK][LdM]
    double* sb = smem + kPStages * kPBK * LdM;  // [kPStages][BN][kPLdK]

    const int jb = blockIdx.z;
    const ProductJob& job = prm.job[jb];
    const int64_t tile = blockIdx.x + static_cast<int64_t>(blockIdx.y) * gridDim.x;
    if (tile >= prm.tiles[jb]) return;
    const int tn = static_cast<int>(tile % prm.tiles_n[jb]);
    const int64_t tm = tile / prm.tiles_n[jb];
    const int64_t m0 = tm * BM;
    const int n0 = tn * BN;
    // structured C (triangular coefficients): the K loop stops at the tile's last nonzero row
    const int kend = tn < 16 ? prm.kend[jb][tn] : 0;
    const int kcols = kend > 0 ? min(job.a.cols(), kend) : job.a.cols();
    ColList cl;  // C as a one-segment list (k-contiguous columns)
    cl.p[0] = job.c;
    cl.ld[0] = job.ldc;
    cl.start[1] = job.ncols;
    cl.nseg = 1;
    for (int i = 2; i <= kMaxSeg; ++i) cl.start[i] = job.ncols;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int wm0 = (warp / WN) * WTM, wn0 = (warp % WN) * WTN;

    double acc[MT][NTL][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int nk = (kcols + kPBK - 1) / kPBK;
    // column base pointers of A for the whole K range (a table in shared memory, behind the
    // pipeline buffers), so the stage loads never search the ColList segments
    const double** coltab = reinterpret_cast<const double**>(smem + kPStages * (kPBK * LdM + BN * kPLdK));
    const bool tab = kcols <= kProdTab;
    if (tab) {
        for (int c = threadIdx.x; c < kcols; c += NT) coltab[c] = colptr(job.a, c);
        __syncthreads();
    }
    McontigLoader<BM, NT, kPBK> lda;
    lda.init(job.a.p[0], m0, prm.n);
    KcontigLoader<BN, NT, kPBK> ldb;
    ldb.init(cl, n0, job.ncols);
    auto load_stage = [&](int st, int s) {
        if (tab) lda.load(sa + st * kPBK * LdM, coltab, s * kPBK, kcols);
        else load_mcontig<BM, NT, kPBK>(sa + st * kPBK * LdM, job.a, s * kPBK, kcols, m0, prm.n);
        ldb.load(sb + st * BN * kPLdK, s * kPBK, kcols);
    };
#pragma unroll
    for (int s = 0; s < kPStages - 1; ++s) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        cp_async_wait<kPStages - 2>();
        __syncthreads();
        const int st = it % kPStages;
        const double* a = sa + st * kPBK * LdM;
        const double* b = sb + st * BN * kPLdK;
#pragma unroll
        for (int kk = 0; kk < kPBK; kk += 4) {
            double af[MT], bf[NTL];
#pragma unroll
            for (int i = 0; i < MT; ++i) af[i] = a[(kk + tig) * LdM + wm0 + i * 8 + gid];
#pragma unroll
            for (int j = 0; j < NTL; ++j) bf[j] = b[(wn0 + j * 8 + gid) * kPLdK + kk + tig];
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NTL; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        const int nxt = it + kPStages - 1;
        if (nxt < nk) load_stage(nxt % kPStages, nxt);
        cp_async_commit();
    }
    cp_async_wait<0>();
    __syncthreads();

    // Epilogue through shared memory so that every column of Out is written as one contiguous
    // BM-row run: so[n * LdM + m].
    double* so = smem;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j) {
            const int m = wm0 + i * 8 + gid;
            const int nn = wn0 + j * 8 + 2 * tig;
            so[nn * LdM + m] = acc[i][j][0];
            so[(nn + 1) * LdM + m] = acc[i][j][1];
        }
    __syncthreads();
    const double alpha = job.alpha, beta = job.beta;
    if ((job.ldo & 1) == 0 && (reinterpret_cast<uintptr_t>(job.out) & 15) == 0) {
        // row pairs as 16-byte accesses, 4 pairs per thread and round with every load of Out
        // (beta != 0) issued before the first store (a scalar load -> store chain per element
        // left the epilogue latency bound)
        constexpr int kPairs = BM * BN / 2, kU = 4;
        for (int q0 = threadIdx.x; q0 < kPairs; q0 += NT * kU) {
            double2 old[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int q = q0 + u * NT;
                const int m = 2 * (q % (BM / 2)), nn = q / (BM / 2);
                const int64_t gm = m0 + m;
                const int gn = n0 + nn;
                old[u] = make_double2(0.0, 0.0);
                if (beta != 0.0 && q < kPairs && gn < job.ncols) {
                    const double* o = job.out + gn * job.ldo + gm;
                    if (gm + 1 < prm.n) old[u] = *reinterpret_cast<const double2*>(o);
                    else if (gm < prm.n) old[u].x = *o;
                }
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const int q = q0 + u * NT;
                if (q >= kPairs) continue;
                const int m = 2 * (q % (BM / 2)), nn = q / (BM / 2);
                const int64_t gm = m0 + m;
                const int gn = n0 + nn;
                if (gn >= job.ncols || gm >= prm.n) continue;
                double* o = job.out + gn * job.ldo + gm;
                const double v0 = alpha * so[nn * LdM + m], v1 = alpha * so[nn * LdM + m + 1];
                const double r0 = beta == 0.0 ? v0 : v0 + beta * old[u].x;
                const double r1 = beta == 0.0 ? v1 : v1 + beta * old[u].y;
                if (gm + 1 < prm.n) *reinterpret_cast<double2*>(o) = make_double2(r0, r1);
                else *o = r0;
            }
        }
        return;
    }
    for (int e = threadIdx.x; e < BM * BN; e += NT) {
        const int m = e % BM, nn = e / BM;
        const int64_t gm = m0 + m;
        const int gn = n0 + nn;
        if (gm < prm.n && gn < job.ncols) {
            double* o = job.out + gn * job.ldo + gm;
            const double v = alpha * so[nn * LdM + m];
            *o = (beta == 0.0) ? v : v + beta * *o;
        }
    }
}


template <int BM, int BN, int WM, int WN, int PBK = kPBK, int PST = kPStages>
void launch_product(const ProductJob* jobs, int njobs, int64_t n) {
    constexpr int kPBK = PBK, kPStages = PST, kPLdK = PBK + 4;
    Runtime& rt = Runtime::get();
    ProductParams prm{};
    int64_t max_tiles = 0;
    double flops = 0, bytes = 0;
    for (int j = 0; j < njobs; ++j) {
        prm.job[j] = jobs[j];
        prm.tiles_n[j] = (jobs[j].ncols + BN - 1) / BN;
        prm.tiles[j] = ((n + BM - 1) / BM) * prm.tiles_n[j];
        max_tiles = std::max(max_tiles, prm.tiles[j]);
        if (jobs[j].col_kend && prm.tiles_n[j] <= 16) {
            for (int t = 0; t < prm.tiles_n[j]; ++t) {
                int ke = 1;
                for (int c = t * BN; c < std::min(jobs[j].ncols, (t + 1) * BN); ++c) ke = std::max(ke, jobs[j].col_kend[c]);
                prm.kend[j][t] = static_cast<int16_t>(std::min(ke, 32767));
            }
        }
        const double k = jobs[j].a.cols(), b = jobs[j].ncols;
        flops += 2.0 * n * k * b;
        bytes += 8.0 * n * (k + b * (jobs[j].beta != 0.0 ? 2.0 : 1.0));
    }
    prm.n = n;
    constexpr int NT = WM * WN * 32;
    constexpr size_t smem_pipe = sizeof(double) * (kPStages * (kPBK * (BM + 4) + BN * kPLdK) + kProdTab);
    constexpr size_t smem_epi = sizeof(double) * BN * (BM + 4);
    constexpr size_t smem = smem_pipe > smem_epi ? smem_pipe : smem_epi;
    static unsigned attr_mask = 0;
    rt.once_per_device(attr_mask, [&] { BOSP_CUDA(cudaFuncSetAttribute(k_product<BM, BN, WM, WN, PBK, PST>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); });
    int kmx = 0, bmx = 0;
    for (int j = 0; j < njobs; ++j) {
        kmx = std::max(kmx, jobs[j].a.cols());
        bmx = std::max(bmx, jobs[j].ncols);
    }
    LaunchScope ls(shape_family("product_wide", kmx, bmx, jobs[0].col_kend != nullptr, njobs), bytes, flops);
    const unsigned gx = static_cast<unsigned>(std::min<int64_t>(max_tiles, 65535));
    const unsigned gy = static_cast<unsigned>((max_tiles + gx - 1) / gx);
    dim3 grid(gx, gy, njobs);
    k_product<BM, BN, WM, WN, PBK, PST><<<grid, NT, smem, rt.stream()>>>(prm);
    BOSP_LAUNCH_CHECK();
}

// ------------------------------------------------------------------------------------------
// Skinny product: k <= 64 and b <= 64 (the Ritz pullbacks, Step-5 P~/Q~, biorth_against and
// MGS applications at the configs' widths).  HBM-bound: A streams once.  Each CTA keeps the
// whole C (k x BN) in shared memory and walks row tiles of 128 rows (grid-stride, persistent),
// double-buffering the next A tile with cp.async while the DMMA pipe works on the current one.
// BN is b rounded up to 8 so no tensor work is spent on padding columns.
// ------------------------------------------------------------------------------------------

struct SkinnyParams {
    ProductJob job[4];
    int64_t n;
    int64_t tiles;
    int kp;     // k rounded up to 4 (max over jobs)
    int ldc;    // smem ld of C (== 4 mod 16)
};

template <int BN, int RT>
__global__ void __launch_bounds__(256) k_product_skinny(SkinnyParams prm) {
    constexpr int NT = BN / 8;
    constexpr int kSkBM = 64 * RT, kSkLdM = kSkBM + 4;  // rows per tile: 8 warps x RT m-tiles
    extern __shared__ __align__(16) double smem[];
    const int kp = prm.kp, ldc = prm.ldc;
    double* sc = smem;                                // [BN][ldc]
    double* sa = smem + BN * ldc;                     // [2][kp][kSkLdM]
    const ProductJob& job = prm.job[blockIdx.z];
    const int kcols = job.a.cols();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;

    // C -> shared (zero-padded to kp x BN)
    {
        ColList cl;
        cl.p[0] = job.c;
        cl.ld[0] = job.ldc;
        cl.start[1] = job.ncols;
        cl.nseg = 1;
        for (int i = 2; i <= kMaxSeg; ++i) cl.start[i] = job.ncols;
        const int chunks = BN * (kp / 2);
        for (int ch = threadIdx.x; ch < chunks; ch += 256) {
            const int c = ch / (kp / 2), k2 = 2 * (ch % (kp / 2));
            int bytes = 0;
            const double* src = job.c;
            if (c < job.ncols && k2 < kcols) {
                bytes = (kcols - k2) >= 2 ? 16 : 8;
                src = colptr(cl, c) + k2;
            }
            cp_async16(sc + c * ldc + k2, src, bytes);
        }
    }
    auto load_a = [&](int buf, int64_t tile) {
        double* dst = sa + buf * kp * kSkLdM;
        const int64_t m0 = tile * kSkBM;
        const int chunks = kp * (kSkBM / 2);
        for (int ch = threadIdx.x; ch < chunks; ch += 256) {
            const int kk = ch / (kSkBM / 2), m2 = 2 * (ch % (kSkBM / 2));
            const int64_t m = m0 + m2;
            int bytes = 0;
            const double* src = job.c;
            if (kk < kcols && m < prm.n) {
                bytes = (prm.n - m) >= 2 ? 16 : 8;
                src = colptr(job.a, kk) + m;
            }
            cp_async16(dst + kk * kSkLdM + m2, src, bytes);
        }
    };
    int64_t tile = blockIdx.x;
    if (tile < prm.tiles) load_a(0, tile);
    cp_async_commit();
    int buf = 0;
    for (; tile < prm.tiles; tile += gridDim.x, buf ^= 1) {
        const int64_t next = tile + gridDim.x;
        if (next < prm.tiles) load_a(buf ^ 1, next);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double* a = sa + buf * kp * kSkLdM;
        const int wm0 = warp * 8 * RT;
        const double alpha = job.alpha, beta = job.beta;
        const int64_t r0 = tile * kSkBM + wm0 + gid;
        // beta != 0: issue the loads of Out now so their latency hides under the DMMA loop
        double old[RT][NT][2];
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int64_t row = r0 + i * 8;
                    const int col = j * 8 + 2 * tig + h;
                    old[i][j][h] = (beta != 0.0 && row < prm.n && col < job.ncols)
                                       ? __ldcs(job.out + static_cast<int64_t>(col) * job.ldo + row)
                                       : 0.0;
                }
        double acc[RT][NT][2];
#pragma unroll
        for (int i = 0; i < RT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int kk = 0; kk < kp; kk += 4) {
            double af[RT], bf[NT];
#pragma unroll
            for (int i = 0; i < RT; ++i) af[i] = a[(kk + tig) * kSkLdM + wm0 + i * 8 + gid];
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[j] = sc[(j * 8 + gid) * ldc + kk + tig];
#pragma unroll
            for (int i = 0; i < RT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
#pragma unroll
        for (int i = 0; i < RT; ++i) {
            const int64_t row = r0 + i * 8;
            if (row >= prm.n) continue;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = j * 8 + 2 * tig + h;
                    if (col < job.ncols) {
                        const double v = alpha * acc[i][j][h];
                        __stcs(job.out + static_cast<int64_t>(col) * job.ldo + row,
                               beta == 0.0 ? v : v + beta * old[i][j][h]);
                    }
                }
        }
        __syncthreads();  // everyone is done with `buf` before it is refilled
    }
    cp_async_wait<0>();
}

template <int BN, int RT>
void launch_skinny_rt(const ProductJob* jobs, int njobs, int64_t n);

template <int BN>
void launch_skinny(const ProductJob* jobs, int njobs, int64_t n) {
    // one m-tile per warp (64-row tiles, ~half the shared memory, 2+ blocks per SM) measured
    // 20-30 % faster than two for C widths >= 16 on config 2's shapes; width 8 keeps two
    if (BN > 8) return launch_skinny_rt<BN, 1>(jobs, njobs, n);
    return launch_skinny_rt<BN, 2>(jobs, njobs, n);
}

template <int BN, int RT>
void launch_skinny_rt(const ProductJob* jobs, int njobs, int64_t n) {
    constexpr int kSkBM = 64 * RT, kSkLdM = kSkBM + 4;
    Runtime& rt = Runtime::get();
    SkinnyParams prm{};
    int kmax = 0;
    double flops = 0, bytes = 0;
    for (int j = 0; j < njobs; ++j) {
        prm.job[j] = jobs[j];
        kmax = std::max(kmax, jobs[j].a.cols());
        const double k = jobs[j].a.cols(), b = jobs[j].ncols;
        flops += 2.0 * n * k * b;
        bytes += 8.0 * n * (k + b * (jobs[j].beta != 0.0 ? 2.0 : 1.0));
    }
    prm.n = n;
    prm.tiles = (n + kSkBM - 1) / kSkBM;
    prm.kp = std::max(4, (kmax + 3) / 4 * 4);
    prm.ldc = (prm.kp + 15) / 16 * 16 + 4;
    const size_t smem = sizeof(double) * (static_cast<size_t>(BN) * prm.ldc + 2ull * prm.kp * kSkLdM);
    static unsigned attr_mask = 0;
    rt.once_per_device(attr_mask, [&] { BOSP_CUDA(cudaFuncSetAttribute(k_product_skinny<BN, RT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)); });
    int per_sm = 1;
    BOSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_product_skinny<BN, RT>, 256, smem));
    const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(prm.tiles, int64_t(std::max(per_sm, 1)) * rt.sm_count()));
    int bmx = 0;
    for (int j = 0; j < njobs; ++j) bmx = std::max(bmx, jobs[j].ncols);
    LaunchScope ls(shape_family("product", kmax, bmx, jobs[0].beta != 0.0, njobs), bytes, flops);
    dim3 grid(static_cast<unsigned>(ctas), 1, njobs);
    k_product_skinny<BN, RT><<<grid, 256, smem, rt.stream()>>>(prm);
    BOSP_LAUNCH_CHECK();
}


// ------------------------------------------------------------------------------------------
// TMA-staged skinny Grams: the MGS-Biorth pair Gram Z^T Z of Z = [X | Y]
// ------------------------------------------------------------------------------------------
// One persistent CTA per SM owns a contiguous range of R-row stages.  A producer warp lands a
// stage of every column segment with ONE tensor-map TMA load per segment (cp.async.bulk.tensor,
// completion counted in bytes on the stage's "full" mbarrier), several stages deep; eight
// consumer warps take alternate 4-row k-steps of a stage, load one fragment double per 8-column
// block from shared memory and issue the upper fragment pairs on the DMMA pipe (for G = Z^T Z the
// B fragment of a block is its A fragment), then arrive on the stage's "empty" mbarrier, which
// releases the slot to the producer -- no CTA-wide barrier in the main loop.
//
// The tensor maps are 3-D views of a column-major segment: (16 rows, columns, row groups of 16)
// with strides (8 B, ld * 8 B, 128 B) and the 128-byte swizzle.  A stage box (16, c, R / 16)
// lands as 128-byte lines [row group][column] of 16 rows each, the 16-byte chunks of line L
// XOR-permuted by (L mod 8); a fragment load (4 rows x 8 consecutive columns = 8 lines) then
// spreads over the banks (at most 2-way per half-warp), while every TMA line is a full 128-byte
// L2 line of one column.  (Measured on the way there: one 1-D cp.async.bulk per column and stage
// capped an SM at ~19 requests/us, 2.9 TB/s; 32- and 64-byte lines without swizzle, 1.1-2.2
// TB/s from DRAM.)  Rows past n are zero-filled by the TMA unit (out-of-bounds row groups); n
// must be a multiple of 16.  Warps fold in order, CTAs through k_gram_reduce: deterministic.
constexpr int kTmaWarps = 8;   // consumer warps; warp kTmaWarps is the producer
constexpr int kTmaMaxSt = 8;   // pipeline depth bound
constexpr int kTmaSeg = 4;     // tensor maps (column segments) per operand set
constexpr int kTmaQ = 16;      // rows per 128-byte swizzled line

// Byte offset of element `rr` (0..15) of 128-byte line `line` under the 128-byte swizzle: the
// 16-byte chunk index XOR (absolute line mod 8); bl = the buffer base's line mod 8.
__device__ __forceinline__ int swz(int line, int rr, int bl) {
    return line * 128 + ((((rr >> 1) ^ (line + bl)) & 7) << 4) + ((rr & 1) << 3);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// 3-D tiled TMA load of box (16, cols, groups) at coordinates (0, 0, group0)
__device__ __forceinline__ void tma_load3(void* dst, const CUtensorMap* map, int group0, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(0), "r"(0), "r"(group0), "r"(smem_u32(bar))
        : "memory");
}

// One segment set: up to kTmaSeg column segments (tensor maps), each `cols` wide, consecutive
// in the stage buffer.
struct TmaSegs {
    CUtensorMap map[kTmaSeg];
    int cols[kTmaSeg];
    int off[kTmaSeg];  // box offset in the stage buffer (doubles, 1024-byte aligned)
    int stage;         // doubles per stage buffer
    int nseg;
};

// Encode the 3-D view (qr rows, cols, n / qr row groups) of a column-major segment with a
// (qr, cols, rows / qr) box, 128-byte swizzle; false when the driver cannot encode it.
bool encode_seg(CUtensorMap* m, const double* p, int64_t ld, int64_t n, int cols, int qr, int rows) {
    using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    static const Fn fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            f = nullptr;
        }
        return reinterpret_cast<Fn>(f);
    }();
    if (!fn) return false;  // no driver entry point: the callers use their cp.async kernels
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(qr), static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(n / qr)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 8u, static_cast<cuuint64_t>(qr) * 8u};
    const cuuint32_t box[3] = {static_cast<cuuint32_t>(qr), static_cast<cuuint32_t>(cols), static_cast<cuuint32_t>(rows / qr)};
    const cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(p), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The segments of a ColList as tensor maps; false when TMA cannot stage it (n % 16, alignment,
// > kTmaSeg segments).  Each segment's box starts 1024-byte aligned in the stage buffer:
// t.off[s] (doubles), t.stage (doubles per stage).
bool make_segs(TmaSegs& t, const ColList& cl, int64_t n, int rows) {
    if (n % kTmaQ != 0 || n < kTmaQ || cl.nseg > kTmaSeg || n / kTmaQ > (1LL << 32)) return false;
    t.nseg = cl.nseg;
    int off = 0;
    for (int s = 0; s < cl.nseg; ++s) {
        const int cols = cl.start[s + 1] - cl.start[s];
        if ((reinterpret_cast<uintptr_t>(cl.p[s]) & 15) || ((cl.ld[s] * 8) & 15) || cols > 256) return false;
        t.cols[s] = cols;
        t.off[s] = off;
        off += (cols * rows + 127) / 128 * 128;  // 1024-byte boundary
        if (!encode_seg(&t.map[s], cl.p[s], cl.ld[s], n, cols, kTmaQ, rows)) return false;
    }
    t.stage = off;
    return true;
}

// Producer side of one stage: arm the full barrier with the stage's bytes, one TMA per segment.
__device__ __forceinline__ void tma_stage(const TmaSegs& t, double* buf, int rows, int64_t stage,
                                          unsigned long long* full) {
    int total = 0;
    for (int s = 0; s < t.nseg; ++s) total += t.cols[s];
    mbar_expect_tx(full, static_cast<unsigned>(rows) * 8u * static_cast<unsigned>(total));
    for (int s = 0; s < t.nseg; ++s)
        tma_load3(buf + t.off[s], &t.map[s], static_cast<int>(stage * (rows / kTmaQ)), full);
}

struct GramTmaParams {
    TmaSegs seg;
    GramJob job;
    int64_t n;
    int64_t stages;     // R-row stages (the last one may be partial: TMA zero-fills)
    int R, nst;         // rows per stage, pipeline depth
    int ncols;          // real columns (a == b)
    int ldp;            // partial layout (k_gram_reduce<ldp, ldp>)
    double* partial;
};

template <int F>
__global__ void __launch_bounds__((kTmaWarps + 1) * 32, 1) k_gram_tma(const __grid_constant__ GramTmaParams prm) {
    constexpr int C = F * 8, NP = F * (F + 1) / 2;
    extern __shared__ __align__(1024) double sm[];
    __shared__ __align__(8) unsigned long long full_bar[kTmaMaxSt], empty_bar[kTmaMaxSt];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int R = prm.R, NST = prm.nst, stage_d = prm.seg.stage;
    const int64_t s0 = prm.stages * blockIdx.x / gridDim.x, s1 = prm.stages * (blockIdx.x + 1) / gridDim.x;
    const int64_t mine = s1 - s0;
    const int nc = prm.ncols;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&empty_bar[i], kTmaWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // per fragment block: this lane's first line (bytes / 128, within a stage) and the lines per
    // row group of its segment; padding columns (past nc) read as zero
    int fline[F], fstr[F];
    bool fpad[F];
#pragma unroll
    for (int i = 0; i < F; ++i) {
        int c = i * 8 + gid, s = 0;
        while (s < prm.seg.nseg && c >= prm.seg.cols[s]) c -= prm.seg.cols[s++];
        fpad[i] = s >= prm.seg.nseg;
        fline[i] = fpad[i] ? 0 : prm.seg.off[s] / 16 + c;
        fstr[i] = fpad[i] ? 0 : prm.seg.cols[s];
    }
    const int bl = static_cast<int>(smem_u32(sm) >> 7) & 7;
    __syncthreads();
    double acc[NP][2];
#pragma unroll
    for (int t = 0; t < NP; ++t) acc[t][0] = acc[t][1] = 0.0;
    if (warp == kTmaWarps) {
        if (lane == 0) {
            int slot = 0, round = 0;
            for (int64_t k = 0; k < mine; ++k) {
                if (round > 0) mbar_wait(&empty_bar[slot], static_cast<unsigned>((round - 1) & 1));
                tma_stage(prm.seg, sm + slot * stage_d, R, s0 + k, &full_bar[slot]);
                if (++slot == NST) {
                    slot = 0;
                    ++round;
                }
            }
        }
    } else {
        // A warp takes k-steps warp, warp + 8, ... of every stage, so a lane's swizzled fragment
        // offsets within a stage are fixed: computed once (ncu on the per-step form: 58 % of the
        // kernel's instructions were this address arithmetic, ~100 instructions per 15 DMMAs).
        constexpr int kSteps = 128 / 4 / kTmaWarps;  // k-steps per warp and stage at R = 128
        int foff[F][kSteps];
#pragma unroll
        for (int i = 0; i < F; ++i)
#pragma unroll
            for (int t = 0; t < kSteps; ++t) {
                const int row = (warp + t * kTmaWarps) * 4 + tig, q = row >> 4, rr = row & 15;
                foff[i][t] = swz(fline[i] + q * fstr[i], rr, bl);
            }
        const int nsteps = R / 4 / kTmaWarps;  // 4 (R = 128) or 2 (R = 64)
        int slot = 0;
        unsigned ph = 0;
        for (int64_t k = 0; k < mine; ++k) {
            mbar_wait(&full_bar[slot], ph);
            const char* buf = reinterpret_cast<const char*>(sm + slot * stage_d);
#pragma unroll
            for (int t = 0; t < kSteps; ++t) {
                if (t >= nsteps) break;
                double f[F];
#pragma unroll
                for (int i = 0; i < F; ++i)
                    f[i] = fpad[i] ? 0.0 : *reinterpret_cast<const double*>(buf + foff[i][t]);
                int tt = 0;
#pragma unroll
                for (int i = 0; i < F; ++i)
#pragma unroll
                    for (int j = i; j < F; ++j, ++tt) dmma(acc[tt][0], acc[tt][1], f[i], f[j]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[slot]);
            if (++slot == NST) {
                slot = 0;
                ph ^= 1u;
            }
        }
    }
    __syncthreads();  // the ring is drained
    // fold the consumer warps in order into red[C x C] (upper fragment pairs only)
    double* red = sm;
    for (int w = 0; w < kTmaWarps; ++w) {
        if (warp == w) {
            int t = 0;
#pragma unroll
            for (int i = 0; i < F; ++i)
#pragma unroll
                for (int j = i; j < F; ++j, ++t) {
                    const int m = i * 8 + gid, nn = j * 8 + 2 * tig;
                    red[m + nn * C] = (w == 0 ? 0.0 : red[m + nn * C]) + acc[t][0];
                    red[m + (nn + 1) * C] = (w == 0 ? 0.0 : red[m + (nn + 1) * C]) + acc[t][1];
                }
        }
        __syncthreads();
    }
    double* part = prm.partial + static_cast<int64_t>(blockIdx.x) * prm.ldp * prm.ldp;
    for (int e = threadIdx.x; e < C * C; e += blockDim.x) {
        const int m = e % C, nn = e / C;
        if ((m >> 3) > (nn >> 3)) continue;  // lower fragment tiles were not computed
        if (gridDim.x == 1) {
            if (m < nc && nn < nc) gram_store(prm.job, true, m, nn, red[e]);
        } else {
            part[m + nn * prm.ldp] = red[e];
        }
    }
}

template <int F>
bool launch_gram_tma(const GramJob& job, int64_t n, const CoefParams* coef = nullptr) {
    Runtime& rt = Runtime::get();
    GramTmaParams prm{};
    constexpr int C = F * 8;
    const int sms = rt.sm_count();
    // 128-row stages when every CTA gets >= 24 of them, else 64 (config 2's n = 2^18: 28 each)
    prm.R = (n / 128) >= 24LL * sms ? 128 : 64;
    if (!make_segs(prm.seg, job.a, n, prm.R)) return false;
    prm.job = job;
    prm.n = n;
    prm.ncols = job.a.cols();
    prm.stages = (n + prm.R - 1) / prm.R;
    const size_t stage_b = sizeof(double) * prm.seg.stage;
    prm.nst = static_cast<int>(std::min<size_t>(kTmaMaxSt, (200u * 1024u) / stage_b));
    const size_t smem = std::max(stage_b * prm.nst, sizeof(double) * C * C);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(sms, prm.stages)));
    prm.ldp = C <= 32 ? 32 : 64;
    prm.partial = rt.scratch(static_cast<size_t>(grid) * prm.ldp * prm.ldp);
    static unsigned attr_mask = 0;
    rt.once_per_device(attr_mask, [&] {
        BOSP_CUDA(cudaFuncSetAttribute(k_gram_tma<F>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    });
    const double flops = 1.0 * n * prm.ncols * prm.ncols;  // symmetric: the upper half
    const double bytes = 8.0 * n * prm.ncols;
    {
        LaunchScope ls("gram", bytes, flops);
        k_gram_tma<F><<<grid, (kTmaWarps + 1) * 32, smem, rt.stream()>>>(prm);
        BOSP_LAUNCH_CHECK();
    }
    if (grid > 1) {
        GramParams gp{};
        gp.job[0] = job;
        gp.tiles_n[0] = 1;
        gp.tiles[0] = 1;
        gp.sym[0] = 1;
        gp.splits = grid;
        gp.partial = prm.partial;
        gp.job_stride = static_cast<int64_t>(grid) * prm.ldp * prm.ldp;
        if (coef) {
            LaunchScope ls("gram_reduce");
            if (prm.ldp == 32)
                k_gram_reduce_coef<32><<<dim3(32 * 32 / 32), kCoefThreads, 0, rt.stream()>>>(gp, *coef);
            else
                k_gram_reduce_coef<64><<<dim3(64 * 64 / 32), kCoefThreads, 0, rt.stream()>>>(gp, *coef);
            BOSP_LAUNCH_CHECK();
            return true;
        }
        LaunchScope ls("gram_reduce");
        if (prm.ldp == 32)
            k_gram_reduce<32, 32><<<dim3(32 * 32 / kRedElems, 1, 1), kRedElems * kRedGroups, 0, rt.stream()>>>(gp);
        else
            k_gram_reduce<64, 64><<<dim3(64 * 64 / kRedElems, 1, 1), kRedElems * kRedGroups, 0, rt.stream()>>>(gp);
        BOSP_LAUNCH_CHECK();
    }
    if (coef) coef_mgs_dev(job.g, job.ldg, coef->m, coef->c, coef->ldc, coef->status, coef->drop_tol, coef->cancel_tol);
    return true;
}


void check_aligned(const ColList& cl) {
    for (int s = 0; s < cl.nseg; ++s)
        if ((reinterpret_cast<uintptr_t>(cl.p[s]) & 15) || (cl.ld[s] & 1))
            throw ContractViolation("dmma: operand columns must be 16-byte aligned with even ld");
}

}  // namespace

void gram(const GramJob* jobs, int njobs, int64_t n) {
    require(njobs >= 1 && njobs <= 4, "gram: 1..4 jobs per launch");
    int amax = 0, bmax = 0;
    for (int j = 0; j < njobs; ++j) {
        check_aligned(jobs[j].a);
        check_aligned(jobs[j].b);
        amax = std::max(amax, jobs[j].a.cols());
        bmax = std::max(bmax, jobs[j].b.cols());
    }
    if (amax == 0 || bmax == 0) return;
    if (n == 0) {
        for (int j = 0; j < njobs; ++j)
            for (int c = 0; c < jobs[j].b.cols(); ++c)
                BOSP_CUDA(cudaMemsetAsync(jobs[j].g + c * jobs[j].ldg, 0,
                                          sizeof(double) * jobs[j].a.cols(), Runtime::get().stream()));
        return;
    }
    // register-fragment Grams (n rows = the MMA k dimension, operands straight from global):
    // up to 4 x 4 fragment tiles (32 columns) every warp holds the whole tile; a side wider
    // than 32 is split over two warp groups (a 2 x 1, 1 x 2 or 2 x 2 group layout, each warp
    // <= 4 x 4 tiles); beyond wide_max columns the shared-memory tiled DMMA kernel
    // 48: config 2 is flat between 32 and 64; at 64 the rounding of config 5's 64-wide Grams
    // pushed its (repair-heavy) run into the reference's NumericalAbort path -- 48 converges
    constexpr int lim = 48;
    // one symmetric Gram of <= 64 columns (MGS-Biorth's [X | Y] pair Gram) over many rows:
    // bulk-async staged, one persistent CTA per SM
    // (57-64 columns: 36 fragment pairs of accumulators spill -- the register kernels below)
    if (njobs == 1 && jobs[0].sym && amax == bmax && amax <= 56 && n >= 8192 &&
        same_columns(jobs[0].a, jobs[0].b)) {
        bool done = false;
        switch ((amax + 7) / 8) {
            case 1: done = launch_gram_tma<1>(jobs[0], n); break;
            case 2: done = launch_gram_tma<2>(jobs[0], n); break;
            case 3: done = launch_gram_tma<3>(jobs[0], n); break;
            case 4: done = launch_gram_tma<4>(jobs[0], n); break;
            case 5: done = launch_gram_tma<5>(jobs[0], n); break;
            case 6: done = launch_gram_tma<6>(jobs[0], n); break;
            default: done = launch_gram_tma<7>(jobs[0], n); break;
        }
        if (done) return;
    }
    if (amax <= lim && bmax <= lim) {
        const int mt = (amax + 7) / 8, nt = (bmax + 7) / 8;
        // a symmetric Gram up to 48 columns ([X | Y] of MGS-Biorth, m <= 24): every warp holds
        // all upper fragment pairs and loads each column fragment once (the 2 x 2 group layout
        // re-loads every fragment per group)
        if (njobs == 1 && jobs[0].sym && mt == nt && (mt == 5 || mt == 6))
            return mt == 5 ? launch_gram_regs<5, 5>(jobs, njobs, n) : launch_gram_regs<6, 6>(jobs, njobs, n);
        if (mt <= 4 && nt <= 4) {
            switch (mt * 4 + nt) {
#define BOSP_G(M, N) case M * 4 + N: return launch_gram_regs<M, N>(jobs, njobs, n);
                BOSP_G(1, 1) BOSP_G(1, 2) BOSP_G(1, 3) BOSP_G(1, 4)
                BOSP_G(2, 1) BOSP_G(2, 2) BOSP_G(2, 3) BOSP_G(2, 4)
                BOSP_G(3, 1) BOSP_G(3, 2) BOSP_G(3, 3) BOSP_G(3, 4)
                BOSP_G(4, 1) BOSP_G(4, 2) BOSP_G(4, 3) BOSP_G(4, 4)
#undef BOSP_G
                default: break;
            }
        }
        const int mp = mt <= 4 ? mt : (mt <= 6 ? 6 : 8), np = nt <= 4 ? nt : (nt <= 6 ? 6 : 8);
        switch (mp * 16 + np) {
#define BOSP_A(M, N) case M * 16 + N: return launch_gram_regs<M, N, 2, 1>(jobs, njobs, n);
#define BOSP_B(M, N) case M * 16 + N: return launch_gram_regs<M, N, 1, 2>(jobs, njobs, n);
#define BOSP_C(M, N) case M * 16 + N: return launch_gram_regs<M, N, 2, 2>(jobs, njobs, n);
            BOSP_A(6, 1) BOSP_A(6, 2) BOSP_A(6, 3) BOSP_A(6, 4) BOSP_A(8, 1) BOSP_A(8, 2) BOSP_A(8, 3) BOSP_A(8, 4)
            BOSP_B(1, 6) BOSP_B(2, 6) BOSP_B(3, 6) BOSP_B(4, 6) BOSP_B(1, 8) BOSP_B(2, 8) BOSP_B(3, 8) BOSP_B(4, 8)
            BOSP_C(6, 6) BOSP_C(6, 8) BOSP_C(8, 6) BOSP_C(8, 8)
#undef BOSP_A
#undef BOSP_B
#undef BOSP_C
            default: break;
        }
    }
    if (amax <= 32 && bmax <= 32)
        launch_gram<32, 32, 2, 2>(jobs, njobs, n);
    else if (bmax <= 32 && amax >= 128)
        // many output rows, <= 32 columns (the dense operator's A x = (A^T)^T x at the CG's
        // widths): 128 x 32 tiles, 4 warps of 32 x 32, 4 x 16-row stages, no padding of b to
        // 64 -- n = 16384, 32 columns: 0.71 ms (24.3 TF/s; 2 x 32-row stages 23.7, 8 warps of
        // 32 x 16: 23.0, 256-row tiles 17-22, 64 x 32 tiles: 19-21)
        launch_gram<128, 32, 4, 1, 16, 4>(jobs, njobs, n);
    else
        // 4 warps of 32 x 32, 3 x 32-row stages: 32.6 TF/s at n = 2^21, 320 x 320 (8 warps of
        // 32 x 16: 31.4; 16-row stages: 29.7-32.2)
        launch_gram<64, 64, 2, 2>(jobs, njobs, n);
}

bool gram_pair_coef(const ColList& z, int64_t n, double* g, int64_t ldg, double* c, int64_t ldc, int* status,
                    double drop_tol, double cancel_tol) {
    const int w = z.cols();
    if (w < 2 || (w & 1) || w > 56 || w / 2 > kCoefM || n < 8192 || Runtime::get().nranks() > 1)
        return false;
    check_aligned(z);
    GramJob job{z, z, g, ldg};
    job.sym = true;
    CoefParams cp{c, ldc, status, Runtime::get().tickets(1), w / 2, drop_tol, cancel_tol};
    switch ((w + 7) / 8) {
        case 1: return launch_gram_tma<1>(job, n, &cp);
        case 2: return launch_gram_tma<2>(job, n, &cp);
        case 3: return launch_gram_tma<3>(job, n, &cp);
        case 4: return launch_gram_tma<4>(job, n, &cp);
        case 5: return launch_gram_tma<5>(job, n, &cp);
        case 6: return launch_gram_tma<6>(job, n, &cp);
        default: return launch_gram_tma<7>(job, n, &cp);
    }
}

namespace {
// ------------------------------------------------------------------------------------------
// Fused MGS-Biorth application: P = X A, Q = Y B and the check Gram P^T Q in one pass
// ------------------------------------------------------------------------------------------
// (biorth.cpp:19-69 projections/normalisation applied through the coefficient matrices, then
// the second-pass test of mgs_biorth, biorth.cpp:104-107, on the P^T Q of the written P, Q.)
// Persistent CTAs walk 64-row tiles; X and Y tiles are double-buffered in shared memory by
// cp.async, A and B stay resident.  Warp w computes rows 8w..8w+7 of P and Q on the DMMA pipe,
// streams them out and parks them (column-major, stride 68) in a warp-private shared strip,
// from which the same warp feeds its rows into the running P^T Q fragments -- no CTA barrier
// between product and Gram, and P, Q are never re-read from memory.  Warps fold in order,
// CTAs through k_gram_reduce: deterministic.
constexpr int kBaLd = 68;  // smem stride of the 64-row tiles

struct BiorthApplyParams {
    ColList x, y;
    const double *ca, *cb;
    int64_t ldc;
    int k, kb, kp, ldcs;
    double *p, *q;
    int64_t ldp, ldq, n, tiles;
    double* partial;
    const int* status;  // optional device flag: nonzero -> the coefficients are invalid, no work
};

template <int BN>
__global__ void __launch_bounds__(256) k_biorth_apply(BiorthApplyParams prm) {
    constexpr int NT = BN / 8;
    extern __shared__ __align__(16) double smem[];
    if (prm.status && *prm.status) return;
    const int kp = prm.kp, ldcs = prm.ldcs;
    double* sca = smem;                        // [BN][ldcs]
    double* scb = sca + BN * ldcs;             // [BN][ldcs]
    double* sx = scb + BN * ldcs;              // [2][kp][kBaLd]
    double* sy = sx + 2 * kp * kBaLd;          // [2][kp][kBaLd]
    double* sp = sy + 2 * kp * kBaLd;          // [BN][kBaLd]
    double* sq = sp + BN * kBaLd;              // [BN][kBaLd]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int k = prm.k, kb = prm.kb;
    // A, B -> shared, zero-padded to kp x BN
    for (int e = threadIdx.x; e < BN * (kp / 2); e += 256) {
        const int c = e / (kp / 2), k2 = 2 * (e % (kp / 2));
        int bytes = 0;
        const double *srca = prm.ca, *srcb = prm.cb;
        if (c < kb && k2 < k) {
            bytes = (k - k2) >= 2 ? 16 : 8;
            srca = prm.ca + c * prm.ldc + k2;
            srcb = prm.cb + c * prm.ldc + k2;
        }
        cp_async16(sca + c * ldcs + k2, srca, bytes);
        cp_async16(scb + c * ldcs + k2, srcb, bytes);
    }
    // column base pointers once per CTA (see k_biorth_apply4); null past k: zero fill
    __shared__ const double* colx[32];
    __shared__ const double* coly[32];
    if (threadIdx.x < 32) {
        const int kk = threadIdx.x;
        colx[kk] = kk < k ? colptr(prm.x, kk) : nullptr;
        coly[kk] = kk < k ? colptr(prm.y, kk) : nullptr;
    }
    __syncthreads();
    const int lm2 = 2 * (threadIdx.x & 31), lk0 = threadIdx.x >> 5;
    auto load = [&](int buf, int64_t tile) {
        const int64_t m = tile * 64 + lm2;
        const int rb = m < prm.n ? ((prm.n - m) >= 2 ? 16 : 8) : 0;
        for (int kk = lk0; kk < kp; kk += 8) {
            const double* px = colx[kk];
            const double* py = coly[kk];
            const int bytes = px ? rb : 0;
            cp_async16(sx + (buf * kp + kk) * kBaLd + lm2, bytes ? px + m : prm.ca, bytes);
            cp_async16(sy + (buf * kp + kk) * kBaLd + lm2, bytes ? py + m : prm.ca, bytes);
        }
    };
    double g[NT][NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) g[i][j][0] = g[i][j][1] = 0.0;
    int64_t tile = blockIdx.x;
    if (tile < prm.tiles) load(0, tile);
    cp_async_commit();
    int buf = 0;
    const int wr = warp * 8;  // this warp's rows within the tile
    for (; tile < prm.tiles; tile += gridDim.x, buf ^= 1) {
        const int64_t next = tile + gridDim.x;
        if (next < prm.tiles) load(buf ^ 1, next);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double* ax = sx + buf * kp * kBaLd;
        const double* ay = sy + buf * kp * kBaLd;
        double accp[NT][2], accq[NT][2];
#pragma unroll
        for (int j = 0; j < NT; ++j) accp[j][0] = accp[j][1] = accq[j][0] = accq[j][1] = 0.0;
        for (int kk = 0; kk < kp; kk += 4) {
            const double fx = ax[(kk + tig) * kBaLd + wr + gid];
            const double fy = ay[(kk + tig) * kBaLd + wr + gid];
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                dmma(accp[j][0], accp[j][1], fx, sca[(j * 8 + gid) * ldcs + kk + tig]);
                dmma(accq[j][0], accq[j][1], fy, scb[(j * 8 + gid) * ldcs + kk + tig]);
            }
        }
        const int64_t row = tile * 64 + wr + gid;
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = j * 8 + 2 * tig + h;
                sp[col * kBaLd + wr + gid] = accp[j][h];
                sq[col * kBaLd + wr + gid] = accq[j][h];
                if (row < prm.n && col < kb) {
                    __stcs(prm.p + static_cast<int64_t>(col) * prm.ldp + row, accp[j][h]);
                    __stcs(prm.q + static_cast<int64_t>(col) * prm.ldq + row, accq[j][h]);
                }
            }
        __syncwarp();
        // P^T Q over this warp's 8 rows (two 4-row k-steps); rows past n are zero
#pragma unroll
        for (int s2 = 0; s2 < 8; s2 += 4) {
            double fp[NT], fq[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                fp[i] = sp[(i * 8 + gid) * kBaLd + wr + s2 + tig];
                fq[i] = sq[(i * 8 + gid) * kBaLd + wr + s2 + tig];
            }
#pragma unroll
            for (int i = 0; i < NT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(g[i][j][0], g[i][j][1], fp[i], fq[j]);
        }
        __syncthreads();  // everyone is done with `buf` (and its strip) before refills
    }
    cp_async_wait<0>();
    // fold the warps in order (reusing the A/B area), then the CTA partial (32 x 32 layout)
    __syncthreads();
    double* red = smem;
    for (int w = 0; w < 8; ++w) {
        if (warp == w) {
#pragma unroll
            for (int i = 0; i < NT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const int m = i * 8 + gid, nn = j * 8 + 2 * tig;
                    red[m + nn * BN] = (w == 0 ? 0.0 : red[m + nn * BN]) + g[i][j][0];
                    red[m + (nn + 1) * BN] = (w == 0 ? 0.0 : red[m + (nn + 1) * BN]) + g[i][j][1];
                }
        }
        __syncthreads();
    }
    double* part = prm.partial + static_cast<int64_t>(blockIdx.x) * (32 * 32);
    for (int e = threadIdx.x; e < BN * BN; e += 256) {
        const int m = e % BN, nn = e / BN;
        part[m + nn * 32] = red[e];
    }
}

// Compile-time variant for the common widths (<= 24 kept columns, KP = X columns rounded to 4):
// the K loop is unrolled, upper-triangular coefficients (TRI) stop the K loop of column block j
// after row 8 j + 7 at compile time, a warp owns RG groups of 8 rows (each coefficient fragment
// read from shared memory feeds RG DMMAs: the kernel is bound by the shared-memory data pipe
// next to the DMMA pipe, ncu: 67 % / 52 %), and the warp-private P, Q strips alias the warp's own
// rows of the X, Y stage (completely consumed before the strip is written).
template <int BN, int KP, bool TRI, int RG>
__global__ void __launch_bounds__(256, 2) k_biorth_apply4(BiorthApplyParams prm) {
    constexpr int NT = BN / 8;
    constexpr int TR = 64 * RG;           // rows per tile
    constexpr int LD = TR + 4;            // smem stride of a stage column
    constexpr int LDCS = (KP + 15) / 16 * 16 + 4;
    extern __shared__ __align__(16) double smem[];
    if (prm.status && *prm.status) return;
    double* sca = smem;                   // [BN][LDCS]
    double* scb = sca + BN * LDCS;        // [BN][LDCS]
    double* sx = scb + BN * LDCS;         // [2][KP][LD]
    double* sy = sx + 2 * KP * LD;        // [2][KP][LD]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int k = prm.k, kb = prm.kb;
    for (int e = threadIdx.x; e < BN * (KP / 2); e += 256) {
        const int c = e / (KP / 2), k2 = 2 * (e % (KP / 2));
        int bytes = 0;
        const double *srca = prm.ca, *srcb = prm.cb;
        if (c < kb && k2 < k) {
            bytes = (k - k2) >= 2 ? 16 : 8;
            srca = prm.ca + c * prm.ldc + k2;
            srcb = prm.cb + c * prm.ldc + k2;
        }
        cp_async16(sca + c * LDCS + k2, srca, bytes);
        cp_async16(scb + c * LDCS + k2, srcb, bytes);
    }
    // column base pointers once per CTA (the ColList segment search per cp.async was ~55 % of
    // the kernel's instructions); columns past k stay null and are zero-filled
    __shared__ const double* colx[KP];
    __shared__ const double* coly[KP];
    if (threadIdx.x < KP) {
        const int kk = threadIdx.x;
        colx[kk] = kk < k ? colptr(prm.x, kk) : nullptr;
        coly[kk] = kk < k ? colptr(prm.y, kk) : nullptr;
    }
    __syncthreads();
    constexpr int CPI = 256 / (TR / 2);   // columns per pass of the 256 threads
    const int lm2 = 2 * (threadIdx.x % (TR / 2)), lk0 = threadIdx.x / (TR / 2);
    auto load = [&](int buf, int64_t tile) {
        const int64_t m = tile * TR + lm2;
        const int rb = m < prm.n ? ((prm.n - m) >= 2 ? 16 : 8) : 0;
        double* dx = sx + (buf * KP + lk0) * LD + lm2;
        double* dy = sy + (buf * KP + lk0) * LD + lm2;
#pragma unroll
        for (int it = 0; it < (KP + CPI - 1) / CPI; ++it) {
            const int kk = it * CPI + lk0;
            if (KP % CPI != 0 && kk >= KP) break;
            const double* px = colx[kk];
            const double* py = coly[kk];
            const int bytes = px ? rb : 0;
            cp_async16(dx + it * CPI * LD, bytes ? px + m : prm.ca, bytes);
            cp_async16(dy + it * CPI * LD, bytes ? py + m : prm.ca, bytes);
        }
    };
    double g[NT][NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) g[i][j][0] = g[i][j][1] = 0.0;
    int64_t tile = blockIdx.x;
    if (tile < prm.tiles) load(0, tile);
    cp_async_commit();
    int buf = 0;
    const int wr = warp * 8 * RG;
    for (; tile < prm.tiles; tile += gridDim.x, buf ^= 1) {
        const int64_t next = tile + gridDim.x;
        if (next < prm.tiles) load(buf ^ 1, next);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        double* ax = sx + buf * KP * LD + wr;
        double* ay = sy + buf * KP * LD + wr;
        double accp[RG][NT][2], accq[RG][NT][2];
#pragma unroll
        for (int r = 0; r < RG; ++r)
#pragma unroll
            for (int j = 0; j < NT; ++j) accp[r][j][0] = accp[r][j][1] = accq[r][j][0] = accq[r][j][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KP; kk += 4) {
            double fx[RG], fy[RG];
#pragma unroll
            for (int r = 0; r < RG; ++r) {
                fx[r] = ax[(kk + tig) * LD + 8 * r + gid];
                fy[r] = ay[(kk + tig) * LD + 8 * r + gid];
            }
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                if (TRI && kk >= 8 * (j + 1)) continue;
                const double ca = sca[(j * 8 + gid) * LDCS + kk + tig];
                const double cb = scb[(j * 8 + gid) * LDCS + kk + tig];
#pragma unroll
                for (int r = 0; r < RG; ++r) {
                    dmma(accp[r][j][0], accp[r][j][1], fx[r], ca);
                    dmma(accq[r][j][0], accq[r][j][1], fy[r], cb);
                }
            }
        }
        __syncwarp();  // every lane has consumed its X, Y fragments: the rows become the strip
#pragma unroll
        for (int r = 0; r < RG; ++r) {
            const int64_t row = tile * TR + wr + 8 * r + gid;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    // lanes tig = 0..3 store columns 0, 2, 5, 7 (then 1, 3, 4, 6) of the block:
                    // distinct mod 4, so the strip stores (stride LD = 4 mod 16) hit 16
                    // distinct banks per half-warp (same-h stores were 2-way conflicts)
                    const int h = (tig >> 1) ^ s;
                    const int col = j * 8 + 2 * tig + h;
                    const double vp = h ? accp[r][j][1] : accp[r][j][0];
                    const double vq = h ? accq[r][j][1] : accq[r][j][0];
                    if (col < KP) {  // columns kb..KP-1 are exact zeros (zero-padded coefficients)
                        ax[col * LD + 8 * r + gid] = vp;
                        ay[col * LD + 8 * r + gid] = vq;
                    }
                    if (row < prm.n && col < kb) {
                        __stcs(prm.p + static_cast<int64_t>(col) * prm.ldp + row, vp);
                        __stcs(prm.q + static_cast<int64_t>(col) * prm.ldq + row, vq);
                    }
                }
        }
        __syncwarp();
#pragma unroll
        for (int s2 = 0; s2 < 8 * RG; s2 += 4) {
            double fp[NT], fq[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) {
                const bool in = i * 8 + gid < KP;
                fp[i] = in ? ax[(i * 8 + gid) * LD + s2 + tig] : 0.0;
                fq[i] = in ? ay[(i * 8 + gid) * LD + s2 + tig] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < NT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(g[i][j][0], g[i][j][1], fp[i], fq[j]);
        }
        __syncthreads();  // everyone is done with `buf` before it is refilled
    }
    cp_async_wait<0>();
    __syncthreads();
    double* red = smem;
    for (int w = 0; w < 8; ++w) {
        if (warp == w) {
#pragma unroll
            for (int i = 0; i < NT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const int m = i * 8 + gid, nn = j * 8 + 2 * tig;
                    red[m + nn * BN] = (w == 0 ? 0.0 : red[m + nn * BN]) + g[i][j][0];
                    red[m + (nn + 1) * BN] = (w == 0 ? 0.0 : red[m + (nn + 1) * BN]) + g[i][j][1];
                }
        }
        __syncthreads();
    }
    double* part = prm.partial + static_cast<int64_t>(blockIdx.x) * (32 * 32);
    for (int e = threadIdx.x; e < BN * BN; e += 256) {
        const int m = e % BN, nn = e / BN;
        part[m + nn * 32] = red[e];
    }
}

template <int BN, int KP, bool TRI, int RG>
void launch_biorth_apply4(BiorthApplyParams prm, int64_t n, double* g, int64_t ldg, const DMat& pv, const DMat& qv) {
    Runtime& rt = Runtime::get();
    constexpr int TR = 64 * RG, LD = TR + 4, LDCS = (KP + 15) / 16 * 16 + 4;
    constexpr size_t smem = sizeof(double) * (2ull * BN * LDCS + 4ull * KP * LD);
    static int per_sm[32] = {0};
    static unsigned attr_mask = 0;
    rt.once_per_device(attr_mask, [&] {  // ranks sharing a GPU (ThreadComm) set it up once
        BOSP_CUDA(cudaFuncSetAttribute(k_biorth_apply4<BN, KP, TRI, RG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
        int r = 0;
        BOSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_biorth_apply4<BN, KP, TRI, RG>, 256, smem));
        per_sm[rt.device() & 31] = std::max(1, r);
    });
    prm.tiles = (n + TR - 1) / TR;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(prm.tiles, per_sm[rt.device() & 31] * rt.sm_count())));
    prm.partial = rt.scratch(static_cast<size_t>(grid) * 32 * 32);
    const double flops = 2.0 * n * prm.k * prm.kb * 2 + 2.0 * n * prm.kb * prm.kb;
    const double bytes = 8.0 * n * (2.0 * prm.k + 2.0 * prm.kb);
    {
        LaunchScope ls("product", bytes, flops);
        k_biorth_apply4<BN, KP, TRI, RG><<<grid, 256, smem, rt.stream()>>>(prm);
        BOSP_LAUNCH_CHECK();
    }
    GramParams gp{};
    gp.job[0] = GramJob{ColList(pv), ColList(qv), g, ldg};
    gp.tiles_n[0] = 1;
    gp.tiles[0] = 1;
    gp.splits = grid;
    gp.partial = prm.partial;
    gp.job_stride = static_cast<int64_t>(grid) * 32 * 32;
    {
        LaunchScope ls("gram_reduce");
        k_gram_reduce<32, 32><<<dim3(32 * 32 / kRedElems, 1, 1), kRedElems * kRedGroups, 0, rt.stream()>>>(gp);
        BOSP_LAUNCH_CHECK();
    }
}

template <int BN, int KP>
bool dispatch_biorth_apply4(const BiorthApplyParams& prm, int tri, int rg, int64_t n, double* g, int64_t ldg,
                            const DMat& pv, const DMat& qv) {
    if (tri) {
        if (rg == 2) launch_biorth_apply4<BN, KP, true, 2>(prm, n, g, ldg, pv, qv);
        else launch_biorth_apply4<BN, KP, true, 1>(prm, n, g, ldg, pv, qv);
    } else {
        if (rg == 2) launch_biorth_apply4<BN, KP, false, 2>(prm, n, g, ldg, pv, qv);
        else launch_biorth_apply4<BN, KP, false, 1>(prm, n, g, ldg, pv, qv);
    }
    return true;
}

template <int BN>
void launch_biorth_apply(BiorthApplyParams prm, int64_t n, double* g, int64_t ldg, const DMat& pv, const DMat& qv) {
    Runtime& rt = Runtime::get();
    const size_t smem = sizeof(double) * (2ull * BN * prm.ldcs + 4ull * prm.kp * kBaLd + 2ull * BN * kBaLd);
    static int per_sm[64] = {0};
    if (per_sm[rt.device() & 63] == 0) {
        BOSP_CUDA(cudaFuncSetAttribute(k_biorth_apply<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(232448 - 1024)));
        int r = 0;
        BOSP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, k_biorth_apply<BN>, 256, smem));
        per_sm[rt.device() & 63] = std::max(1, r);
    }
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(prm.tiles, per_sm[rt.device() & 63] * rt.sm_count())));
    prm.partial = rt.scratch(static_cast<size_t>(grid) * 32 * 32);
    const double flops = 2.0 * n * prm.k * prm.kb * 2 + 2.0 * n * prm.kb * prm.kb;
    const double bytes = 8.0 * n * (2.0 * prm.k + 2.0 * prm.kb);
    {
        LaunchScope ls("product", bytes, flops);
        k_biorth_apply<BN><<<grid, 256, smem, rt.stream()>>>(prm);
        BOSP_LAUNCH_CHECK();
    }
    GramParams gp{};
    gp.job[0] = GramJob{ColList(pv), ColList(qv), g, ldg};
    gp.tiles_n[0] = 1;
    gp.tiles[0] = 1;
    gp.splits = grid;
    gp.partial = prm.partial;
    gp.job_stride = static_cast<int64_t>(grid) * 32 * 32;
    {
        LaunchScope ls("gram_reduce");
        k_gram_reduce<32, 32><<<dim3(32 * 32 / kRedElems, 1, 1), kRedElems * kRedGroups, 0, rt.stream()>>>(gp);
        BOSP_LAUNCH_CHECK();
    }
}

// The same fused application with TMA staging: one persistent CTA per SM owns a contiguous range
// of 64-row stages of X and Y (one 3-D tensor-map load per operand and stage -- box (16 rows, k
// columns, 4 row groups), 128-byte swizzle, see k_gram_tma -- issued by a producer warp into a several-deep
// mbarrier ring); consumer warp w computes rows 8w..8w+7 of P and Q from the stage, releases
// the stage, streams its rows out and feeds them into its P^T Q fragments from a warp-private
// shared strip.  Compile-time widths: the k loop is unrolled and the coefficient fragments stay
// in registers (the kernel is issue-bound: ncu saw ~650 instructions per 8 rows, 7 % DMMA, with
// a runtime k loop, per-row coefficient reloads and per-column store guards).
struct BiorthTmaParams {
    TmaSegs seg;            // X (k columns), Y (k columns)
    const double *ca, *cb;
    int64_t ldc;
    int k, kb, kp;
    int tri;                // coefficients upper triangular (column c: rows <= c)
    double *p, *q;
    int64_t ldp, ldq, n, stages;
    int nst;
    double* partial;
    const int* status;  // optional device flag: nonzero -> the coefficients are invalid, no work
};
// Consumer warps and 8-row blocks per consumer warp.  Measured at n = 2^21, m = 20 (the
// kernel is DMMA-latency bound, not byte bound): 8 warps x 1 block, coefficients in registers:
// 390-398 us; 8 warps x 2 blocks: 390 us; 16 warps x 1 block, coefficients in shared memory
// (17 warps: <= 96 registers): 395 us -- all slower than the cp.async kernel (k_biorth_apply,
// 350 us) except at 32 columns (704 vs 797 us), where biorth_apply uses this one.
#ifndef BOSP_BA_CW
#define BOSP_BA_CW 8
#endif
constexpr int ba_cw(int bn) { return bn >= 32 ? 8 : BOSP_BA_CW; }
constexpr int ba_mb(int bn) { return ba_cw(bn) > 8 || bn >= 32 ? 1 : 2; }
constexpr int ba_rows(int bn) { return ba_cw(bn) * 8 * ba_mb(bn); }  // stage rows

template <int BN, int KP>
__global__ void __launch_bounds__((ba_cw(BN) + 1) * 32, 1) k_biorth_apply_tma(const __grid_constant__ BiorthTmaParams prm) {
    constexpr int NT = BN / 8, KS = KP / 4, MB = ba_mb(BN), kBaR = ba_rows(BN), kBaS = kBaR + 4, CW = ba_cw(BN);
    // coefficient fragments live in registers when they fit (KS x NT x 2 doubles per lane; 9
    // warps leave 168 registers per thread -- 3 warps share one SM sub-partition's file)
    constexpr bool kRegC = CW <= 8 && KS * NT * MB <= 12;
    extern __shared__ __align__(1024) double sm_bat[];
    __shared__ __align__(8) unsigned long long full_bar[kTmaMaxSt], empty_bar[kTmaMaxSt];
    if (prm.status && *prm.status) return;
    const int k = prm.k, kb = prm.kb, NST = prm.nst;
    constexpr int ldcs = KP + 4;
    const int stage_d = prm.seg.stage;
    double* ring = sm_bat;                  // [NST][X box | Y box], 128-byte lines [row group][column]
    double* sca = ring + NST * stage_d;     // [BN][ldcs]
    double* scb = sca + BN * ldcs;          // [BN][ldcs]
    double* sp = scb + BN * ldcs;           // [BN][kBaS] strip of P rows
    double* sq = sp + BN * kBaS;            // [BN][kBaS]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int64_t s0 = prm.stages * blockIdx.x / gridDim.x, s1 = prm.stages * (blockIdx.x + 1) / gridDim.x;
    const int64_t mine = s1 - s0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&full_bar[i], 1);
            mbar_init(&empty_bar[i], CW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // A, B -> shared, zero-padded to KP x BN
    for (int e = threadIdx.x; e < BN * ldcs; e += blockDim.x) {
        const int c = e / ldcs, kk = e % ldcs;
        const bool v = c < kb && kk < k;
        sca[e] = v ? prm.ca[c * prm.ldc + kk] : 0.0;
        scb[e] = v ? prm.cb[c * prm.ldc + kk] : 0.0;
    }
    __syncthreads();
    double cfa[kRegC ? KS : 1][NT], cfb[kRegC ? KS : 1][NT];
    if constexpr (kRegC) {
#pragma unroll
        for (int s = 0; s < KS; ++s)
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                cfa[s][j] = sca[(j * 8 + gid) * ldcs + 4 * s + tig];
                cfb[s][j] = scb[(j * 8 + gid) * ldcs + 4 * s + tig];
            }
    }
    double g[NT][NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) g[i][j][0] = g[i][j][1] = 0.0;
    const int wr = warp * 8 * MB;  // this warp's MB 8-row blocks: rows wr .. wr + 8 MB - 1
    // this lane's X / Y fragment addresses: row wr + 8 b + gid of a box (row group wr / 16),
    // column 4 s + tig; lines of columns 8 apart share the swizzle phase, so k-steps s and s + 2
    // differ by 8 lines
    const int bl = static_cast<int>(smem_u32(sm_bat) >> 7) & 7;
    const int xl = prm.seg.off[0] / 16 + (wr >> 4) * k + tig;
    const int yl = prm.seg.off[1] / 16 + (wr >> 4) * k + tig;
    int xa[MB][2], ya[MB][2];
#pragma unroll
    for (int b = 0; b < MB; ++b) {
        const int rr = (wr + 8 * b + gid) & 15;
        xa[b][0] = swz(xl, rr, bl);
        xa[b][1] = swz(xl + 4, rr, bl) - 4 * 128;
        ya[b][0] = swz(yl, rr, bl);
        ya[b][1] = swz(yl + 4, rr, bl) - 4 * 128;
    }
    const bool full_cols = kb == BN, tri = prm.tri != 0;
    if (warp == CW) {
        if (lane == 0)
            for (int64_t s = 0; s < mine; ++s) {
                const int slot = static_cast<int>(s % NST);
                if (s >= NST) mbar_wait(&empty_bar[slot], static_cast<unsigned>((s / NST - 1) & 1));
                tma_stage(prm.seg, ring + slot * stage_d, kBaR, s0 + s, &full_bar[slot]);
            }
    } else {
        for (int64_t s = 0; s < mine; ++s) {
            const int slot = static_cast<int>(s % NST);
            mbar_wait(&full_bar[slot], static_cast<unsigned>((s / NST) & 1));
            const char* buf = reinterpret_cast<const char*>(ring + slot * stage_d);
            double accp[MB][NT][2], accq[MB][NT][2];
#pragma unroll
            for (int b = 0; b < MB; ++b)
#pragma unroll
                for (int j = 0; j < NT; ++j) accp[b][j][0] = accp[b][j][1] = accq[b][j][0] = accq[b][j][1] = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int kr = 4 * ks + tig;
                const int off = 4 * ks * 128;
                double fx[MB], fy[MB];
#pragma unroll
                for (int b = 0; b < MB; ++b) {
                    fx[b] = *reinterpret_cast<const double*>(buf + xa[b][ks & 1] + off);
                    fy[b] = *reinterpret_cast<const double*>(buf + ya[b][ks & 1] + off);
                    if (4 * ks + 4 > k && kr >= k) fx[b] = fy[b] = 0.0;  // columns past k (last k-step only)
                }
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    // triangular coefficients: column block j has nonzero rows < 8 j + 8 only
                    if (tri && ks > 2 * j + 1) continue;
                    double ca, cb;
                    if constexpr (kRegC) {
                        ca = cfa[ks][j];
                        cb = cfb[ks][j];
                    } else {
                        ca = sca[(j * 8 + gid) * ldcs + kr];
                        cb = scb[(j * 8 + gid) * ldcs + kr];
                    }
#pragma unroll
                    for (int b = 0; b < MB; ++b) {
                        dmma(accp[b][j][0], accp[b][j][1], fx[b], ca);
                        dmma(accq[b][j][0], accq[b][j][1], fy[b], cb);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_bar[slot]);  // the stage may be refilled
#pragma unroll
            for (int b = 0; b < MB; ++b) {
                const int lr = wr + 8 * b + gid;
                const int64_t row = (s0 + s) * kBaR + lr;
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = j * 8 + 2 * tig + h;
                        sp[col * kBaS + lr] = accp[b][j][h];
                        sq[col * kBaS + lr] = accq[b][j][h];
                    }
                if (full_cols && row < prm.n) {
#pragma unroll
                    for (int j = 0; j < NT; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int col = j * 8 + 2 * tig + h;
                            __stcs(prm.p + static_cast<int64_t>(col) * prm.ldp + row, accp[b][j][h]);
                            __stcs(prm.q + static_cast<int64_t>(col) * prm.ldq + row, accq[b][j][h]);
                        }
                } else if (row < prm.n) {
#pragma unroll
                    for (int j = 0; j < NT; ++j)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int col = j * 8 + 2 * tig + h;
                            if (col < kb) {
                                __stcs(prm.p + static_cast<int64_t>(col) * prm.ldp + row, accp[b][j][h]);
                                __stcs(prm.q + static_cast<int64_t>(col) * prm.ldq + row, accq[b][j][h]);
                            }
                        }
                }
            }
            __syncwarp();
            // P^T Q over this warp's rows (rows past n are zero: TMA zero-filled X, Y)
#pragma unroll
            for (int s2 = 0; s2 < 8 * MB; s2 += 4) {
                double fp[NT], fq[NT];
#pragma unroll
                for (int i = 0; i < NT; ++i) {
                    fp[i] = sp[(i * 8 + gid) * kBaS + wr + s2 + tig];
                    fq[i] = sq[(i * 8 + gid) * kBaS + wr + s2 + tig];
                }
#pragma unroll
                for (int i = 0; i < NT; ++i)
#pragma unroll
                    for (int j = 0; j < NT; ++j) dmma(g[i][j][0], g[i][j][1], fp[i], fq[j]);
            }
            __syncwarp();  // the strip is rewritten by this warp's next rows
        }
    }
    __syncthreads();
    // fold the consumer warps in order (reusing the ring), then the CTA partial (32 x 32 layout)
    double* red = ring;
    for (int w = 0; w < CW; ++w) {
        if (warp == w) {
#pragma unroll
            for (int i = 0; i < NT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                    const int m = i * 8 + gid, nn = j * 8 + 2 * tig;
                    red[m + nn * BN] = (w == 0 ? 0.0 : red[m + nn * BN]) + g[i][j][0];
                    red[m + (nn + 1) * BN] = (w == 0 ? 0.0 : red[m + (nn + 1) * BN]) + g[i][j][1];
                }
        }
        __syncthreads();
    }
    double* part = prm.partial + static_cast<int64_t>(blockIdx.x) * (32 * 32);
    for (int e = threadIdx.x; e < BN * BN; e += blockDim.x) {
        const int m = e % BN, nn = e / BN;
        part[m + nn * 32] = red[e];
    }
}

template <int BN, int KP>
void launch_biorth_apply_tma(BiorthTmaParams prm, int64_t n, double* g, int64_t ldg, const DMat& pv, const DMat& qv) {
    Runtime& rt = Runtime::get();
    const size_t fixed = sizeof(double) * (2ull * BN * (KP + 4) + 2ull * BN * (ba_rows(BN) + 4));
    const size_t stage_b = sizeof(double) * prm.seg.stage;
    prm.nst = static_cast<int>(std::max<size_t>(2, std::min<size_t>(kTmaMaxSt, (218u * 1024u - fixed) / stage_b)));
    const size_t smem = std::max(fixed + stage_b * prm.nst, fixed + sizeof(double) * BN * BN);
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(rt.sm_count(), prm.stages)));
    prm.partial = rt.scratch(static_cast<size_t>(grid) * 32 * 32);
    static unsigned attr_mask = 0;
    rt.once_per_device(attr_mask, [&] {
        BOSP_CUDA(cudaFuncSetAttribute(k_biorth_apply_tma<BN, KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    });
    const double flops = 2.0 * n * prm.k * prm.kb * 2 + 2.0 * n * prm.kb * prm.kb;
    const double bytes = 8.0 * n * (2.0 * prm.k + 2.0 * prm.kb);
    {
        LaunchScope ls("product", bytes, flops);
        k_biorth_apply_tma<BN, KP><<<grid, (ba_cw(BN) + 1) * 32, smem, rt.stream()>>>(prm);
        BOSP_LAUNCH_CHECK();
    }
    GramParams gp{};
    gp.job[0] = GramJob{ColList(pv), ColList(qv), g, ldg};
    gp.tiles_n[0] = 1;
    gp.tiles[0] = 1;
    gp.splits = grid;
    gp.partial = prm.partial;
    gp.job_stride = static_cast<int64_t>(grid) * 32 * 32;
    {
        LaunchScope ls("gram_reduce");
        k_gram_reduce<32, 32><<<dim3(32 * 32 / kRedElems, 1, 1), kRedElems * kRedGroups, 0, rt.stream()>>>(gp);
        BOSP_LAUNCH_CHECK();
    }
}

// (BN, KP) dispatch: BN = kept columns rounded to 8, KP = X columns rounded to 4 (kb <= k)
template <int BN>
void launch_biorth_apply_tma_k(BiorthTmaParams prm, int64_t n, double* g, int64_t ldg, const DMat& pv, const DMat& qv) {
    switch (prm.kp) {
        case 4: if constexpr (BN <= 8) return launch_biorth_apply_tma<BN, 4>(prm, n, g, ldg, pv, qv); break;
        case 8: if constexpr (BN <= 8) return launch_biorth_apply_tma<BN, 8>(prm, n, g, ldg, pv, qv); break;
        case 12: if constexpr (BN <= 16) return launch_biorth_apply_tma<BN, 12>(prm, n, g, ldg, pv, qv); break;
        case 16: if constexpr (BN <= 16) return launch_biorth_apply_tma<BN, 16>(prm, n, g, ldg, pv, qv); break;
        case 20: if constexpr (BN <= 24) return launch_biorth_apply_tma<BN, 20>(prm, n, g, ldg, pv, qv); break;
        case 24: if constexpr (BN <= 24) return launch_biorth_apply_tma<BN, 24>(prm, n, g, ldg, pv, qv); break;
        case 28: return launch_biorth_apply_tma<BN, 28>(prm, n, g, ldg, pv, qv);
        default: return launch_biorth_apply_tma<BN, 32>(prm, n, g, ldg, pv, qv);
    }
    throw ContractViolation("biorth_apply: kept columns exceed the block width");
}

}  // namespace

void biorth_apply(const DMat& x, const DMat& y, const double* ca, const double* cb, int64_t ldc, int kb,
                  const DMat& p, const DMat& q, double* g, int64_t ldg, const int32_t* col_kend,
                  const int* status_dev) {
    require(x.cols == y.cols && x.rows == y.rows && p.rows == x.rows && q.rows == x.rows, "biorth_apply: shapes");
    require(x.cols <= 32 && kb <= 32 && kb >= 1 && p.cols >= kb && q.cols >= kb, "biorth_apply: widths <= 32");
    check_aligned(ColList(x));
    check_aligned(ColList(y));
    const int64_t n = x.rows;
    const DMat pv = p.cols_range(0, kb), qv = q.cols_range(0, kb);
    const int kpad = std::max(4, (static_cast<int>(x.cols) + 3) / 4 * 4);
    BiorthTmaParams tp{};
    if (kb > 24 && n >= 8192 &&
        make_segs(tp.seg, ColList(x).add(y), n, ba_rows((kb + 7) / 8 * 8))) {
        const int k = static_cast<int>(x.cols);
        tp.ca = ca;
        tp.cb = cb;
        tp.ldc = ldc;
        tp.k = k;
        tp.kb = kb;
        tp.kp = kpad;
        // upper triangular (column c nonzero in rows <= c only): the K loop of column block j
        // stops after row 8 j + 7
        tp.tri = col_kend != nullptr;
        for (int c = 0; tp.tri && c < kb; ++c) tp.tri = col_kend[c] <= c + 1;
        tp.p = p.p;
        tp.q = q.p;
        tp.ldp = p.ld;
        tp.ldq = q.ld;
        tp.n = n;
        tp.stages = (n + ba_rows((kb + 7) / 8 * 8) - 1) / ba_rows((kb + 7) / 8 * 8);
        tp.status = status_dev;
        switch ((kb + 7) / 8) {
            case 1: return launch_biorth_apply_tma_k<8>(tp, n, g, ldg, pv, qv);
            case 2: return launch_biorth_apply_tma_k<16>(tp, n, g, ldg, pv, qv);
            case 3: return launch_biorth_apply_tma_k<24>(tp, n, g, ldg, pv, qv);
            default: return launch_biorth_apply_tma_k<32>(tp, n, g, ldg, pv, qv);
        }
    }
    BiorthApplyParams prm{};
    prm.x = ColList(x);
    prm.y = ColList(y);
    prm.ca = ca;
    prm.cb = cb;
    prm.ldc = ldc;
    prm.k = static_cast<int>(x.cols);
    prm.kb = kb;
    prm.kp = kpad;
    prm.ldcs = (prm.kp + 15) / 16 * 16 + 4;
    prm.p = p.p;
    prm.q = q.p;
    prm.ldp = p.ld;
    prm.ldq = q.ld;
    prm.n = n;
    prm.tiles = (n + 63) / 64;
    prm.status = status_dev;
    int tri = col_kend != nullptr;
    for (int c = 0; tri && c < kb; ++c) tri = col_kend[c] <= c + 1;
    // the common widths run the compile-time kernel (BOSP_APPLY4=0: the runtime-width one;
    // =1 / =2: 8 / 16 rows per warp)
    static const int v4 = std::getenv("BOSP_APPLY4") ? std::atoi(std::getenv("BOSP_APPLY4")) : 2;
    if (v4 > 0 && n >= 8192) {
        const int bn = (kb + 7) / 8 * 8;
#define BOSP_A4(BN_, KP_) \
    if (bn == BN_ && kpad == KP_ && dispatch_biorth_apply4<BN_, KP_>(prm, tri, v4, n, g, ldg, pv, qv)) return;
        BOSP_A4(24, 20) BOSP_A4(24, 24) BOSP_A4(16, 12) BOSP_A4(16, 16) BOSP_A4(8, 4) BOSP_A4(8, 8)
#undef BOSP_A4
    }
    switch ((kb + 7) / 8) {
        case 1: return launch_biorth_apply<8>(prm, n, g, ldg, pv, qv);
        case 2: return launch_biorth_apply<16>(prm, n, g, ldg, pv, qv);
        case 3: return launch_biorth_apply<24>(prm, n, g, ldg, pv, qv);
        default: return launch_biorth_apply<32>(prm, n, g, ldg, pv, qv);
    }
}

namespace {
// ------------------------------------------------------------------------------------------
// Rank-k update Out = alpha A C + beta Out for k <= 8 and wide Out (the projection of a
// 320-column block against the one-column null basis, biorth_against / the repair's sampled
// projection): a streaming pass over Out (16-byte row pairs, coalesced per column), A's k
// values of a row pair loaded once per column group, C broadcast from shared memory.  The tiled
// DMMA kernel spent 14.7 ms on it at n = 2^21, d = 320 (a 16-deep K loop for k = 1).
constexpr int kRkThreads = 256, kRkCols = 32;

struct RankKParams {
    ProductJob job[4];
    int64_t n;
    int groups[4];  // column groups per job
};

template <int K>
__global__ void __launch_bounds__(kRkThreads) k_rankk(RankKParams prm) {
    __shared__ double cs[8][kRkCols];
    const int jb = blockIdx.z;
    const ProductJob& job = prm.job[jb];
    if (static_cast<int>(blockIdx.y) >= prm.groups[jb]) return;
    const int c0 = blockIdx.y * kRkCols;
    const int nc = min(kRkCols, job.ncols - c0);
    const int k = job.a.cols();
    for (int e = threadIdx.x; e < 8 * kRkCols; e += kRkThreads) {
        const int t = e / kRkCols, c = e % kRkCols;
        cs[t][c] = (t < k && c < nc) ? job.alpha * job.c[t + static_cast<int64_t>(c0 + c) * job.ldc] : 0.0;
    }
    __syncthreads();
    const double* ap[K];
#pragma unroll
    for (int t = 0; t < K; ++t) ap[t] = t < k ? colptr(job.a, t) : nullptr;
    const double beta = job.beta;
    const int64_t npair = prm.n >> 1;
    for (int64_t q = blockIdx.x * static_cast<int64_t>(kRkThreads) + threadIdx.x; q < npair;
         q += static_cast<int64_t>(gridDim.x) * kRkThreads) {
        const int64_t i = 2 * q;
        double2 a[K];
#pragma unroll
        for (int t = 0; t < K; ++t) a[t] = ap[t] ? __ldg(reinterpret_cast<const double2*>(ap[t] + i)) : make_double2(0.0, 0.0);
        double* out = job.out + static_cast<int64_t>(c0) * job.ldo + i;
#pragma unroll 4
        for (int c = 0; c < nc; ++c) {
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int t = 0; t < K; ++t) {
                s0 = fma(a[t].x, cs[t][c], s0);
                s1 = fma(a[t].y, cs[t][c], s1);
            }
            double2* o = reinterpret_cast<double2*>(out + static_cast<int64_t>(c) * job.ldo);
            if (beta != 0.0) {
                const double2 v = *o;
                s0 = fma(beta, v.x, s0);
                s1 = fma(beta, v.y, s1);
            }
            *o = make_double2(s0, s1);
        }
    }
    if ((prm.n & 1) && blockIdx.x == 0 && threadIdx.x < nc) {  // the last row of an odd n
        const int64_t i = prm.n - 1;
        const int c = threadIdx.x;
        double s = 0.0;
        for (int t = 0; t < k; ++t) s = fma(ap[t][i], cs[t][c], s);
        double* o = job.out + static_cast<int64_t>(c0 + c) * job.ldo + i;
        *o = beta != 0.0 ? fma(beta, *o, s) : s;
    }
}

template <int K>
void launch_rankk(const ProductJob* jobs, int njobs, int64_t n) {
    Runtime& rt = Runtime::get();
    RankKParams prm{};
    int gmax = 0;
    double bytes = 0.0, flops = 0.0;
    for (int j = 0; j < njobs; ++j) {
        prm.job[j] = jobs[j];
        prm.groups[j] = (jobs[j].ncols + kRkCols - 1) / kRkCols;
        gmax = std::max(gmax, prm.groups[j]);
        bytes += 8.0 * n * (jobs[j].a.cols() + jobs[j].ncols * (jobs[j].beta != 0.0 ? 2.0 : 1.0));
        flops += 2.0 * n * jobs[j].a.cols() * jobs[j].ncols;
    }
    prm.n = n;
    const int64_t npair = std::max<int64_t>(1, n / 2);
    const int64_t want = 8LL * rt.sm_count() * 2048 / kRkThreads;  // ~8 waves of resident blocks
    const unsigned gx = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((npair + kRkThreads - 1) / kRkThreads,
                                                                                     want / std::max(1, gmax * njobs) + 1)));
    LaunchScope ls(shape_family("product", K, jobs[0].ncols, jobs[0].beta != 0.0, njobs), bytes, flops);
    k_rankk<K><<<dim3(gx, gmax, njobs), kRkThreads, 0, rt.stream()>>>(prm);
    BOSP_LAUNCH_CHECK();
}
}  // namespace

void product(const ProductJob* jobs, int njobs, int64_t n) {
    require(njobs >= 1 && njobs <= 4, "product: 1..4 jobs per launch");
    int bmax = 0;
    for (int j = 0; j < njobs; ++j) {
        check_aligned(jobs[j].a);
        require((reinterpret_cast<uintptr_t>(jobs[j].c) & 15) == 0 && (jobs[j].ldc & 1) == 0,
                "product: C must be 16-byte aligned with even ldc");
        bmax = std::max(bmax, jobs[j].ncols);
    }
    if (n == 0 || bmax == 0) return;
    int kmax = 0;
    for (int j = 0; j < njobs; ++j) kmax = std::max(kmax, jobs[j].a.cols());
    if (kmax <= 64 && bmax <= 64 && kmax > 0) {
        switch ((bmax + 7) / 8) {
            case 1: return launch_skinny<8>(jobs, njobs, n);
            case 2: return launch_skinny<16>(jobs, njobs, n);
            case 3: return launch_skinny<24>(jobs, njobs, n);
            case 4: return launch_skinny<32>(jobs, njobs, n);
            case 5: return launch_skinny<40>(jobs, njobs, n);
            case 6: return launch_skinny<48>(jobs, njobs, n);
            case 7: return launch_skinny<56>(jobs, njobs, n);
            default: return launch_skinny<64>(jobs, njobs, n);
        }
    }
    // rank-k updates of wide blocks (k <= 8, e.g. the projection against the null basis): a
    // streaming pass, not a DMMA tile loop
    if (kmax > 0 && kmax <= 8) {
        bool aligned = true;
        for (int j = 0; j < njobs; ++j) aligned = aligned && (jobs[j].ldo & 1) == 0 && (reinterpret_cast<uintptr_t>(jobs[j].out) & 15) == 0;
        if (aligned) return kmax <= 1 ? launch_rankk<1>(jobs, njobs, n)
                          : kmax <= 2 ? launch_rankk<2>(jobs, njobs, n)
                          : kmax <= 4 ? launch_rankk<4>(jobs, njobs, n) : launch_rankk<8>(jobs, njobs, n);
    }
    // k == 0: Out = beta * Out (handled by the kernel with an empty K loop)
    // 4 warps of 32 x 32 (16 DMMAs per 8 fragment loads), 3 x 16-deep stages, 3 CTAs/SM:
    // 31.5 TF/s at n = 2^21, 320 -> 192 (8 warps of 32 x 16: 30.3; 128-row tiles: 28.6-30.6)
    if (bmax <= 32)
        launch_product<64, 32, 2, 2>(jobs, njobs, n);
    else
        launch_product<64, 64, 2, 2, 16, 3>(jobs, njobs, n);
}

}  // namespace b200
}  // namespace bosp
