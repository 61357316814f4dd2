// Bit-exact std::mt19937_64 + uniform_real_distribution<double>(-1, 1) stream on the device.
//
// The reference seeds X, P, W, Y, Q, Z from one mt19937_64(seed) stream in that order
// (bosp_solver.cpp:144-150, block_vectors.cpp:27-30).  Reproducing the stream keeps the B200
// solver on the reference's starting vectors.  MT19937-64 is sequential across 312-word
// blocks but parallel within one: a single CTA twists the whole state per step (two dependent
// halves separated by a barrier), tempers and converts 312 draws and writes them straight into
// their column of U or V.  ~100k steps for config 2 -> a few ms instead of ~0.3 s on the host.
//
// Jump-ahead (default): the stream is cut into segments of 2^16 draws.  CTA c jumps the seeded
// window straight to its first segment with the precomputed polynomials g = x^J mod p(x)
// (tools/mt_jump_tables.cpp; J = b 2^24 then a 2^16): the 19937-term sequence from the window is
// generated in shared memory and word j of the jumped window is the XOR of y_{i+j} over the set
// coefficients i of g (g(T) W with T the one-step map).  Every CTA then twists its own segments,
// so ~150 CTAs run the stream in parallel instead of one.  Same bits as the sequential kernel.
#include <array>
#include <cstring>
#include <mutex>

#include "runtime.hpp"
#include "rng.hpp"

namespace bosp {
inline namespace b200 {

namespace {

constexpr int kN = 312, kM = 156;

struct MtSeed {
    unsigned long long mt[kN];
};

__device__ __forceinline__ unsigned long long mt_mag(unsigned long long x) {
    return (0ULL - (x & 1ULL)) & 0xB5026F5AA96619E9ULL;
}

__global__ void __launch_bounds__(320) k_mt_fill(MtSeed seed, double* u, int64_t ldu, double* v,
                                                  int64_t ldv, int64_t n, int64_t d, int64_t row0,
                                                  int64_t nloc) {
    __shared__ unsigned long long mt[kN];
    const int t = threadIdx.x;
    if (t < kN) mt[t] = seed.mt[t];
    __syncthreads();
    const int64_t total = 2 * n * d;
    constexpr unsigned long long um = 0xFFFFFFFF80000000ULL, lm = 0x7FFFFFFFULL;
    for (int64_t base = 0; base < total; base += kN) {
        // twist, first half: new mt[i] from old mt[i], mt[i+1], mt[i+M]
        unsigned long long nv = 0;
        if (t < kN - kM) {
            const unsigned long long x = (mt[t] & um) | (mt[t + 1] & lm);
            nv = mt[t + kM] ^ (x >> 1) ^ mt_mag(x);
        }
        // second half reads old mt[i], mt[i+1] (i+1 <= N-1) before anyone overwrites them
        unsigned long long xo = 0;
        if (t >= kN - kM && t < kN - 1) xo = (mt[t] & um) | (mt[t + 1] & lm);
        const unsigned long long last_hi = mt[kN - 1] & um;
        __syncthreads();
        if (t < kN - kM) mt[t] = nv;
        __syncthreads();
        if (t >= kN - kM && t < kN - 1) nv = mt[t + kM - kN] ^ (xo >> 1) ^ mt_mag(xo);
        if (t == kN - 1) {
            const unsigned long long x = last_hi | (mt[0] & lm);
            nv = mt[kM - 1] ^ (x >> 1) ^ mt_mag(x);
        }
        __syncthreads();
        if (t >= kN - kM && t < kN) mt[t] = nv;
        __syncthreads();
        if (t < kN) {
            const int64_t k = base + t;
            if (k < total) {
                unsigned long long y = mt[t];
                y ^= (y >> 29) & 0x5555555555555555ULL;
                y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
                y ^= (y << 37) & 0xFFF7EEE000000000ULL;
                y ^= (y >> 43);
                double r = __ull2double_rn(y) * 0x1p-64;
                if (r >= 1.0) r = 0x1.fffffffffffffp-1;
                r = __dadd_rn(__dmul_rn(r, 2.0), -1.0);
                const int64_t c = k / n, grow = k - c * n;   // global row of this draw
                const int64_t row = grow - row0;            // this rank keeps its window
                if (row >= 0 && row < nloc) {
                    if (c < d) u[c * ldu + row] = r;
                    else v[(c - d) * ldv + row] = r;
                }
            }
        }
        // no barrier needed here: the next step only reads mt[] before its first barrier
    }
}

constexpr int64_t kLogSeg = 16, kSeg = 1LL << kLogSeg;  // draws per segment
constexpr int kSeqLen = 20280;                             // >= 19937 + 312, multiple of 312
constexpr int kJumpThreads = 1024;
constexpr size_t kJumpSmem = sizeof(unsigned long long) * (kSeqLen + kN + 3 * kN);

__device__ __forceinline__ unsigned long long mt_twist(unsigned long long a, unsigned long long b) {
    const unsigned long long x = (a & 0xFFFFFFFF80000000ULL) | (b & 0x7FFFFFFFULL);
    return (x >> 1) ^ mt_mag(x);
}

__device__ __forceinline__ double mt_uniform(unsigned long long y) {
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= (y >> 43);
    double r = __ull2double_rn(y) * 0x1p-64;
    if (r >= 1.0) r = 0x1.fffffffffffffp-1;
    return __dadd_rn(__dmul_rn(r, 2.0), -1.0);
}

// y[0..311] holds a window; replace it by g(T) window.  All threads of the block take part.
__device__ void mt_jump(unsigned long long* y, unsigned long long* g, unsigned long long* red,
                        const unsigned long long* __restrict__ poly) {
    const int t = threadIdx.x;
    for (int w = t; w < kN; w += blockDim.x) g[w] = poly[w];
    // extend the sequence: y[m] = y[m-156] ^ twist(y[m-312], y[m-311]), 312 words per barrier
    for (int base = kN; base < kSeqLen; base += kN) {
        __syncthreads();
        if (t < kN) {
            const int m = base + t;
            unsigned long long v;
            if (t < kM) {
                v = y[m - kM] ^ mt_twist(y[m - kN], y[m - kN + 1]);
            } else {
                // y[m-156] is being produced in this step: expand it one level
                const unsigned long long ym156 = y[m - kN] ^ mt_twist(y[m - kN - kM], y[m - kN - kM + 1]);
                const unsigned long long y311 =
                    (t == kN - 1) ? (y[base - kM] ^ mt_twist(y[base - kN], y[base - kN + 1])) : y[m - kN + 1];
                v = ym156 ^ mt_twist(y[m - kN], y311);
            }
            y[m] = v;
        }
    }
    __syncthreads();
    // correlation: word j = XOR over set bits i of g of y[i + j]; three groups split the bits
    if (t < 3 * kN) {
        const int q = t / kN, j = t - q * kN;
        unsigned long long acc = 0;
        for (int w = q * (kN / 3); w < (q + 1) * (kN / 3); ++w) {
            unsigned long long bits = g[w];
            const unsigned long long* yy = y + 64 * w + j;
            while (bits) {
                const int b = __ffsll(static_cast<long long>(bits)) - 1;
                bits &= bits - 1;
                acc ^= yy[b];
            }
        }
        red[t] = acc;
    }
    __syncthreads();
    if (t < kN) y[t] = red[t] ^ red[t + kN] ^ red[t + 2 * kN];
    __syncthreads();
}

__global__ void __launch_bounds__(kJumpThreads, 1) k_mt_jump_fill(
    MtSeed seed, const unsigned long long* __restrict__ tables, double* u, int64_t ldu, double* v, int64_t ldv,
    int64_t n, int64_t d, int64_t row0, int64_t nloc, int64_t per) {
    extern __shared__ unsigned long long smem[];
    unsigned long long* y = smem;                // sequence / ring buffer
    unsigned long long* g = smem + kSeqLen;      // jump polynomial
    unsigned long long* red = g + kN;            // correlation partials
    const int t = threadIdx.x;
    const int64_t total = 2 * n * d;
    const int64_t s0 = static_cast<int64_t>(blockIdx.x) * per;
    const int64_t first = s0 * kSeg, last = min(total, (s0 + per) * kSeg);
    if (first >= total) return;
    if (t < kN) y[t] = seed.mt[t];
    const int a = static_cast<int>(s0 & 255), b = static_cast<int>(s0 >> 8);
    if (b) mt_jump(y, g, red, tables + (256 + b) * kN);
    if (a) mt_jump(y, g, red, tables + a * kN);
    __syncthreads();
    // twist forward from the window x_{first..first+311}: ring of 3 slots of 312 words; the
    // window of step k is slot k % 3 and its 312 new words (draws base + t) go to the next slot,
    // which nobody reads in this step -> one barrier per step
    constexpr int kRing = 3 * kN;
    int win = 0;
    for (int64_t base = first; base < last; base += kN) {
        const int nxt = win + kN == kRing ? 0 : win + kN;
        if (t < kN) {
            const unsigned long long* x = y + win;  // x[o] = x_{base + o}
            unsigned long long w;
            if (t < kM) {
                w = x[t + kM] ^ mt_twist(x[t], x[t + 1]);
            } else {
                // x_{base+156+t} is produced in this step: expand it one level
                const unsigned long long ym156 = x[t] ^ mt_twist(x[t - kM], x[t - kM + 1]);
                const unsigned long long y311 = (t == kN - 1) ? (x[kM] ^ mt_twist(x[0], x[1])) : x[t + 1];
                w = ym156 ^ mt_twist(x[t], y311);
            }
            y[nxt + t] = w;
            const int64_t k = base + t;
            if (k < last) {
                const double r = mt_uniform(w);
                const int64_t c = k / n, grow = k - c * n;
                const int64_t row = grow - row0;
                if (row >= 0 && row < nloc) {
                    if (c < d) u[c * ldu + row] = r;
                    else v[(c - d) * ldv + row] = r;
                }
            }
        }
        __syncthreads();
        win = nxt;
    }
}

}  // namespace

// Jump polynomials (generated at build time, build/mt_jump_tables.cpp).
extern const uint64_t kMtJump[2][256][312];

namespace {

const unsigned long long* jump_tables() {
    static std::mutex mu;
    static std::array<unsigned long long*, 64> dev{};
    int d = 0;
    BOSP_CUDA(cudaGetDevice(&d));
    std::lock_guard<std::mutex> lk(mu);
    if (!dev[d]) {
        void* p = nullptr;
        BOSP_CUDA(cudaMalloc(&p, sizeof(kMtJump)));
        BOSP_CUDA(cudaMemcpy(p, kMtJump, sizeof(kMtJump), cudaMemcpyHostToDevice));
        BOSP_CUDA(cudaFuncSetAttribute(k_mt_jump_fill, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(kJumpSmem)));
        dev[d] = static_cast<unsigned long long*>(p);
    }
    return dev[d];
}

}  // namespace

void mt_fill_uv(uint64_t seed, const DMat& u, const DMat& v, int64_t n_global, int64_t row0) {
    if (n_global <= 0) n_global = u.rows;
    require(u.rows == v.rows && u.cols == v.cols, "mt_fill_uv: U and V must have equal shape");
    if (u.rows == 0 || u.cols == 0) return;
    MtSeed s;
    s.mt[0] = seed;
    for (int i = 1; i < kN; ++i) s.mt[i] = 6364136223846793005ULL * (s.mt[i - 1] ^ (s.mt[i - 1] >> 62)) + i;
    Runtime& rt = Runtime::get();
    const int64_t total = 2 * n_global * u.cols;
    const int64_t nseg = (total + kSeg - 1) / kSeg;
    static const bool sequential = std::getenv("BOSP_RNG_SEQUENTIAL") != nullptr;
    if (nseg > 65536 || sequential) {  // beyond the tables (2^32 draws): one CTA, whole stream
        LaunchScope ls("rng", 16.0 * u.rows * u.cols, 0.0);
        k_mt_fill<<<1, 320, 0, rt.stream()>>>(s, u.p, u.ld, v.p, v.ld, n_global, u.cols, row0, u.rows);
        BOSP_LAUNCH_CHECK();
        return;
    }
    const unsigned long long* tab = jump_tables();
    const int64_t ncta0 = std::min<int64_t>(nseg, rt.sm_count());
    const int64_t per = (nseg + ncta0 - 1) / ncta0;
    const int64_t ncta = (nseg + per - 1) / per;
    LaunchScope ls("rng", 16.0 * u.rows * u.cols, 0.0);
    k_mt_jump_fill<<<static_cast<unsigned>(ncta), kJumpThreads, kJumpSmem, rt.stream()>>>(
        s, tab, u.p, u.ld, v.p, v.ld, n_global, u.cols, row0, u.rows, per);
    BOSP_LAUNCH_CHECK();
}

}  // namespace b200
}  // namespace bosp
