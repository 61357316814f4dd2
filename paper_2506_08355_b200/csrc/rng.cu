// Bit-exact std::mt19937_64 + uniform_real_distribution<double>(-1, 1) stream on the device.
//
// The reference seeds X, P, W, Y, Q, Z from one mt19937_64(seed) stream in that order
// (bosp_solver.cpp:144-150, block_vectors.cpp:27-30).  Reproducing the stream keeps the B200
// solver on the reference's starting vectors.  MT19937-64 is sequential across 312-word
// blocks but parallel within one: a single CTA twists the whole state per step (two dependent
// halves separated by a barrier), tempers and converts 312 draws and writes them straight into
// their column of U or V.  ~100k steps for config 2 -> a few ms instead of ~0.3 s on the host.
#include <cstring>

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

}  // namespace

void mt_fill_uv(uint64_t seed, const DMat& u, const DMat& v, int64_t n_global, int64_t row0) {
    if (n_global <= 0) n_global = u.rows;
    require(u.rows == v.rows && u.cols == v.cols, "mt_fill_uv: U and V must have equal shape");
    if (u.rows == 0 || u.cols == 0) return;
    MtSeed s;
    s.mt[0] = seed;
    for (int i = 1; i < kN; ++i) s.mt[i] = 6364136223846793005ULL * (s.mt[i - 1] ^ (s.mt[i - 1] >> 62)) + i;
    Runtime& rt = Runtime::get();
    LaunchScope ls("rng", 16.0 * u.rows * u.cols, 0.0);
    k_mt_fill<<<1, 320, 0, rt.stream()>>>(s, u.p, u.ld, v.p, v.ld, n_global, u.cols, row0, u.rows);
    BOSP_LAUNCH_CHECK();
}

}  // namespace b200
}  // namespace bosp
