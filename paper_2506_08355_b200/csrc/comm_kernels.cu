// Device helpers of the communicators: fixed-order sum over ranks, halo packing.
#include <algorithm>
#include "comm.hpp"

namespace bosp {
inline namespace b200 {

namespace {

__global__ void k_sum_ranks(RankPtrs src, double* __restrict__ dst, int64_t count) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int r = 0; r < src.n; ++r) s += src.p[r][i];  // rank order: identical on every rank
        dst[i] = s;
    }
}

__global__ void k_gather_rows(const double* __restrict__ x, int64_t ldx, const int32_t* __restrict__ idx,
                              int64_t cnt, int64_t m, double* __restrict__ out, int64_t ldo) {
    const int64_t total = cnt * m;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e % cnt, j = e / cnt;
        out[i + j * ldo] = x[idx[i] + j * ldx];
    }
}

}  // namespace

void sum_ranks(const RankPtrs& src, double* dst, int64_t count, cudaStream_t stream) {
    if (count <= 0) return;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((count + 255) / 256, 1184));
    LaunchScope ls("comm");
    k_sum_ranks<<<blocks, 256, 0, stream>>>(src, dst, count);
    BOSP_LAUNCH_CHECK();
}

void gather_rows(const double* x, int64_t ldx, const int32_t* idx, int64_t cnt, int64_t m, double* out,
                 int64_t ldo, cudaStream_t stream) {
    if (cnt <= 0 || m <= 0) return;
    const unsigned blocks = static_cast<unsigned>(std::min<int64_t>((cnt * m + 255) / 256, 2368));
    LaunchScope ls("comm");
    k_gather_rows<<<blocks, 256, 0, stream>>>(x, ldx, idx, cnt, m, out, ldo);
    BOSP_LAUNCH_CHECK();
}

}  // namespace b200
}  // namespace bosp
