// Device-clock timing of one kernel launch (Runtime::timer_begin) -- usable inside CUDA graphs,
// where event nodes cannot time individual kernels.  Shared by the SpMM and vector kernels.
#pragma once

namespace bosp {
inline namespace b200 {
namespace {

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Device-clock timing of one launch (Runtime::timer_begin): slot[0] = max(~start) -> earliest
// start, slot[1] = max(end) -> latest end, slot[2] = columns applied (reported by block 0).
struct KTimer {
    unsigned long long* slot;
    __device__ __forceinline__ void start() const {
        if (slot && threadIdx.x == 0) atomicMax(&slot[0], ~gtimer());
    }
    __device__ __forceinline__ void columns(const int* active, int j0, int n, int ncols_total) const {
        // one block reports the applied column count of the whole launch
        if (!slot || threadIdx.x != 0 || blockIdx.x != 0 || blockIdx.y != 0) return;
        (void)j0;
        (void)n;
        int c = ncols_total;
        if (active) {
            c = 0;
            for (int j = 0; j < ncols_total; ++j) c += active[j] != 0;
        }
        slot[2] = static_cast<unsigned long long>(c);
    }
    // one more column applied by this launch (a block owning the column reports it)
    __device__ __forceinline__ void add_column() const {
        if (slot) atomicAdd(&slot[2], 1ull);
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

}  // namespace
}  // namespace b200
}  // namespace bosp
