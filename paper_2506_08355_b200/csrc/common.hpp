// Shared types for the B200 BOSP core: error taxonomy, CUDA checking, device views.
#pragma once

#include <cuda_runtime.h>

#ifdef __CUDACC__
#define BOSP_HD __host__ __device__
#else
#define BOSP_HD
#endif

#include <cstdint>
#include <stdexcept>
#include <string>

namespace bosp {
inline namespace b200 {

// Exception taxonomy of the reference (proj/include/bosp/core/errors.hpp:9-69), same names and
// meaning so callers can catch the same types; CudaError is new (device failures).
class Error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class ContractViolation : public Error { public: using Error::Error; };
class IngestionError : public Error { public: using Error::Error; };
class NullspaceLeak : public Error { public: using Error::Error; };
class DegenerateSpectrum : public Error { public: using Error::Error; };
class RankMismatch : public Error { public: using Error::Error; };
class InvalidNullspace : public Error { public: using Error::Error; };
class InitializationFailure : public Error { public: using Error::Error; };
class NotEnoughSamples : public Error { public: using Error::Error; };
class NumericalAbort : public Error { public: using Error::Error; };
class CudaError : public Error { public: using Error::Error; };

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define BOSP_CUDA(call)                                                         \
    do {                                                                        \
        cudaError_t bosp_e_ = (call);                                           \
        if (bosp_e_ != cudaSuccess) ::bosp::throw_cuda(bosp_e_, #call, __FILE__, __LINE__); \
    } while (0)

#define BOSP_LAUNCH_CHECK() BOSP_CUDA(cudaGetLastError())

inline void require(bool ok, const char* msg) {
    if (!ok) throw ContractViolation(msg);
}

// Non-owning view of an n x m column-major fp64 block in HBM (column j at p + j*ld).
struct DMat {
    double* p = nullptr;
    int64_t ld = 0;
    int64_t rows = 0;
    int64_t cols = 0;

    double* col(int64_t j) const { return p + j * ld; }
    DMat cols_range(int64_t c0, int64_t nc) const { return DMat{p + c0 * ld, ld, rows, nc}; }
    bool empty() const { return cols == 0 || rows == 0; }
};

// Up to kMaxSeg column segments viewed as one logical block (e.g. U = [X(frozen:), P, W] without
// concatenating copies; the reference's hcat, block_vectors.cpp:32-48, is never materialised).
constexpr int kMaxSeg = 4;
struct ColList {
    const double* p[kMaxSeg];
    int64_t ld[kMaxSeg];
    int32_t start[kMaxSeg + 1];  // prefix sums of segment widths
    int32_t nseg = 0;

    BOSP_HD ColList() {
        for (int i = 0; i < kMaxSeg; ++i) { p[i] = nullptr; ld[i] = 0; start[i] = 0; }
        start[kMaxSeg] = 0;
    }
    explicit ColList(const DMat& m) : ColList() { add(m); }
    ColList& add(const DMat& m) {
        if (m.cols <= 0) return *this;
        if (nseg >= kMaxSeg) throw ContractViolation("ColList: too many segments");
        p[nseg] = m.p;
        ld[nseg] = m.ld;
        start[nseg + 1] = start[nseg] + static_cast<int32_t>(m.cols);
        ++nseg;
        for (int i = nseg + 1; i <= kMaxSeg; ++i) start[i] = start[nseg];
        return *this;
    }
    BOSP_HD int32_t cols() const { return start[nseg]; }
};

}  // namespace b200
}  // namespace bosp
