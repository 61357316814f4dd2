// MGS-Biorth coefficient recurrence on the device for blocks of m <= 32 columns: the standalone
// launch (row-partitioned solves, whose pair Gram is allreduced between the Gram and this
// kernel).  The algorithm and its exactness rules are in coef_ldu.cuh; single-rank solves run it
// fused into the pair Gram's split reduction (gram_sym_coef, dmma_gemm.cu).
#include "coef_ldu.cuh"
#include "dense_ops.hpp"
#include "runtime.hpp"

namespace bosp {
inline namespace b200 {

namespace {

__global__ void __launch_bounds__(kCoefThreads) k_coef_ldu(const double* __restrict__ z, int64_t ldz, int m, double* c,
                                                 int64_t ldc, int* status, double drop_tol, double cancel_tol) {
    __shared__ double work[kCoefSmem];
    coef_ldu_cta(z, ldz, m, c, ldc, status, drop_tol, cancel_tol, work);
}

}  // namespace

void coef_mgs_dev(const double* z, int64_t ldz, int m, double* c, int64_t ldc, int* status, double drop_tol,
                  double cancel_tol) {
    require(m >= 1 && m <= kCoefM, "coef_mgs_dev: 1..32 columns");
    Runtime& rt = Runtime::get();
    LaunchScope ls("coef");
    k_coef_ldu<<<1, kCoefThreads, 0, rt.stream()>>>(z, ldz, m, c, ldc, status, drop_tol, cancel_tol);
    BOSP_LAUNCH_CHECK();
}

}  // namespace b200
}  // namespace bosp
