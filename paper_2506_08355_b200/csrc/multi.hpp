// Row-partitioned multi-rank solve (in-process ranks) and the partition rule.
#pragma once

#include <optional>
#include <vector>

#include "api.hpp"

namespace bosp {
inline namespace b200 {

// A global operator description that every rank slices (host memory, read only).
struct GlobalOp {
    enum class Kind { dense = 0, csr = 1, stencil = 2 } kind = Kind::csr;
    int64_t n = 0;
    const double* dense = nullptr;  // n x n column-major
    const int64_t* rowptr = nullptr;
    const int64_t* colidx = nullptr;
    const double* vals = nullptr;
    StencilSpec stencil;            // unpartitioned spec (s_global = 0)
};

// Contiguous rows of one rank: balanced over rows (dense / CSR) or over slow-axis planes
// (stencils: z-planes in 3-D, grid rows in 2-D), in rank order.
struct RowSlice {
    int64_t row0 = 0, n = 0;
    int64_t s0 = 0, scount = 0;  // slow-axis planes (stencils)
};
RowSlice row_slice(const GlobalOp& op, int nranks, int rank);
LinearOperator local_operator(const GlobalOp& op, const RowSlice& s);

// nranks ranks on ngpus devices (round-robin; ngpus <= 0 -> all visible).  Eigenvectors are
// returned assembled in global row order; stats are rank 0's with max wall/device time.  No
// nullspace -> each rank runs the partitioned compute_nullspace (as bosp::solve does).
// b (nullable): a B-weighted inner product (inner_product.hpp:12-29); each rank applies its rows
// of B (halo rows / planes exchanged as for K and M).
EigenResult solve_multi(int nranks, int ngpus, const GlobalOp& k, const GlobalOp& m, const GlobalOp* b,
                        const BospConfig& cfg, const std::optional<GeneralizedNullspace>& ns,
                        std::vector<SolverStats>* rank_stats = nullptr);

}  // namespace b200
}  // namespace bosp
