// Device-resident building blocks of the BOSP iteration: inner-product Grams, blocked
// biorthogonal projection, MGS-Biorth (coefficient-space recurrence + DMMA products) and the
// batched multi-RHS CG.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "api.hpp"
#include "dense_ops.hpp"
#include "runtime.hpp"

namespace bosp {
inline namespace b200 {

// G = A^T (W B) for the inner product's weight W (identity when unweighted); a x b.
DenseMatrix ip_gram_host(const InnerProduct& ip, const DMat& a, const DMat& b);
// Several Grams in as few launches as possible (<= 4 jobs each) and one device->host copy.
std::vector<DenseMatrix> ip_grams_host(const InnerProduct& ip, const std::vector<std::pair<DMat, DMat>>& pairs);
void ip_gram_dev(const InnerProduct& ip, const DMat& a, const DMat& b, const DMat& g);
// W B into `out` (copy when unweighted).
void apply_weight(const InnerProduct& ip, const DMat& b, const DMat& out);

struct DevBasis {
    DMat p, q;
    // Consecutive bases flagged `group` are mutually biorthogonal (the solver's locked pairs)
    // and are projected out in one concatenated pass (dev_biorth_against).
    bool group = false;
};

// (I - sum P_k Q_k^T) W and (I - sum Q_k P_k^T) Z in place, bases in order (biorth.cpp:116-133).
void dev_biorth_against(const std::vector<DevBasis>& bases, const DMat& w, const DMat& z,
                        const InnerProduct& ip);

// biorth_against with the Grams already known: cross[2i] = Q_i^T W, cross[2i+1] = P_i^T Z for
// bases[i] (unweighted), e.g. sampled by the drift monitor -- products only, up to kMaxSeg bases
// per launch (one concatenated pass: the bases are mutually biorthogonal).
void dev_project_sampled(const std::vector<DevBasis>& bases, const DMat& w, const DMat& z,
                         const std::vector<DenseMatrix>& cross);

struct DevBiorthOutcome {
    int64_t kept = 0;
    std::vector<int64_t> kept_columns, dropped_columns;
    bool second_pass = false;
    // inputs_scratch: the second pass wrote its result into the first `kept` columns of X, Y
    // (instead of P, Q plus a copy back)
    bool result_in_inputs = false;
};
// MGS-Biorth of (X, Y) into (P, Q) (first `kept` columns written; P/Q need >= m columns and
// must not alias X/Y).  Semantics of mgs_biorth (biorth.cpp:102-109); classical -> cgs_biorth.
// The reference's column-sequential gs_biorth (biorth.cpp:19-69) in n-space, pair by pair in
// its exact order, plus the mgs second pass (:73-107): the API-level mgs/cgs_biorth for small m,
// where ill-conditioned inputs (Table 1) need the n-space recurrence, not Grams.
DevBiorthOutcome dev_gs_biorth_seq(const DMat& x, const DMat& y, const DMat& p, const DMat& q,
                                   const InnerProduct& ip, double drop_tol, bool classical);
// gxy_hint: X^T Y already known on the host (unweighted only) -- the pair Grams then compute
// only X^T X and Y^T Y (the drift repair reuses the invariant sample's U^T V, lrep_solver.cpp).
// inputs_scratch: X, Y are dead after the call and may receive the result (see
// DevBiorthOutcome::result_in_inputs).
DevBiorthOutcome dev_mgs_biorth(const DMat& x, const DMat& y, const DMat& p, const DMat& q,
                                const InnerProduct& ip, double drop_tol = 1e-12,
                                bool classical = false, const DenseMatrix* gxy_hint = nullptr,
                                bool inputs_scratch = false);
// ||P^T Q - I||_2 (biorth.cpp:135-143).
double dev_biorth_residual(const DMat& p, const DMat& q, const InnerProduct& ip);

// One instantiated CUDA graph of a whole batched CG solve: [start] -> while(any active)
// { A p; p^T A p; x, r update; p update }.  Keyed by everything the recorded launches capture.
struct CgGraph {
    uint64_t op = 0;              // OperatorImpl::uid() (never reused, unlike an address)
    uint64_t scratch_gen = 0;     // Runtime::scratch_generation() at recording
    const double *rhs = nullptr, *x = nullptr;
    int64_t ldr = 0, ldx = 0, m = 0, max_iter = 0;
    double tol = 0.0;
    std::string prof_family;  // kernel family timed inside the graph ("" = none)
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    std::map<std::string, int64_t> start_launches, body_launches;
    std::vector<Runtime::ProfPair> prof_pairs;
};

// Batched CG workspace (per operator size / width).
class CgWorkspace {
public:
    void ensure(int64_t n, int64_t m);
    DBlock r, p, ap;
    CgScalars s{};
    int* m_live = nullptr;       // device: live width of a graph recorded wider (see dev_cg)
    int* host_active = nullptr;  // pinned ring
    cudaEvent_t ev[2] = {nullptr, nullptr};
    std::vector<CgGraph> graphs;
    double* pap_parts() const { return parts_; }
    // batched CG iterations of every solve run on this workspace (synchronises)
    int64_t total_sweeps();
    unsigned* ticket() const { return ticket_; }
    ~CgWorkspace();
    static constexpr int64_t kPartsPerRegion = 160 * 512;

private:
    void* scal_ = nullptr;
    double* parts_ = nullptr;
    unsigned* ticket_ = nullptr;
    int64_t m_cap_ = 0;
};
struct DevCgOutcome {
    bool breakdown = false;
    int64_t max_iterations_used = 0;
    int64_t sweeps = 0;  // batched iterations executed
};
// x = CG(A, rhs) column by column with masks (cg.cpp:11-58); x0 = 0 when x0 == nullptr.
// defer_sweeps: the unrolled-graph path returns without waiting for the solve (sweeps = -1;
// the count accumulates on the device, CgWorkspace::total_sweeps()).
DevCgOutcome dev_cg(const LinearOperator& a, const DMat& rhs, const DMat& x, double tol,
                    int64_t max_iter, CgWorkspace& ws, const DMat* x0 = nullptr,
                    bool want_stats = false, bool defer_sweeps = false);

}  // namespace b200
}  // namespace bosp
