// Public C++ API of the B200 BOSP core -- a source-level drop-in for the reference's
// bosp::solve / LinearOperator plugin surface (proj/include/bosp/solver/bosp_solver.hpp,
// proj/include/bosp/core/linear_operator.hpp).  Same names, argument meaning and exception
// types; everything lives in bosp::b200 (inline) so the mangled symbols never collide with a
// linked reference build.  Vectors of the solve live in HBM; the host sees them only at the
// boundary (operator construction, callbacks, results).
#pragma once

#include <cstdlib>
#include <functional>
#include <memory>
#include <optional>
#include <random>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "common.hpp"
#include "small_dense.hpp"

namespace bosp {
inline namespace b200 {

// Host storage for large blocks: 2 MB-aligned with transparent huge pages requested (n x nev
// eigenvector blocks are tens of MB; 4 KB first-touch faults cost more than the copy), and
// default-initialisation left to the owner (BlockVectors zero-fills in parallel).
template <class T>
struct BigAlloc {
    using value_type = T;
    BigAlloc() = default;
    template <class U>
    BigAlloc(const BigAlloc<U>&) noexcept {}
    T* allocate(size_t n);
    void deallocate(T* p, size_t) noexcept { std::free(p); }
    template <class U>
    void construct(U* p) noexcept { (void)p; }  // no value-initialisation
    template <class U, class... A>
    void construct(U* p, A&&... a) { ::new (static_cast<void*>(p)) U(std::forward<A>(a)...); }
    template <class U>
    bool operator==(const BigAlloc<U>&) const noexcept { return true; }
    template <class U>
    bool operator!=(const BigAlloc<U>&) const noexcept { return false; }
};
void* big_alloc_bytes(size_t bytes);
template <class T>
T* BigAlloc<T>::allocate(size_t n) {
    return static_cast<T*>(big_alloc_bytes(n * sizeof(T)));
}
void parallel_zero(double* p, size_t n);

// Host column-major n x m block (block_vectors.hpp:10-50).
class BlockVectors {
public:
    BlockVectors() = default;
    BlockVectors(int64_t dim, int64_t ncols) : dim_(dim), ncols_(ncols), data_(static_cast<size_t>(dim * ncols)) {
        parallel_zero(data_.data(), data_.size());
    }
    int64_t dim() const { return dim_; }
    int64_t cols() const { return ncols_; }
    bool empty() const { return ncols_ == 0; }
    double& operator()(int64_t i, int64_t j) { return data_[static_cast<size_t>(i + j * dim_)]; }
    double operator()(int64_t i, int64_t j) const { return data_[static_cast<size_t>(i + j * dim_)]; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    // Contiguous view of column j (block_vectors.hpp:23-24).
    std::span<double> col(int64_t j) { return {data_.data() + j * dim_, static_cast<size_t>(dim_)}; }
    std::span<const double> col(int64_t j) const { return {data_.data() + j * dim_, static_cast<size_t>(dim_)}; }
    BlockVectors columns(int64_t first, int64_t count) const;
    void assign_columns(int64_t first, const BlockVectors& src);
    void fill_zero();
    void fill_uniform(std::mt19937_64& rng);
    static BlockVectors hcat(const std::vector<const BlockVectors*>& parts);

private:
    int64_t dim_ = 0, ncols_ = 0;
    std::vector<double, BigAlloc<double>> data_;
};

// CSR (sparse_csr.hpp:12-28): the reference's size_t index vectors at the boundary, int32 on
// the device.
struct SparseMatrixCSR {
    std::size_t rows = 0, cols = 0;
    std::vector<std::size_t> row_offsets, col_indices;
    std::vector<double> values;
    std::size_t nnz() const { return values.size(); }
    void check_invariants() const;
    // y = A x for one column on the host (sparse_csr.hpp:24-25); the solver never calls it --
    // its operators apply on the device.
    void apply(std::span<const double> x, std::span<double> y) const;
};
// Unsorted triplets -> CSR, duplicates summed (sparse_csr.hpp:29-32).
SparseMatrixCSR csr_from_triplets(std::size_t rows, std::size_t cols, std::vector<std::size_t> ti,
                                  std::vector<std::size_t> tj, std::vector<double> tv);

// Structured-grid Laplacian family applied matrix-free by the stencil kernel (new: the
// reference reaches matrix-free operators only through from_callback).
struct StencilSpec {
    int64_t nx = 0, ny = 0, nz = 1;
    enum class Boundary { neumann = 0, dirichlet = 1 } bc = Boundary::neumann;
    double scale = 1.0;
    enum class Potential { none = 0, harmonic = 1, array = 2 } potential = Potential::none;
    double origin = 0.0, h = 1.0;
    std::vector<double> v;  // potential == array (local rows)
    // Row partition along the slowest axis (z for 3-D, y for 2-D): this rank holds slow planes
    // [s0, s0 + nz) (3-D) or [s0, s0 + ny) (2-D) of s_global; nz_global = global z extent.
    // s_global = 0: unpartitioned.
    int64_t s0 = 0, s_global = 0, nz_global = 0;
};

// read_matrix_market (matrix_market.hpp:10-13): coordinate real general|symmetric.
SparseMatrixCSR read_matrix_market(const std::string& path);

class OperatorImpl;

class LinearOperator {
public:
    enum class Kind { dense, sparse_csr, matrix_free_callback };
    using ApplyFn = std::function<void(const BlockVectors&, BlockVectors&)>;
    // Device matrix-free hook (the device analog of ApplyFn): y(:, j) = A x(:, j) for
    // j < ncols, both column-major in HBM of `device`, enqueued on `stream`; returns 0 on
    // success, anything else aborts the solve (bosp::Error "device callback returned <s>").
    using DeviceApplyFn = std::function<int(int device, const double* x, int64_t ldx, double* y, int64_t ldy,
                                            int64_t ncols, cudaStream_t stream)>;

    LinearOperator() = default;
    static LinearOperator from_dense(const DenseMatrix& a);
    static LinearOperator from_dense(const double* colmajor, int64_t n);
    static LinearOperator from_csr(const SparseMatrixCSR& a);
    static LinearOperator from_csr(int64_t n, const int64_t* rowptr, const int64_t* colidx,
                                   const double* vals);
    static LinearOperator from_callback(int64_t dim, ApplyFn fn);
    static LinearOperator from_device_callback(int64_t dim, DeviceApplyFn fn);
    static LinearOperator stencil(const StencilSpec& s);
    static LinearOperator identity(int64_t dim);
    static LinearOperator scaled_identity(int64_t dim, double alpha);
    static LinearOperator diagonal(std::vector<double> d);
    static LinearOperator shifted(const LinearOperator& a, double sigma);
    // Row-partitioned operators (one rank = one thread/process with a communicator, see
    // comm.hpp): this rank's rows [row0, row0 + n_local) of an n_global operator.
    static LinearOperator from_csr_rows(int64_t n_global, int64_t row0, int64_t n_local,
                                        const int64_t* rowptr, const int64_t* colidx_global,
                                        const double* vals);
    // a_rows: n_local x n_global column-major (ld n_local)
    static LinearOperator from_dense_rows(int64_t n_global, int64_t row0, int64_t n_local,
                                          const double* a_rows);

    int64_t dim() const;
    Kind kind() const;
    bool valid() const { return impl_ != nullptr; }

    // out = A x on host blocks (the reference's apply, linear_operator.cpp:94-106).
    void apply(const BlockVectors& x, BlockVectors& out) const;
    BlockVectors apply(const BlockVectors& x) const;
    // out = A x on device blocks (the hot path).
    void apply_device(const DMat& x, const DMat& out) const;

    const OperatorImpl* impl() const { return impl_.get(); }
    explicit LinearOperator(std::shared_ptr<const OperatorImpl> p) : impl_(std::move(p)) {}

private:
    std::shared_ptr<const OperatorImpl> impl_;
};

BlockVectors block_apply(const LinearOperator& op, const BlockVectors& x);

// <x, y> = x^T B y, identity when no weight (inner_product.hpp:12-29).
class InnerProduct {
public:
    InnerProduct() = default;
    explicit InnerProduct(LinearOperator weight) : weight_(std::make_shared<LinearOperator>(std::move(weight))) {}
    bool weighted() const { return weight_ != nullptr; }
    const LinearOperator* weight() const { return weight_.get(); }
    // inner_product.hpp:20-27: B y (a copy when unweighted), x^T B y, sqrt(x^T B x) on host
    // spans (each weighted call is one device apply).
    BlockVectors apply_weight(const BlockVectors& y) const;
    double dot(std::span<const double> x, std::span<const double> y) const;
    double norm(std::span<const double> x) const;

private:
    std::shared_ptr<const LinearOperator> weight_;
};

struct GeneralizedNullspace {
    int64_t r = 0;
    BlockVectors x0, y0;
    bool empty() const { return r == 0; }
};

struct BospConfig {  // bosp_solver.hpp:15-34
    int64_t nev = 1;
    int64_t nb = 0;
    double tol = 1e-8;
    int64_t ngs = 1;
    int64_t s = 3;
    std::optional<bool> moving;
    int64_t max_outer_iter = 500;
    uint64_t rng_seed = 0;
    double inner_cg_tol = 1e-2;
    int64_t inner_cg_max_iter = 20;
    double tol_null = 1e-10;
    std::optional<int64_t> rank_hint;

    int64_t effective_nb() const;
    bool effective_moving() const;
    void validate() const;
};

struct SolverStats {  // bosp_solver.hpp:36-47 (+ B200 counters)
    int64_t iterations = 0;
    int64_t matvec_count = 0;
    int64_t step3_matvecs = 0;
    int64_t step3_vecprods = 0;
    int64_t max_width_u = 0;
    double max_biorth_deviation = 0.0;
    double max_deflation_crossgram = 0.0;
    double final_biorth_deviation = 0.0;
    bool nevconv_monotone = true;
    double wall_seconds = 0.0;
    // B200 additions
    int64_t repairs = 0;            // rebiorthogonalize_state calls
    int64_t cg_iterations = 0;      // batched CG iterations (all solves)
    double host_small_seconds = 0;  // host small-solve time
    double device_seconds = 0;      // CUDA events on the solver stream around the solve
    int64_t gpu_launches = 0;
};

struct EigenResult {  // bosp_solver.hpp:71-81
    std::vector<double> lambdas;
    BlockVectors x, y;
    int64_t iterations = 0;
    std::vector<double> residuals;
    std::vector<std::vector<double>> history;
    std::vector<int64_t> nevconv_history;
    bool converged = false;
    int64_t nev_converged = 0;
    SolverStats stats;
};

struct DeviceState;  // HBM-resident blocks of the solve
// SolverState (bosp_solver.hpp:53-69).  The n-length blocks x, y, p, q, w, z and the locked
// bases live in HBM (dev()); the reference's host-side fields are public mirrors refreshed by
// initialize / iterate_once, so code that reads st.iter, st.nev_conv, st.lambdas, ... compiles
// and behaves as against the reference.
class SolverState {
public:
    SolverState();
    ~SolverState();
    SolverState(SolverState&&) noexcept;
    SolverState& operator=(SolverState&&) noexcept;
    DeviceState& dev() { return *d_; }
    const DeviceState& dev() const { return *d_; }

    std::vector<double> lambdas;    // one per column of x
    std::vector<double> residuals;  // last normalized residual per column of x
    int64_t frozen = 0;
    int64_t nev_conv = 0;           // global converged prefix, never decreases
    std::vector<double> locked_lambdas;
    std::vector<std::vector<double>> residual_history;  // [iteration][eigenindex]
    std::vector<double> last_residual;                  // per global index
    std::vector<int64_t> nevconv_history;
    int64_t iter = 0;
    bool leak_recovered = false;
    SolverStats stats;
    int64_t locked_count() const { return static_cast<int64_t>(locked_lambdas.size()); }

private:
    std::unique_ptr<DeviceState> d_;
};

SolverState initialize(const LinearOperator& k, const LinearOperator& m, const InnerProduct& ip,
                        const GeneralizedNullspace& ns, const BospConfig& cfg);
bool iterate_once(SolverState& st, const LinearOperator& k, const LinearOperator& m,
                  const InnerProduct& ip, const GeneralizedNullspace& ns, const BospConfig& cfg);
// Caller-owned host buffers for the eigenvectors (n x cap each, column-major): when given, the
// result's x / y are written there straight from HBM (through the pinned ring) and
// EigenResult::x / y stay empty -- no intermediate host copy.
struct HostVectorsOut {
    double* x = nullptr;
    double* y = nullptr;
    int64_t cap = 0;
    bool discard = false;  // the caller wants eigenvalues/residuals only: no vector copy-out
};
EigenResult solve(const LinearOperator& k, const LinearOperator& m, const InnerProduct& ip,
                  const BospConfig& cfg, std::optional<GeneralizedNullspace> ns = std::nullopt,
                  const HostVectorsOut* out = nullptr);

struct RegressionFit {
    double alpha = 0.0, beta = 0.0;
    bool degenerate = false;
};
RegressionFit regression_coefficients(const std::vector<std::vector<double>>& history,
                                      int64_t eigenindex, double tol);

// Generalized nullspace (nullspace.hpp:27-39): closed form for T(-1)/T(0) and the detector.
GeneralizedNullspace analytic_nullspace_T(int64_t n);
GeneralizedNullspace compute_nullspace(const LinearOperator& k, const LinearOperator& m,
                                       std::optional<int64_t> r_hint = std::nullopt,
                                       double tol_null = 1e-10,
                                       const InnerProduct& ip = InnerProduct{},
                                       uint64_t seed = 777);

// ---- kernel-level API on host blocks (each call runs on the device) -----------------------
struct BiorthBasis {  // biorth.hpp:12-16
    BlockVectors p, q;
    InnerProduct ip;
};
struct BiorthOutcome {
    BiorthBasis basis;
    std::vector<int64_t> kept_columns, dropped_columns;
};
DenseMatrix block_inner(const InnerProduct& ip, const BlockVectors& x, const BlockVectors& y);
BlockVectors block_product(const BlockVectors& x, const DenseMatrix& c);
void block_axpy(const BlockVectors& x, const DenseMatrix& c, BlockVectors& y);
BiorthOutcome mgs_biorth(const BlockVectors& x, const BlockVectors& y, const InnerProduct& ip,
                         double drop_tol = 1e-12);
BiorthOutcome cgs_biorth(const BlockVectors& x, const BlockVectors& y, const InnerProduct& ip,
                         double drop_tol = 1e-12);
std::pair<BlockVectors, BlockVectors> biorth_against(const std::vector<const BiorthBasis*>& bases,
                                                     const BlockVectors& x, const BlockVectors& y,
                                                     const InnerProduct& ip);
double biorth_residual(const BlockVectors& p, const BlockVectors& q, const InnerProduct& ip);
struct CgResult {
    BlockVectors x;
    bool breakdown = false;
    int64_t max_iterations_used = 0;
};
CgResult cg_solve(const LinearOperator& op, const BlockVectors& rhs, const BlockVectors& x0,
                  double tol, int64_t max_iter);

// ---- the rest of the reference's public helpers (host side) -------------------------------
// kernels.hpp:13-21: unit-stride vector helpers and the host kernel thread count (here: the
// OpenMP threads of the host small dense algebra; the block kernels run on the GPU).
double vdot(std::span<const double> x, std::span<const double> y);
double vnorm2(std::span<const double> x);
void vaxpy(double alpha, std::span<const double> x, std::span<double> y);
void vscale(double alpha, std::span<double> x);
void set_kernel_threads(int nthreads);
int kernel_threads();
// projected_lrep.hpp:27-36: K^ = U^T (K U), M^ = V^T (M V) (Grams on the device) + finish_assembly.
ProjectedLrep assemble_projected(const LinearOperator& k, const LinearOperator& m, const BlockVectors& u,
                                 const BlockVectors& v, const InnerProduct& ip);
ProjectedLrep assemble_projected_applied(const BlockVectors& u, const BlockVectors& ku,
                                         const BlockVectors& v, const BlockVectors& mv);
// nullspace.hpp:21-23: power-iteration estimate of ||op||_2 (applies on the device).
double estimate_operator_norm(const LinearOperator& op, int64_t iters = 50, uint64_t seed = 12345);
// dense_kernels.hpp:24-40 (host small dense algebra).
double condition_number_2(const DenseMatrix& a);
struct LuFactors {
    DenseMatrix lu;
    std::vector<std::size_t> perm;
};
LuFactors lu_factor(DenseMatrix a);
std::vector<double> lu_solve(const LuFactors& f, std::vector<double> b);
DenseMatrix lu_solve(const LuFactors& f, const DenseMatrix& b);
DenseMatrix transpose_times(const DenseMatrix& l, const DenseMatrix& r);

}  // namespace b200
}  // namespace bosp
