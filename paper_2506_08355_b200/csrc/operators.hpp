// Operator implementation interface (device apply) behind bosp::LinearOperator.
#pragma once

#include "api.hpp"
#include "runtime.hpp"
#include "sparse_ops.hpp"

namespace bosp {
inline namespace b200 {

class OperatorImpl {
public:
    OperatorImpl(int64_t n, LinearOperator::Kind k) : n_(n), kind_(k), uid_(next_uid()) {}
    virtual ~OperatorImpl();
    // Process-unique id (never reused, unlike the object's address): caches of recorded CUDA
    // graphs key on it, so a rebuilt operator at a recycled address never replays a stale graph.
    uint64_t uid() const { return uid_; }
    // y(:, j) = A x(:, j), x and y device blocks with rows == dim(), y fully overwritten.
    virtual void apply(const DMat& x, const DMat& y) const = 0;
    int64_t dim() const { return n_; }
    LinearOperator::Kind kind() const { return kind_; }
    // Whether apply() only enqueues device work on the solver stream (so it can be recorded
    // into a CUDA graph); host callbacks cannot.
    virtual bool capturable() const { return true; }
    // Allocate whatever apply() of an m-column block allocates lazily (halo / gather buffers),
    // so that a CUDA graph recorded afterwards never allocates during capture.
    virtual void reserve(int64_t m) const { (void)m; }
    // y = A x with x(:,j)^T y(:,j) (the CG's p^T A p) fused into the apply: per-block partials
    // (dot.parts[j * blocks + b]) and, with a ticket, folded into dot.out.  Returns the number of
    // partial blocks per column, 0 when unsupported (nothing done).
    virtual int apply_dot(const DMat& x, const DMat& y, const SpmmDot& dot) const {
        (void)x; (void)y; (void)dot;
        return 0;
    }
    // apply_dot honours the column mask (converged CG columns cost nothing): unrolled CG graphs
    // are only worth it then -- otherwise every idle iteration would still pay a full apply.
    virtual bool has_masked_dot() const { return false; }
    // An apply costs about one streaming pass over x and y (stencil, DIA-stored CSR, diagonal):
    // cheaper than a d-wide DMMA product once d >= 128 (ritz_step then forms K X~ = K (U X^)
    // instead of (K U) X^).
    virtual bool cheap_apply() const { return false; }

private:
    static uint64_t next_uid();
    int64_t n_;
    LinearOperator::Kind kind_;
    uint64_t uid_;
};

// Row-partitioned operators exchange through the communicator inside apply(): recordable into a
// CUDA graph only when the communicator's calls are stream-ordered (NCCL).
bool comm_capturable();

}  // namespace b200
}  // namespace bosp
