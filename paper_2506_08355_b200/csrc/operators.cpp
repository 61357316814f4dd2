// LinearOperator implementations: every apply runs on the device stream.  The matrix data of
// dense / CSR / stencil-potential operators is uploaded once at construction (HBM-resident for
// the whole solve); host ApplyFn callbacks are supported by staging through the host, exactly
// once per call, for API compatibility with from_callback (linear_operator.cpp:45-47).
#include "operators.hpp"

#include <algorithm>
#include <cstring>

#include "dense_ops.hpp"
#include "runtime.hpp"

namespace bosp {
inline namespace b200 {

// ---- host blocks ----------------------------------------------------------------------------
BlockVectors BlockVectors::columns(int64_t first, int64_t count) const {
    require(first + count <= ncols_, "columns: range exceeds block width");
    BlockVectors out(dim_, count);
    if (count > 0) std::memcpy(out.data(), data_.data() + first * dim_, sizeof(double) * count * dim_);
    return out;
}

void BlockVectors::assign_columns(int64_t first, const BlockVectors& src) {
    require(src.dim() == dim_ && first + src.cols() <= ncols_, "assign_columns: shape mismatch");
    if (src.cols() > 0)
        std::memcpy(data_.data() + first * dim_, src.data(), sizeof(double) * src.cols() * dim_);
}

void BlockVectors::fill_zero() { std::fill(data_.begin(), data_.end(), 0.0); }

void BlockVectors::fill_uniform(std::mt19937_64& rng) {
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (double& v : data_) v = dist(rng);
}

BlockVectors BlockVectors::hcat(const std::vector<const BlockVectors*>& parts) {
    int64_t dim = 0, total = 0;
    for (const BlockVectors* p : parts) {
        if (p == nullptr || p->empty()) continue;
        if (dim == 0) dim = p->dim();
        require(p->dim() == dim, "hcat: dimension mismatch");
        total += p->cols();
    }
    BlockVectors out(dim, total);
    int64_t at = 0;
    for (const BlockVectors* p : parts) {
        if (p == nullptr || p->empty()) continue;
        out.assign_columns(at, *p);
        at += p->cols();
    }
    return out;
}

void SparseMatrixCSR::check_invariants() const {
    require(static_cast<int64_t>(row_offsets.size()) == rows + 1, "csr: row_offsets length must be rows+1");
    require(row_offsets.front() == 0 && row_offsets.back() == nnz(), "csr: row_offsets endpoints invalid");
    require(col_indices.size() == values.size(), "csr: col_indices/values length mismatch");
    for (int64_t r = 0; r < rows; ++r) {
        require(row_offsets[r] <= row_offsets[r + 1], "csr: row_offsets must be nondecreasing");
        for (int64_t k = row_offsets[r]; k + 1 < row_offsets[r + 1]; ++k)
            require(col_indices[k] < col_indices[k + 1], "csr: column indices not strictly increasing");
        for (int64_t k = row_offsets[r]; k < row_offsets[r + 1]; ++k)
            require(col_indices[k] >= 0 && col_indices[k] < cols, "csr: column index out of range");
    }
}

// ---- implementations -----------------------------------------------------------------------
namespace {

template <class T>
T* upload(const T* host, size_t count) {
    if (count == 0) return nullptr;
    T* d = static_cast<T*>(Runtime::get().alloc(sizeof(T) * count));
    BOSP_CUDA(cudaMemcpyAsync(d, host, sizeof(T) * count, cudaMemcpyHostToDevice, Runtime::get().stream()));
    return d;
}

struct DevFree {
    void* p;
    ~DevFree() { Runtime::get().free(p); }
};

// Dense operator.  A^T is stored (transposed once on the device at construction), so
// y = A x = (A^T)^T x is a tall-skinny Gram over the long dimension: split-K DMMA tiles keep
// every SM streaming A even when n is small (config 1) and A is read once per apply.
class DenseOp final : public OperatorImpl {
public:
    DenseOp(const double* a, int64_t n) : OperatorImpl(n, LinearOperator::Kind::dense), t_(n, n) {
        DBlock staged(n, n);
        to_device(a, n, n, n, staged.view());
        transpose(staged.view(), t_.view());
        Runtime::get().sync();
    }
    void apply(const DMat& x, const DMat& y) const override {
        gram(ColList(t_.view()), ColList(x), x.rows, y.p, y.ld);
    }

private:
    DBlock t_;
};

class CsrOp final : public OperatorImpl {
public:
    CsrOp(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv)
        : OperatorImpl(n, LinearOperator::Kind::sparse_csr) {
        require(n < (int64_t(1) << 31), "from_csr: dimension exceeds int32 device indices");
        const int64_t nsl = (n + 31) / 32;
        std::vector<int64_t> sp(static_cast<size_t>(nsl + 1), 0);
        std::vector<int32_t> sw(static_cast<size_t>(nsl), 0);
        for (int64_t s = 0; s < nsl; ++s) {
            int64_t w = 0;
            for (int64_t r = s * 32; r < std::min(n, s * 32 + 32); ++r) w = std::max(w, rp[r + 1] - rp[r]);
            sw[s] = static_cast<int32_t>(w);
            sp[s + 1] = sp[s] + 32 * w;
        }
        std::vector<int32_t> col(static_cast<size_t>(sp[nsl]));
        std::vector<double> val(static_cast<size_t>(sp[nsl]), 0.0);
        for (int64_t s = 0; s < nsl; ++s)
            for (int64_t l = 0; l < 32; ++l) {
                const int64_t r = s * 32 + l;
                const int64_t len = r < n ? rp[r + 1] - rp[r] : 0;
                for (int64_t k = 0; k < sw[s]; ++k) {
                    const int64_t at = sp[s] + 32 * k + l;
                    if (k < len) {
                        col[at] = static_cast<int32_t>(ci[rp[r] + k]);
                        val[at] = vv[rp[r] + k];
                    } else {
                        col[at] = static_cast<int32_t>(r < n ? r : 0);
                        val[at] = 0.0;
                    }
                }
            }
        sp_.p = upload(sp.data(), sp.size());
        sw_.p = upload(sw.data(), sw.size());
        col_.p = upload(col.data(), col.size());
        val_.p = upload(val.data(), val.size());
        dev_.n = n;
        dev_.nslices = nsl;
        dev_.slice_ptr = static_cast<const int64_t*>(sp_.p);
        dev_.slice_w = static_cast<const int32_t*>(sw_.p);
        dev_.col = static_cast<const int32_t*>(col_.p);
        dev_.val = static_cast<const double*>(val_.p);
        dev_.nnz = rp[n];
        Runtime::get().sync();  // host staging vectors die at scope exit
    }
    void apply(const DMat& x, const DMat& y) const override { sell_spmm(dev_, x, y); }
    bool apply_dot(const DMat& x, const DMat& y, const SpmmDot& dot) const override {
        sell_spmm(dev_, x, y, &dot);
        return true;
    }

private:
    DevFree sp_{nullptr}, sw_{nullptr}, col_{nullptr}, val_{nullptr};
    SellDev dev_;
};

class StencilOp final : public OperatorImpl {
public:
    explicit StencilOp(const StencilSpec& s)
        : OperatorImpl(s.nx * s.ny * s.nz, LinearOperator::Kind::matrix_free_callback) {
        dev_.nx = s.nx;
        dev_.ny = s.ny;
        dev_.nz = s.nz;
        dev_.bc = static_cast<int32_t>(s.bc);
        dev_.scale = s.scale;
        dev_.potential = static_cast<int32_t>(s.potential);
        dev_.origin = s.origin;
        dev_.h = s.h;
        if (s.potential == StencilSpec::Potential::array) {
            require(static_cast<int64_t>(s.v.size()) == dim(), "stencil: potential array size mismatch");
            v_.p = upload(s.v.data(), s.v.size());
            dev_.v = static_cast<const double*>(v_.p);
            Runtime::get().sync();
        }
    }
    void apply(const DMat& x, const DMat& y) const override { stencil_spmm(dev_, x, y); }
    bool apply_dot(const DMat& x, const DMat& y, const SpmmDot& dot) const override {
        stencil_spmm(dev_, x, y, &dot);
        return true;
    }

private:
    DevFree v_{nullptr};
    StencilDev dev_;
};

class ScaledIdentityOp final : public OperatorImpl {
public:
    ScaledIdentityOp(int64_t n, double a) : OperatorImpl(n, LinearOperator::Kind::matrix_free_callback), a_(a) {}
    void apply(const DMat& x, const DMat& y) const override {
        if (a_ == 1.0) copy_block(x, y);
        else axpby(a_, x, 0.0, y);
    }

private:
    double a_;
};

class DiagOp final : public OperatorImpl {
public:
    explicit DiagOp(const std::vector<double>& d)
        : OperatorImpl(static_cast<int64_t>(d.size()), LinearOperator::Kind::matrix_free_callback) {
        d_.p = upload(d.data(), d.size());
        Runtime::get().sync();
    }
    void apply(const DMat& x, const DMat& y) const override {
        diag_scale(static_cast<const double*>(d_.p), x, y);
    }

private:
    DevFree d_{nullptr};
};

class ShiftedOp final : public OperatorImpl {
public:
    ShiftedOp(std::shared_ptr<const OperatorImpl> base, double sigma)
        : OperatorImpl(base->dim(), LinearOperator::Kind::matrix_free_callback), base_(std::move(base)), sigma_(sigma) {}
    void apply(const DMat& x, const DMat& y) const override {
        base_->apply(x, y);
        axpby(sigma_, x, 1.0, y);  // y += sigma x (linear_operator.cpp:81-92)
    }
    bool capturable() const override { return base_->capturable(); }

private:
    std::shared_ptr<const OperatorImpl> base_;
    double sigma_;
};

class HostCallbackOp final : public OperatorImpl {
public:
    HostCallbackOp(int64_t n, LinearOperator::ApplyFn fn)
        : OperatorImpl(n, LinearOperator::Kind::matrix_free_callback), fn_(std::move(fn)) {}
    void apply(const DMat& x, const DMat& y) const override {
        BlockVectors hx(x.rows, x.cols), hy(x.rows, x.cols);
        to_host(x, hx.data(), x.rows);
        fn_(hx, hy);
        to_device(hy.data(), x.rows, x.cols, x.rows, y);
        Runtime::get().sync();
    }
    bool capturable() const override { return false; }

private:
    LinearOperator::ApplyFn fn_;
};

class DeviceCallbackOp final : public OperatorImpl {
public:
    DeviceCallbackOp(int64_t n, LinearOperator::DeviceApplyFn fn)
        : OperatorImpl(n, LinearOperator::Kind::matrix_free_callback), fn_(std::move(fn)) {}
    void apply(const DMat& x, const DMat& y) const override {
        fn_(x.p, x.ld, y.p, y.ld, x.cols, Runtime::get().stream());
    }
    bool capturable() const override { return false; }

private:
    LinearOperator::DeviceApplyFn fn_;
};

}  // namespace

OperatorImpl::~OperatorImpl() = default;

LinearOperator LinearOperator::from_dense(const DenseMatrix& a) {
    require(a.rows() == a.cols(), "LinearOperator: dense operator must be square");
    return from_dense(a.data(), a.rows());
}
LinearOperator LinearOperator::from_dense(const double* a, int64_t n) {
    return LinearOperator(std::make_shared<DenseOp>(a, n));
}
LinearOperator LinearOperator::from_csr(const SparseMatrixCSR& a) {
    a.check_invariants();
    require(a.rows == a.cols, "LinearOperator: csr operator must be square");
    return LinearOperator(std::make_shared<CsrOp>(a.rows, a.row_offsets.data(), a.col_indices.data(), a.values.data()));
}
LinearOperator LinearOperator::from_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv) {
    return LinearOperator(std::make_shared<CsrOp>(n, rp, ci, vv));
}
LinearOperator LinearOperator::from_callback(int64_t dim, ApplyFn fn) {
    return LinearOperator(std::make_shared<HostCallbackOp>(dim, std::move(fn)));
}
LinearOperator LinearOperator::from_device_callback(int64_t dim, DeviceApplyFn fn) {
    return LinearOperator(std::make_shared<DeviceCallbackOp>(dim, std::move(fn)));
}
LinearOperator LinearOperator::stencil(const StencilSpec& s) {
    require(s.nx > 0 && s.ny > 0 && s.nz > 0, "stencil: grid must be nonempty");
    return LinearOperator(std::make_shared<StencilOp>(s));
}
LinearOperator LinearOperator::identity(int64_t dim) {
    return LinearOperator(std::make_shared<ScaledIdentityOp>(dim, 1.0));
}
LinearOperator LinearOperator::scaled_identity(int64_t dim, double alpha) {
    return LinearOperator(std::make_shared<ScaledIdentityOp>(dim, alpha));
}
LinearOperator LinearOperator::diagonal(std::vector<double> d) {
    return LinearOperator(std::make_shared<DiagOp>(d));
}
LinearOperator LinearOperator::shifted(const LinearOperator& a, double sigma) {
    require(a.valid(), "shifted: invalid base operator");
    return LinearOperator(std::make_shared<ShiftedOp>(a.impl_, sigma));
}

int64_t LinearOperator::dim() const { return impl_ ? impl_->dim() : 0; }
LinearOperator::Kind LinearOperator::kind() const { return impl_ ? impl_->kind() : Kind::matrix_free_callback; }

void LinearOperator::apply_device(const DMat& x, const DMat& out) const {
    require(impl_ != nullptr, "LinearOperator::apply: invalid operator");
    require(x.rows == dim(), "LinearOperator::apply: dimension mismatch");
    require(out.rows == dim() && out.cols == x.cols, "LinearOperator::apply: output shape mismatch");
    if (x.cols == 0) return;
    impl_->apply(x, out);
}

void LinearOperator::apply(const BlockVectors& x, BlockVectors& out) const {
    require(x.dim() == dim(), "LinearOperator::apply: dimension mismatch");
    require(out.dim() == dim() && out.cols() == x.cols(), "LinearOperator::apply: output shape mismatch");
    if (x.cols() == 0) return;
    DBlock dx(x.dim(), x.cols()), dy(x.dim(), x.cols());
    to_device(x.data(), x.dim(), x.cols(), x.dim(), dx.view());
    impl_->apply(dx.view(), dy.view());
    to_host(dy.view(), out.data(), out.dim());
}

BlockVectors LinearOperator::apply(const BlockVectors& x) const {
    BlockVectors out(dim(), x.cols());
    apply(x, out);
    return out;
}

BlockVectors block_apply(const LinearOperator& op, const BlockVectors& x) { return op.apply(x); }

}  // namespace b200
}  // namespace bosp
