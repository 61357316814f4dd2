// LinearOperator implementations: every apply runs on the device stream.  The matrix data of
// dense / CSR / stencil-potential operators is uploaded once at construction (HBM-resident for
// the whole solve); host ApplyFn callbacks are supported by staging through the host, exactly
// once per call, for API compatibility with from_callback (linear_operator.cpp:45-47).
#include <sys/mman.h>

#include "operators.hpp"

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "comm.hpp"
#include "dense_ops.hpp"
#include "runtime.hpp"

namespace bosp {
inline namespace b200 {

// ---- host blocks ----------------------------------------------------------------------------
void* big_alloc_bytes(size_t bytes) {
    constexpr size_t kHuge = size_t(2) << 20;
    void* p = nullptr;
    if (bytes >= kHuge) {
        if (posix_memalign(&p, kHuge, (bytes + kHuge - 1) / kHuge * kHuge) != 0) throw std::bad_alloc();
        madvise(p, (bytes + kHuge - 1) / kHuge * kHuge, MADV_HUGEPAGE);
    } else {
        p = std::malloc(bytes ? bytes : 1);
        if (!p) throw std::bad_alloc();
    }
    return p;
}

void parallel_zero(double* p, size_t n) {
    if (n < (size_t(1) << 18)) {
        std::memset(p, 0, n * sizeof(double));
        return;
    }
    const int64_t chunks = 64;
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < chunks; ++c) {
        const size_t a = n * c / chunks, b = n * (c + 1) / chunks;
        std::memset(p + a, 0, (b - a) * sizeof(double));
    }
}

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
    require(row_offsets.size() == rows + 1, "csr: row_offsets length must be rows+1");
    require(row_offsets.front() == 0 && row_offsets.back() == nnz(), "csr: row_offsets endpoints invalid");
    require(col_indices.size() == values.size(), "csr: col_indices/values length mismatch");
    for (size_t r = 0; r < rows; ++r) {
        require(row_offsets[r] <= row_offsets[r + 1], "csr: row_offsets must be nondecreasing");
        for (size_t k = row_offsets[r]; k + 1 < row_offsets[r + 1]; ++k)
            require(col_indices[k] < col_indices[k + 1], "csr: column indices not strictly increasing");
        for (size_t k = row_offsets[r]; k < row_offsets[r + 1]; ++k)
            require(col_indices[k] < cols, "csr: column index out of range");
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
    void* p = nullptr;
    DevFree(void* q = nullptr) : p(q) {}
    DevFree(DevFree&& o) noexcept : p(o.p) { o.p = nullptr; }
    DevFree& operator=(DevFree&& o) noexcept {
        std::swap(p, o.p);
        return *this;
    }
    DevFree(const DevFree&) = delete;
    DevFree& operator=(const DevFree&) = delete;
    ~DevFree() {
        if (p) Runtime::get().free(p);
    }
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
        FamilyScope fs("dense_apply");
        gram(ColList(t_.view()), ColList(x), x.rows, y.p, y.ld);
    }

private:
    DBlock t_;
};

// CSR (rows rp[0..n], entries from rp[0]) -> SELL-32 in HBM.  Column indices are taken as given
// (a row-partitioned operator passes them already remapped to [local | halo]).
// CSR arrays copied to the device once (pinned-ring staging); SELL-32 and DIA are built from
// them there, nothing of size nnz is built on the host.
struct DevCsr {
    DevFree rp{nullptr}, ci{nullptr}, vv{nullptr};
    int64_t n = 0, nnz = 0;
    DevCsr(int64_t n_, const int64_t* hrp, const int64_t* hci, const double* hvv) : n(n_) {
        Runtime& rt = Runtime::get();
        nnz = hrp[n] - hrp[0];
        rp.p = rt.alloc(sizeof(int64_t) * (n + 1));
        ci.p = rt.alloc(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
        vv.p = rt.alloc(sizeof(double) * std::max<int64_t>(nnz, 1));
        h2d_bytes(rp.p, hrp, sizeof(int64_t) * (n + 1));
        h2d_bytes(ci.p, hci, sizeof(int64_t) * nnz);
        h2d_bytes(vv.p, hvv, sizeof(double) * nnz);
    }
    const int64_t* rowptr() const { return static_cast<const int64_t*>(rp.p); }
    const int64_t* colidx() const { return static_cast<const int64_t*>(ci.p); }
    const double* vals() const { return static_cast<const double*>(vv.p); }
};

struct SellStore {
    DevFree sp{nullptr}, sw{nullptr}, col{nullptr}, val{nullptr};
    SellDev dev;
    SellStore(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv) { build(DevCsr(n, rp, ci, vv)); }
    explicit SellStore(const DevCsr& c) { build(c); }
    void build(const DevCsr& c) {
        const int64_t n = c.n;
        require(n < (int64_t(1) << 31), "from_csr: dimension exceeds int32 device indices");
        Runtime& rt = Runtime::get();
        const int64_t nsl = (n + 31) / 32;
        sp.p = rt.alloc(sizeof(int64_t) * (nsl + 1));
        sw.p = rt.alloc(sizeof(int32_t) * std::max<int64_t>(nsl, 1));
        const int64_t total = sell_layout(n, c.rowptr(), static_cast<int64_t*>(sp.p), static_cast<int32_t*>(sw.p));
        col.p = rt.alloc(sizeof(int32_t) * std::max<int64_t>(total, 1));
        val.p = rt.alloc(sizeof(double) * std::max<int64_t>(total, 1));
        sell_fill(n, c.rowptr(), c.colidx(), c.vals(), static_cast<const int64_t*>(sp.p),
                  static_cast<const int32_t*>(sw.p), static_cast<int32_t*>(col.p), static_cast<double*>(val.p));
        dev.n = n;
        dev.nslices = nsl;
        dev.slice_ptr = static_cast<const int64_t*>(sp.p);
        dev.slice_w = static_cast<const int32_t*>(sw.p);
        dev.col = static_cast<const int32_t*>(col.p);
        dev.val = static_cast<const double*>(val.p);
        dev.nnz = c.nnz;
        rt.sync();  // the CSR copies may be released after this
    }
};

// Banded / stencil-structured CSR (at most kDiaMax distinct column offsets, padding below 2x,
// n even) is stored by diagonals: gather-free, vectorised applies (the CSR row sums in the same
// order).  Everything else is SELL-32.
struct DiaStore {
    DevFree val{nullptr}, mask{nullptr};
    DiaDev dev;
    bool ok = false;
    explicit DiaStore(const DevCsr& c) {
        static const bool off_switch = std::getenv("BOSP_NO_DIA") != nullptr;
        const int64_t n = c.n;
        if (off_switch || n < 64 || (n & 1) || n >= (int64_t(1) << 31)) return;
        int64_t offs[kDiaMax];
        const int nd = dia_offsets(n, c.rowptr(), c.colidx(), offs);
        if (nd <= 0 || static_cast<int64_t>(nd) * n > 2 * c.nnz) return;
        std::sort(offs, offs + nd);
        dev.n = n;
        dev.ndiag = nd;
        for (int d = 0; d < nd; ++d) dev.off[d] = offs[d];
        Runtime& rt = Runtime::get();
        mask.p = rt.alloc(sizeof(uint16_t) * n);
        DBlock mm(2 * kDiaMax, 1);
        auto* vmin = reinterpret_cast<unsigned long long*>(mm.data());
        auto* vmax = vmin + kDiaMax;
        std::vector<unsigned long long> init(2 * kDiaMax);
        for (int d = 0; d < kDiaMax; ++d) {
            init[d] = ~0ULL;
            init[kDiaMax + d] = 0ULL;
        }
        BOSP_CUDA(cudaMemcpyAsync(vmin, init.data(), sizeof(unsigned long long) * 2 * kDiaMax,
                                  cudaMemcpyHostToDevice, rt.stream()));
        dia_scan(n, c.rowptr(), c.colidx(), c.vals(), dev, static_cast<uint16_t*>(mask.p), vmin, vmax);
        std::vector<unsigned long long> mm_h(2 * kDiaMax);
        BOSP_CUDA(cudaMemcpyAsync(mm_h.data(), vmin, sizeof(unsigned long long) * 2 * kDiaMax,
                                  cudaMemcpyDeviceToHost, rt.stream()));
        rt.sync();
        int nvar = 0;
        for (int d = 0; d < nd; ++d) {
            const bool constant = mm_h[d] == mm_h[kDiaMax + d];  // identical bit patterns
            double cv;
            std::memcpy(&cv, &mm_h[d], sizeof(double));
            dev.cval[d] = constant ? cv : 0.0;
            dev.vidx[d] = constant ? -1 : nvar++;
        }
        val.p = rt.alloc(sizeof(double) * std::max(nvar, 1) * n);
        if (nvar > 0) {
            BOSP_CUDA(cudaMemsetAsync(val.p, 0, sizeof(double) * nvar * n, rt.stream()));
            dia_fill(n, c.rowptr(), c.colidx(), c.vals(), dev, static_cast<double*>(val.p));
        }
        dev.val = static_cast<const double*>(val.p);
        dev.mask = static_cast<const uint16_t*>(mask.p);
        const uint32_t all = (1u << nd) - 1u;
        dev.full_pair = all | (all << 16);
        for (int d = 0; d < nd; ++d)
            if ((offs[d] & 1) == 0) dev.even |= 1u << d;
        dev.nnz = c.nnz;
        ok = true;
    }
};

class CsrOp final : public OperatorImpl {
public:
    CsrOp(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv)
        : CsrOp(n, DevCsr(n, rp, ci, vv)) {}
    CsrOp(int64_t n, const DevCsr& c) : OperatorImpl(n, LinearOperator::Kind::sparse_csr), d_(c), s_(c) {}
    void apply(const DMat& x, const DMat& y) const override {
        if (d_.ok && dia_fits(x, y)) dia_spmm(d_.dev, x, y);
        else sell_spmm(s_.dev, x, y);
    }
    bool cheap_apply() const override { return d_.ok; }
    int apply_dot(const DMat& x, const DMat& y, const SpmmDot& dot) const override {
        if (d_.ok && dia_fits(x, y)) return dia_spmm(d_.dev, x, y, &dot);
        return sell_spmm(s_.dev, x, y, &dot);
    }
    bool has_masked_dot() const override { return true; }

private:
    // DIA needs 16-byte aligned row pairs; odd leading dimensions take the SELL copy
    static bool dia_fits(const DMat& x, const DMat& y) { return (x.ld & 1) == 0 && (y.ld & 1) == 0; }
    DiaStore d_;
    SellStore s_;
};

// ---- row-partitioned operators ---------------------------------------------------------------
struct RankRange {
    int64_t row0, n;
};

// (row0, n) of every rank through the communicator (collective).
std::vector<RankRange> gather_ranges(int64_t row0, int64_t n) {
    Runtime& rt = Runtime::get();
    Comm* c = rt.comm();
    const int P = c->size();
    DBlock buf(2, P + 1);
    const double mine[2] = {static_cast<double>(row0), static_cast<double>(n)};
    BOSP_CUDA(cudaMemcpyAsync(buf.data() + P * buf.ld(), mine, sizeof(mine), cudaMemcpyHostToDevice, rt.stream()));
    // contiguous send (2 doubles) -> contiguous receive (2*P doubles)
    DBlock flat(2 * P, 1);
    c->allgather(buf.data() + P * buf.ld(), 2, flat.data(), rt.stream());
    std::vector<double> h(static_cast<size_t>(2 * P));
    BOSP_CUDA(cudaMemcpyAsync(h.data(), flat.data(), sizeof(double) * 2 * P, cudaMemcpyDeviceToHost, rt.stream()));
    rt.sync();
    std::vector<RankRange> out(static_cast<size_t>(P));
    for (int r = 0; r < P; ++r) out[r] = {static_cast<int64_t>(h[2 * r]), static_cast<int64_t>(h[2 * r + 1])};
    return out;
}

// Local rows [row0, row0 + n) of a global CSR.  Columns owned by other ranks are fetched into a
// halo block before every apply (grouped point-to-point exchange; only the rows actually
// referenced, planned once at construction) and read by the SpMM kernel from there.
class CsrRowsOp final : public OperatorImpl {
public:
    CsrRowsOp(int64_t n_global, int64_t row0, int64_t n, const int64_t* rp, const int64_t* ci, const double* vv)
        : OperatorImpl(n, LinearOperator::Kind::sparse_csr) {
        Runtime& rt = Runtime::get();
        Comm* comm = rt.comm();
        require(comm != nullptr, "from_csr_rows: no communicator on this thread");
        const int P = comm->size(), me = comm->rank();
        const std::vector<RankRange> rg = gather_ranges(row0, n);
        auto owner = [&](int64_t c) {
            for (int r = 0; r < P; ++r)
                if (c >= rg[r].row0 && c < rg[r].row0 + rg[r].n) return r;
            throw ContractViolation("from_csr_rows: column outside every rank's rows");
        };
        const int64_t base = rp[0], nnz = rp[n] - base;
        std::vector<std::vector<int64_t>> need(static_cast<size_t>(P));
        for (int64_t k = 0; k < nnz; ++k) {
            const int64_t c = ci[k];
            require(c >= 0 && c < n_global, "from_csr_rows: column index out of range");
            if (c < row0 || c >= row0 + n) need[owner(c)].push_back(c);
        }
        for (auto& v : need) {
            std::sort(v.begin(), v.end());
            v.erase(std::unique(v.begin(), v.end()), v.end());
        }
        // how many rows every rank needs from every other: P x P counts, allgathered
        DBlock cnt(P, 1), allc(P * P, 1);
        std::vector<double> mycnt(static_cast<size_t>(P));
        for (int r = 0; r < P; ++r) mycnt[r] = static_cast<double>(need[r].size());
        BOSP_CUDA(cudaMemcpyAsync(cnt.data(), mycnt.data(), sizeof(double) * P, cudaMemcpyHostToDevice, rt.stream()));
        comm->allgather(cnt.data(), P, allc.data(), rt.stream());
        std::vector<double> hc(static_cast<size_t>(P * P));
        BOSP_CUDA(cudaMemcpyAsync(hc.data(), allc.data(), sizeof(double) * P * P, cudaMemcpyDeviceToHost, rt.stream()));
        rt.sync();
        // exchange the index lists (as doubles: exact below 2^53)
        std::vector<DBlock> req_out, req_in;
        std::vector<HaloMsg> sends, recvs;
        for (int r = 0; r < P; ++r) {
            if (r == me) continue;
            const int64_t out_n = static_cast<int64_t>(need[r].size());
            const int64_t in_n = static_cast<int64_t>(hc[static_cast<size_t>(r) * P + me]);
            if (out_n > 0) {
                std::vector<double> tmp(need[r].begin(), need[r].end());
                req_out.emplace_back(out_n, 1);
                BOSP_CUDA(cudaMemcpyAsync(req_out.back().data(), tmp.data(), sizeof(double) * out_n, cudaMemcpyHostToDevice, rt.stream()));
                rt.sync();
                sends.push_back({r, req_out.back().data(), out_n});
            }
            if (in_n > 0) {
                req_in.emplace_back(in_n, 1);
                recvs.push_back({r, req_in.back().data(), in_n});
            }
        }
        comm->exchange(sends, recvs, rt.stream());
        // send plan: the local rows each peer asked for
        for (const HaloMsg& m : recvs) {
            std::vector<double> g(static_cast<size_t>(m.count));
            BOSP_CUDA(cudaMemcpyAsync(g.data(), m.ptr, sizeof(double) * m.count, cudaMemcpyDeviceToHost, rt.stream()));
            rt.sync();
            std::vector<int32_t> loc(static_cast<size_t>(m.count));
            for (size_t i = 0; i < g.size(); ++i) loc[i] = static_cast<int32_t>(static_cast<int64_t>(g[i]) - row0);
            SendPlan sp;
            sp.peer = m.peer;
            sp.cnt = m.count;
            sp.idx.p = upload(loc.data(), loc.size());
            send_.push_back(std::move(sp));
        }
        // receive plan + remapped columns: local -> c - row0, halo -> n + offset(owner) + position
        std::vector<int64_t> off(static_cast<size_t>(P), 0);
        n_halo_ = 0;
        for (int r = 0; r < P; ++r) {
            off[r] = n_halo_;
            if (r != me && !need[r].empty()) {
                recv_.push_back({r, static_cast<int64_t>(need[r].size()), n_halo_});
                n_halo_ += static_cast<int64_t>(need[r].size());
            }
        }
        std::vector<int64_t> cir(static_cast<size_t>(nnz));
        for (int64_t k = 0; k < nnz; ++k) {
            const int64_t c = ci[k];
            if (c >= row0 && c < row0 + n) {
                cir[k] = c - row0;
            } else {
                const int o = owner(c);
                const auto it = std::lower_bound(need[o].begin(), need[o].end(), c);
                cir[k] = n + off[o] + (it - need[o].begin());
            }
        }
        std::vector<int64_t> rpl(rp, rp + n + 1);
        store_ = std::make_unique<SellStore>(n, rpl.data(), cir.data(), vv);
        Runtime::get().sync();
    }
    void apply(const DMat& x, const DMat& y) const override { sell_spmm(with_halo(x), x, y); }
    int apply_dot(const DMat& x, const DMat& y, const SpmmDot& dot) const override {
        return sell_spmm(with_halo(x), x, y, &dot);
    }
    bool has_masked_dot() const override { return true; }
    bool capturable() const override { return comm_capturable(); }
    void reserve(int64_t m) const override { buffers(m); }

private:
    struct SendPlan {
        int peer = 0;
        int64_t cnt = 0;
        DevFree idx{nullptr};
    };
    struct RecvPlan {
        int peer;
        int64_t cnt, off;
    };
    void buffers(int64_t m) const {
        if (!halo_ || halo_->capacity() < m) {
            halo_ = std::make_unique<DBlock>(std::max<int64_t>(n_halo_, 1), m);
            sbuf_.clear();
            rbuf_.clear();
            for (const SendPlan& s : send_) sbuf_.emplace_back(s.cnt, m);
            for (const RecvPlan& r : recv_) rbuf_.emplace_back(r.cnt, m);
        }
    }
    SellDev with_halo(const DMat& x) const {
        Runtime& rt = Runtime::get();
        const int64_t m = x.cols;
        buffers(m);
        std::vector<HaloMsg> sends, recvs;
        for (size_t i = 0; i < send_.size(); ++i) {
            gather_rows(x.p, x.ld, static_cast<const int32_t*>(send_[i].idx.p), send_[i].cnt, m, sbuf_[i].data(),
                        send_[i].cnt, rt.stream());
            sends.push_back({send_[i].peer, sbuf_[i].data(), send_[i].cnt * m});
        }
        for (size_t i = 0; i < recv_.size(); ++i) recvs.push_back({recv_[i].peer, rbuf_[i].data(), recv_[i].cnt * m});
        rt.comm()->exchange(sends, recvs, rt.stream());
        const int64_t ldh = halo_->ld();
        for (size_t i = 0; i < recv_.size(); ++i)
            BOSP_CUDA(cudaMemcpy2DAsync(halo_->data() + recv_[i].off, ldh * sizeof(double), rbuf_[i].data(),
                                        recv_[i].cnt * sizeof(double), recv_[i].cnt * sizeof(double), m,
                                        cudaMemcpyDeviceToDevice, rt.stream()));
        SellDev d = store_->dev;
        d.halo = halo_->data();
        d.ldh = ldh;
        return d;
    }
    std::unique_ptr<SellStore> store_;
    std::vector<SendPlan> send_;
    std::vector<RecvPlan> recv_;
    int64_t n_halo_ = 0;
    mutable std::unique_ptr<DBlock> halo_;
    mutable std::vector<DBlock> sbuf_, rbuf_;
};

// Rows [row0, row0 + n) of a dense operator: stores (A_rows)^T (n_global x n); every apply
// allgathers x and runs the split-K Gram over the full dimension.
class DenseRowsOp final : public OperatorImpl {
public:
    DenseRowsOp(int64_t n_global, int64_t row0, int64_t n, const double* a_rows)
        : OperatorImpl(n, LinearOperator::Kind::dense), t_(n_global, n), ng_(n_global) {
        (void)row0;
        DBlock staged(n, n_global);
        to_device(a_rows, n, n_global, n, staged.view());
        transpose(staged.view(), t_.view());
        rg_ = gather_ranges(row0, n);
        for (const RankRange& r : rg_) nmax_ = std::max(nmax_, r.n);
        Runtime::get().sync();
    }
    void reserve(int64_t m) const override {
        if (!full_ || full_->capacity() < m) {
            full_ = std::make_unique<DBlock>(ng_, m);
            send_ = std::make_unique<DBlock>(nmax_ * m, 1);
            recv_ = std::make_unique<DBlock>(static_cast<int64_t>(rg_.size()) * nmax_ * m, 1);
        }
    }
    void apply(const DMat& x, const DMat& y) const override {
        Runtime& rt = Runtime::get();
        const int64_t m = x.cols, P = static_cast<int64_t>(rg_.size());
        reserve(m);
        BOSP_CUDA(cudaMemcpy2DAsync(send_->data(), nmax_ * sizeof(double), x.p, x.ld * sizeof(double),
                                    x.rows * sizeof(double), m, cudaMemcpyDeviceToDevice, rt.stream()));
        rt.comm()->allgather(send_->data(), nmax_ * m, recv_->data(), rt.stream());
        for (int64_t r = 0; r < P; ++r)
            if (rg_[r].n > 0)
                BOSP_CUDA(cudaMemcpy2DAsync(full_->data() + rg_[r].row0, full_->ld() * sizeof(double),
                                            recv_->data() + r * nmax_ * m, nmax_ * sizeof(double),
                                            rg_[r].n * sizeof(double), m, cudaMemcpyDeviceToDevice, rt.stream()));
        gram(ColList(t_.view()), ColList(full_->cols(0, m)), ng_, y.p, y.ld);
    }
    bool capturable() const override { return comm_capturable(); }

private:
    DBlock t_;
    int64_t ng_;
    std::vector<RankRange> rg_;
    int64_t nmax_ = 0;
    mutable std::unique_ptr<DBlock> full_, send_, recv_;
};

class StencilOp final : public OperatorImpl {
public:
    explicit StencilOp(const StencilSpec& s)
        : OperatorImpl(s.nx * s.ny * s.nz, LinearOperator::Kind::matrix_free_callback) {
        dev_.nx = s.nx;
        dev_.ny = s.ny;
        dev_.nz = s.nz;
        // 3-D when the *global* grid has several z planes (a slab may hold a single plane)
        dev_.dims = (s.s_global > 0 ? s.nz_global : s.nz) > 1 ? 3 : 2;
        dev_.bc = static_cast<int32_t>(s.bc);
        dev_.scale = s.scale;
        dev_.potential = static_cast<int32_t>(s.potential);
        dev_.origin = s.origin;
        dev_.h = s.h;
        dev_.s0 = s.s0;
        dev_.s_global = s.s_global;
        if (s.potential == StencilSpec::Potential::array) {
            require(static_cast<int64_t>(s.v.size()) == dim(), "stencil: potential array size mismatch");
            v_.p = upload(s.v.data(), s.v.size());
            dev_.v = static_cast<const double*>(v_.p);
            Runtime::get().sync();
        }
        const int64_t snl = dev_.dims == 3 ? s.nz : s.ny;
        partitioned_ = s.s_global > 0 && (s.s0 > 0 || s.s0 + snl < s.s_global);
    }
    void apply(const DMat& x, const DMat& y) const override { run(x, y, nullptr); }
    int apply_dot(const DMat& x, const DMat& y, const SpmmDot& dot) const override { return run(x, y, &dot); }
    bool has_masked_dot() const override { return true; }
    bool capturable() const override { return !partitioned_ || comm_capturable(); }
    void reserve(int64_t m) const override {
        if (partitioned_) {
            buffers(m);
            side();
        }
    }
    ~StencilOp() override {
        if (ev_pack_) cudaEventDestroy(ev_pack_);
        if (ev_halo_) cudaEventDestroy(ev_halo_);
        if (side_) cudaStreamDestroy(side_);
        cudaGetLastError();
    }

    bool cheap_apply() const override { return true; }

private:
    // Slab partition along the slowest axis: exchange the first / last local plane of every
    // column with the ranks holding the neighbouring slabs (rank - 1 below, rank + 1 above).
    void buffers(int64_t m) const {
        const int64_t plane = dev_.dims == 3 ? dev_.nx * dev_.ny : dev_.nx;
        if (!lo_ || lo_->capacity() < m) {
            lo_ = std::make_unique<DBlock>(plane, m);
            hi_ = std::make_unique<DBlock>(plane, m);
            slo_ = std::make_unique<DBlock>(plane, m);
            shi_ = std::make_unique<DBlock>(plane, m);
        }
    }
    // side stream + events of the halo overlap, created on first use (before any graph capture:
    // reserve() runs ahead of the CG's capture)
    cudaStream_t side() const {
        if (!side_) {
            BOSP_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
            BOSP_CUDA(cudaEventCreateWithFlags(&ev_pack_, cudaEventDisableTiming));
            BOSP_CUDA(cudaEventCreateWithFlags(&ev_halo_, cudaEventDisableTiming));
        }
        return side_;
    }
    // Slab-partitioned apply with the halo exchange overlapped with the interior planes
    // (SURVEY 8e): pack the two boundary planes on the apply stream, launch the interior, run the
    // exchange on the side stream behind the pack, apply the boundary planes behind the exchange.
    // BOSP_HALO_OVERLAP=0: exchange first, one launch.
    int run(const DMat& x, const DMat& y, const SpmmDot* dot) const {
        static const bool overlap = !std::getenv("BOSP_HALO_OVERLAP") || std::atoi(std::getenv("BOSP_HALO_OVERLAP")) != 0;
        if (!partitioned_ || !overlap) return stencil_spmm(with_halo(x), x, y, dot);
        Runtime& rt = Runtime::get();
        const int me = rt.comm()->rank();
        const int64_t plane = dev_.dims == 3 ? dev_.nx * dev_.ny : dev_.nx;
        const int64_t snl = dev_.dims == 3 ? dev_.nz : dev_.ny;
        const int64_t m = x.cols;
        buffers(m);
        const cudaStream_t sd = side();
        StencilOverlap ov;
        ov.plane = plane;
        ov.has_lo = dev_.s0 > 0;
        ov.has_hi = dev_.s0 + snl < dev_.s_global;
        std::vector<HaloMsg> sends, recvs;
        const size_t pb = plane * sizeof(double);
        if (ov.has_lo) {
            BOSP_CUDA(cudaMemcpy2DAsync(slo_->data(), pb, x.p, x.ld * sizeof(double), pb, m,
                                        cudaMemcpyDeviceToDevice, rt.stream()));
            sends.push_back({me - 1, slo_->data(), plane * m});
            recvs.push_back({me - 1, lo_->data(), plane * m});
        }
        if (ov.has_hi) {
            BOSP_CUDA(cudaMemcpy2DAsync(shi_->data(), pb, x.p + (snl - 1) * plane, x.ld * sizeof(double), pb, m,
                                        cudaMemcpyDeviceToDevice, rt.stream()));
            sends.push_back({me + 1, shi_->data(), plane * m});
            recvs.push_back({me + 1, hi_->data(), plane * m});
        }
        BOSP_CUDA(cudaEventRecord(ev_pack_, rt.stream()));
        ov.exchange = [&] {
            BOSP_CUDA(cudaStreamWaitEvent(sd, ev_pack_, 0));
            rt.comm()->exchange(sends, recvs, sd);
            BOSP_CUDA(cudaEventRecord(ev_halo_, sd));
            BOSP_CUDA(cudaStreamWaitEvent(rt.stream(), ev_halo_, 0));
        };
        StencilDev d = dev_;
        d.halo_lo = ov.has_lo ? lo_->data() : nullptr;
        d.halo_hi = ov.has_hi ? hi_->data() : nullptr;
        return stencil_spmm(d, x, y, dot, &ov);
    }
    StencilDev with_halo(const DMat& x) const {
        if (!partitioned_) return dev_;
        Runtime& rt = Runtime::get();
        const int me = rt.comm()->rank();
        const int64_t plane = dev_.dims == 3 ? dev_.nx * dev_.ny : dev_.nx;
        const int64_t snl = dev_.dims == 3 ? dev_.nz : dev_.ny;
        const int64_t m = x.cols;
        buffers(m);
        const bool has_lo = dev_.s0 > 0, has_hi = dev_.s0 + snl < dev_.s_global;
        std::vector<HaloMsg> sends, recvs;
        const size_t pb = plane * sizeof(double);
        if (has_lo) {
            BOSP_CUDA(cudaMemcpy2DAsync(slo_->data(), pb, x.p, x.ld * sizeof(double), pb, m,
                                        cudaMemcpyDeviceToDevice, rt.stream()));
            sends.push_back({me - 1, slo_->data(), plane * m});
            recvs.push_back({me - 1, lo_->data(), plane * m});
        }
        if (has_hi) {
            BOSP_CUDA(cudaMemcpy2DAsync(shi_->data(), pb, x.p + (snl - 1) * plane, x.ld * sizeof(double), pb, m,
                                        cudaMemcpyDeviceToDevice, rt.stream()));
            sends.push_back({me + 1, shi_->data(), plane * m});
            recvs.push_back({me + 1, hi_->data(), plane * m});
        }
        rt.comm()->exchange(sends, recvs, rt.stream());
        StencilDev d = dev_;
        d.halo_lo = has_lo ? lo_->data() : nullptr;
        d.halo_hi = has_hi ? hi_->data() : nullptr;
        return d;
    }
    DevFree v_{nullptr};
    StencilDev dev_;
    bool partitioned_ = false;
    mutable std::unique_ptr<DBlock> lo_, hi_, slo_, shi_;
    mutable cudaStream_t side_ = nullptr;
    mutable cudaEvent_t ev_pack_ = nullptr, ev_halo_ = nullptr;
};

class ScaledIdentityOp final : public OperatorImpl {
public:
    ScaledIdentityOp(int64_t n, double a) : OperatorImpl(n, LinearOperator::Kind::matrix_free_callback), a_(a) {}
    void apply(const DMat& x, const DMat& y) const override {
        if (a_ == 1.0) copy_block(x, y);
        else axpby(a_, x, 0.0, y);
    }

    bool cheap_apply() const override { return true; }

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

    bool cheap_apply() const override { return true; }

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
    void reserve(int64_t m) const override { base_->reserve(m); }
    bool cheap_apply() const override { return base_->cheap_apply(); }

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
        Runtime& rt = Runtime::get();
        const int st = fn_(rt.device(), x.p, x.ld, y.p, y.ld, x.cols, rt.stream());
        if (st != 0) throw Error("device callback returned " + std::to_string(st));
    }
    bool capturable() const override { return false; }

private:
    LinearOperator::DeviceApplyFn fn_;
};

}  // namespace

OperatorImpl::~OperatorImpl() = default;
bool comm_capturable() {
    const Comm* c = Runtime::get().comm();
    return c && c->stream_capturable();
}
uint64_t OperatorImpl::next_uid() {
    static std::atomic<uint64_t> counter{0};
    return ++counter;
}

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
    // size_t and int64_t share width and representation for every valid index (< 2^63)
    static_assert(sizeof(std::size_t) == sizeof(int64_t), "64-bit size_t expected");
    return LinearOperator(std::make_shared<CsrOp>(static_cast<int64_t>(a.rows),
                                                  reinterpret_cast<const int64_t*>(a.row_offsets.data()),
                                                  reinterpret_cast<const int64_t*>(a.col_indices.data()),
                                                  a.values.data()));
}
LinearOperator LinearOperator::from_csr(int64_t n, const int64_t* rp, const int64_t* ci, const double* vv) {
    return LinearOperator(std::make_shared<CsrOp>(n, rp, ci, vv));
}
LinearOperator LinearOperator::from_csr_rows(int64_t n_global, int64_t row0, int64_t n_local, const int64_t* rp,
                                             const int64_t* ci, const double* vv) {
    if (Runtime::get().nranks() == 1) {  // one rank: plain local CSR
        require(row0 == 0 && n_local == n_global, "from_csr_rows: partial rows without a communicator");
        return from_csr(n_local, rp, ci, vv);
    }
    return LinearOperator(std::make_shared<CsrRowsOp>(n_global, row0, n_local, rp, ci, vv));
}
LinearOperator LinearOperator::from_dense_rows(int64_t n_global, int64_t row0, int64_t n_local, const double* a) {
    if (Runtime::get().nranks() == 1) {
        require(row0 == 0 && n_local == n_global, "from_dense_rows: partial rows without a communicator");
        return from_dense(a, n_local);
    }
    return LinearOperator(std::make_shared<DenseRowsOp>(n_global, row0, n_local, a));
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
