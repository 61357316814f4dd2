// Row-partitioned solve driven in one process: one host thread per rank, each with its own
// runtime (stream, pool) and a ThreadComm; ranks are spread over `ngpus` devices round-robin
// (several virtual ranks may share one GPU -- that is how the partitioned path is validated on a
// single B200).  Every rank builds its slice of the operators, runs the same bosp::solve on its
// rows, and the results are stitched back in rank order.
#include <cstring>
#include <exception>
#include <string>
#include <thread>

#include "comm.hpp"
#include "multi.hpp"
#include "runtime.hpp"

namespace bosp {
inline namespace b200 {

RowSlice row_slice(const GlobalOp& op, int nranks, int rank) {
    RowSlice s;
    if (op.kind == GlobalOp::Kind::stencil) {
        const bool three = op.stencil.nz > 1;
        const int64_t sg = three ? op.stencil.nz : op.stencil.ny;
        const int64_t plane = three ? op.stencil.nx * op.stencil.ny : op.stencil.nx;
        s.s0 = sg * rank / nranks;
        s.scount = sg * (rank + 1) / nranks - s.s0;
        s.row0 = s.s0 * plane;
        s.n = s.scount * plane;
    } else {
        s.row0 = op.n * rank / nranks;
        s.n = op.n * (rank + 1) / nranks - s.row0;
    }
    return s;
}

LinearOperator local_operator(const GlobalOp& op, const RowSlice& s) {
    switch (op.kind) {
        case GlobalOp::Kind::dense: {
            std::vector<double> rows(static_cast<size_t>(s.n * op.n));
            for (int64_t c = 0; c < op.n; ++c)
                std::memcpy(rows.data() + c * s.n, op.dense + c * op.n + s.row0, sizeof(double) * s.n);
            return LinearOperator::from_dense_rows(op.n, s.row0, s.n, rows.data());
        }
        case GlobalOp::Kind::csr:
            return LinearOperator::from_csr_rows(op.n, s.row0, s.n, op.rowptr + s.row0, op.colidx + op.rowptr[s.row0],
                                                 op.vals + op.rowptr[s.row0]);
        case GlobalOp::Kind::stencil: {
            StencilSpec sp = op.stencil;
            const bool three = op.stencil.nz > 1;
            sp.nz_global = op.stencil.nz;
            if (three) sp.nz = s.scount;
            else sp.ny = s.scount;
            sp.s0 = s.s0;
            sp.s_global = three ? op.stencil.nz : op.stencil.ny;
            if (sp.potential == StencilSpec::Potential::array)
                sp.v.assign(op.stencil.v.begin() + s.row0, op.stencil.v.begin() + s.row0 + s.n);
            return LinearOperator::stencil(sp);
        }
    }
    throw ContractViolation("local_operator: unknown kind");
}

EigenResult solve_multi(int nranks, int ngpus, const GlobalOp& k, const GlobalOp& m, const GlobalOp* b,
                        const BospConfig& cfg, const std::optional<GeneralizedNullspace>& ns,
                        std::vector<SolverStats>* rank_stats) {
    require(nranks >= 1 && nranks <= kMaxRanks, "solve_multi: 1..16 ranks");
    require(k.n == m.n, "solve_multi: K and M dimension mismatch");
    require(!b || b->n == k.n, "solve_multi: B dimension mismatch");
    if (ngpus <= 0) BOSP_CUDA(cudaGetDeviceCount(&ngpus));
    const int64_t n = k.n;
    auto group = std::make_shared<ThreadGroup>(nranks);
    std::vector<EigenResult> res(static_cast<size_t>(nranks));
    std::vector<RowSlice> slices(static_cast<size_t>(nranks));
    std::vector<std::exception_ptr> err(static_cast<size_t>(nranks));
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r) {
        th.emplace_back([&, r] {
            try {
                const int dev = r % ngpus;
                BOSP_CUDA(cudaSetDevice(dev));
                Runtime& rt = Runtime::get();
                rt.set_comm(std::make_shared<ThreadComm>(group, r, dev));
                const RowSlice s = row_slice(k.kind == GlobalOp::Kind::stencil ? k : m, nranks, r);
                slices[r] = s;
                rt.set_rows(n, s.row0);
                LinearOperator kl = local_operator(k, s), ml = local_operator(m, s);
                // B's rows follow the same slice (a stencil slice is whole planes, still rows)
                const InnerProduct ipl = b ? InnerProduct(local_operator(*b, s)) : InnerProduct{};
                std::optional<GeneralizedNullspace> nl;
                if (ns) {
                    nl.emplace();
                    nl->r = ns->r;
                    nl->x0 = BlockVectors(s.n, ns->r);
                    nl->y0 = BlockVectors(s.n, ns->r);
                    for (int64_t c = 0; c < ns->r; ++c) {
                        std::memcpy(nl->x0.col(c).data(), ns->x0.col(c).data() + s.row0, sizeof(double) * s.n);
                        std::memcpy(nl->y0.col(c).data(), ns->y0.col(c).data() + s.row0, sizeof(double) * s.n);
                    }
                }
                res[r] = solve(kl, ml, ipl, cfg, std::move(nl));
                rt.sync();
                rt.set_comm(nullptr);
            } catch (...) {
                err[r] = std::current_exception();
                group->abort();
            }
        });
    }
    for (auto& t : th) t.join();
    // rethrow the root cause: the other ranks only report that a peer aborted the group
    std::exception_ptr first;
    for (auto& e : err) {
        if (!e) continue;
        if (!first) first = e;
        try {
            std::rethrow_exception(e);
        } catch (const std::exception& x) {
            if (std::string(x.what()).find("another rank failed") == std::string::npos) throw;
        }
    }
    if (first) std::rethrow_exception(first);
    EigenResult out = res[0];
    const int64_t h = static_cast<int64_t>(out.lambdas.size());
    out.x = BlockVectors(n, h);
    out.y = BlockVectors(n, h);
    for (int r = 0; r < nranks; ++r)
        for (int64_t c = 0; c < h; ++c) {
            std::memcpy(out.x.col(c).data() + slices[r].row0, res[r].x.col(c).data(), sizeof(double) * slices[r].n);
            std::memcpy(out.y.col(c).data() + slices[r].row0, res[r].y.col(c).data(), sizeof(double) * slices[r].n);
        }
    for (int r = 1; r < nranks; ++r) {
        out.stats.wall_seconds = std::max(out.stats.wall_seconds, res[r].stats.wall_seconds);
        out.stats.device_seconds = std::max(out.stats.device_seconds, res[r].stats.device_seconds);
        out.stats.gpu_launches += res[r].stats.gpu_launches;
    }
    if (rank_stats)
        for (int r = 0; r < nranks; ++r) rank_stats->push_back(res[r].stats);
    return out;
}

}  // namespace b200
}  // namespace bosp
