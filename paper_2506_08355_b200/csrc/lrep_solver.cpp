// BOSP Algorithm 2 driven from the host with every n-length block resident in HBM.
//
// Mirrors bosp_solver.cpp (initialize :117-177, ritz_step :188-207, iterate_once :211-435,
// assemble_result :439-509, solve :513-536) step for step.  What changes is where the data
// lives and how it moves:
//   * U = [X | P | W] and V = [Y | Q | Z] are single column-major HBM buffers; the active block
//     [X(frozen:), P, W] is a column range, never an hcat copy.
//   * K U, M V, Grams, pullbacks, projections and MGS products are device kernels; only the
//     d x d projected blocks, residual norms and small coefficient matrices cross to the host.
//   * the small LREP and Step-5 algebra run on the host (north star).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <numeric>

#include "api.hpp"
#include "dev_algos.hpp"
#include "operators.hpp"
#include "rng.hpp"

namespace bosp {
inline namespace b200 {

// Wall-time attribution per solver phase (BOSP_PHASES=1 synchronises at each phase end so GPU
// time lands in the phase that issued it; printed at the end of solve()).
enum Phase { PH_INIT, PH_RITZ, PH_SMALL, PH_RESID, PH_STEP5, PH_CG, PH_AGAINST, PH_MGS, PH_STEP7,
             PH_SAMPLE, PH_REPAIR, PH_ASSEMBLE, PH_COUNT };
static const char* kPhaseNames[PH_COUNT] = {"init", "ritz(apply+gram+pullback)", "host small solve",
                                            "residuals", "step5", "cg", "biorth_against", "mgs_biorth",
                                            "step7", "sample_invariants", "repair", "assemble"};

// BOSP_PHASES=1: synchronise at each phase end (GPU time lands in its phase); BOSP_PHASES=2:
// no synchronisation -- host time only (what the host spends issuing each phase)
int phases_mode() {
    static const int m = std::getenv("BOSP_PHASES") ? std::atoi(std::getenv("BOSP_PHASES")) : 0;
    return m;
}
bool phases_enabled() { return phases_mode() == 1; }

struct PhaseClock {
    double acc[PH_COUNT] = {};
    struct Scope {
        PhaseClock* pc;
        Phase ph;
        std::chrono::steady_clock::time_point t0;
        Scope(PhaseClock* p, Phase h) : pc(p), ph(h), t0(std::chrono::steady_clock::now()) {}
        ~Scope() {
            if (phases_enabled()) Runtime::get().sync();
            pc->acc[ph] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
    };
    Scope scope(Phase p) { return Scope(this, p); }
};

struct DeviceState {
    PhaseClock phases;
    int64_t n = 0;
    DBlock U, V;                  // [X | P | W], [Y | Q | Z]
    int64_t wx = 0, wp = 0, ww = 0;
    std::vector<double> lambdas, residuals;
    int64_t frozen = 0, nev_conv = 0;
    std::vector<DBlock> locked_p, locked_q;
    std::vector<double> locked_lambdas;
    std::vector<std::vector<double>> residual_history;
    std::vector<double> last_residual;
    std::vector<int64_t> nevconv_history;
    int64_t iter = 0;
    bool leak_recovered = false;
    SolverStats stats;
    // nullspace on device
    DBlock x0, y0;
    // workspaces
    DBlock ku, mv, xt, yt, kxt, myt, xtb, ytb, pt, qt, rz, rw, zg, wg, tmp;
    DBlock small;                 // device copies of small coefficient matrices
    DBlock scal;                  // per-column scalars: 4 slots of scal_cap doubles
    int64_t scal_cap = 0;         // >= every window width / block size of this solve
    CgWorkspace cg;
    bool cg_deferred = false;  // some CG sweep counts are still on the device (cg.total_sweeps)

    int64_t width() const { return wx + wp + ww; }
    DMat X() const { return U.cols(0, wx); }
    DMat Y() const { return V.cols(0, wx); }
    int64_t locked_count() const { return static_cast<int64_t>(locked_lambdas.size()); }
};

SolverState::SolverState() : d_(std::make_unique<DeviceState>()) {}
SolverState::~SolverState() = default;
SolverState::SolverState(SolverState&&) noexcept = default;
SolverState& SolverState::operator=(SolverState&&) noexcept = default;

namespace {
// Refresh the reference-visible host fields of SolverState from the device-side state
// (histories grow by the rows added since the last refresh).
void mirror_state(SolverState& ss) {
    const DeviceState& st = ss.dev();
    ss.lambdas = st.lambdas;
    ss.residuals = st.residuals;
    ss.frozen = st.frozen;
    ss.nev_conv = st.nev_conv;
    ss.locked_lambdas = st.locked_lambdas;
    for (size_t i = ss.residual_history.size(); i < st.residual_history.size(); ++i)
        ss.residual_history.push_back(st.residual_history[i]);
    for (size_t i = ss.nevconv_history.size(); i < st.nevconv_history.size(); ++i)
        ss.nevconv_history.push_back(st.nevconv_history[i]);
    ss.last_residual = st.last_residual;
    ss.iter = st.iter;
    ss.leak_recovered = st.leak_recovered;
    ss.stats = st.stats;
}
}  // namespace

int64_t BospConfig::effective_nb() const {
    if (nb > 0) return std::min(nb, nev);
    const int64_t by_rule = (nev + 4) / 5;
    return std::max<int64_t>(1, std::min<int64_t>(by_rule, 150));
}

bool BospConfig::effective_moving() const {
    if (moving.has_value()) return *moving;
    return nev > 3 * effective_nb();
}

void BospConfig::validate() const {
    if (nev <= 0) throw ContractViolation("BospConfig: nev must be positive");
    if (effective_nb() > nev) throw ContractViolation("BospConfig: nb exceeds nev");
    if (s < 2) throw ContractViolation("BospConfig: s must be >= 2");
    if (!(tol > 0.0)) throw ContractViolation("BospConfig: tol must be positive");
}

namespace {

using Clock = std::chrono::steady_clock;

bool debug_enabled() {
    static const bool on = std::getenv("BOSP_DEBUG") != nullptr;
    return on;
}

double secs(Clock::time_point a, Clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

void ensure_block(DBlock& b, int64_t rows, int64_t cols) {
    if (b.rows() != rows || b.capacity() < cols) b = DBlock(rows, std::max<int64_t>(cols, 1));
    b.set_cols(cols);
}

std::vector<DevBasis> deflation_bases(const DeviceState& st) {
    std::vector<DevBasis> bases;
    if (st.x0.ncols() > 0) bases.push_back({st.x0.view(), st.y0.view()});
    for (size_t i = 0; i < st.locked_p.size(); ++i)
        bases.push_back({st.locked_p[i].view(), st.locked_q[i].view(), true});
    return bases;
}

// Per-column scalar slots on the device: 0 = window lambdas, 1 = residual numerators,
// 2 = residual denominators, 3 = Step-6 block lambdas; each scal_cap doubles.
double* scal_slot(DeviceState& st, int slot) {
    if (st.scal.rows() != st.scal_cap) ensure_block(st.scal, st.scal_cap, 4);
    return st.scal.data() + slot * st.scal.ld();
}

// Scalars (per-column lambdas) to the device.
const double* upload_scalars(DeviceState& st, const std::vector<double>& v, int slot) {
    require(static_cast<int64_t>(v.size()) <= st.scal_cap, "bosp: scalar slot overflow");
    double* d = scal_slot(st, slot);
    if (!v.empty())
        BOSP_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(double) * v.size(), cudaMemcpyHostToDevice, Runtime::get().stream()));
    return d;
}

// Full MGS repair of (U, V) (bosp_solver.cpp:79-95).  gxy_hint: U^T V of the projected pair when
// the caller already has it (see sample_invariants) -- the MGS then Grams only U^T U and V^T V.
// cross (optional): the sampled deflation cross-Grams Q_k^T U, P_k^T V of the same (U, V) --
// the projection against the deflation bases then needs no Grams of its own (config 5: three
// 128-column locked pairs per repair).
void rebiorthogonalize_state(DeviceState& st, const InnerProduct& ip, const DenseMatrix* gxy_hint = nullptr,
                             const std::vector<DenseMatrix>* cross = nullptr) {
    ++st.stats.repairs;
    const int64_t d = st.width();
    const DMat u = st.U.cols(0, d), v = st.V.cols(0, d);
    if (cross && !ip.weighted()) dev_project_sampled(deflation_bases(st), u, v, *cross);
    else dev_biorth_against(deflation_bases(st), u, v, ip);
    DBlock nu(st.n, st.U.capacity()), nv(st.n, st.V.capacity());
    DevBiorthOutcome out = dev_mgs_biorth(u, v, nu.cols(0, d), nv.cols(0, d), ip, 1e-12, false, gxy_hint, true);
    if (!out.dropped_columns.empty())
        throw NumericalAbort("bosp: rebiorthogonalization dropped columns");
    if (out.result_in_inputs) return;  // the second pass wrote U, V in place
    nu.set_cols(st.U.ncols());
    nv.set_cols(st.V.ncols());
    std::swap(st.U, nu);
    std::swap(st.V, nv);
}

// Returns the max |U^T V - I| deviation and records cross-Gram statistics (:63-76).
// projected_gxy (optional): U'^T V' of the pair after biorth_against(deflation bases), i.e. what
// the drift repair's MGS would Gram first.  With U' = U - P_k (Q_k^T U), V' = V - Q_k (P_k^T V)
// and P_k^T Q_k = I: U'^T V' = U^T V - sum_k (Q_k^T U)^T (P_k^T V) -- every term is one of the
// Grams sampled here (cross terms between bases are products of two cross-Grams, ~1e-26).
double sample_invariants(DeviceState& st, const InnerProduct& ip, DenseMatrix* projected_gxy = nullptr,
                         std::vector<DenseMatrix>* cross = nullptr) {
    const int64_t d = st.width();
    const DMat u = st.U.cols(0, d), v = st.V.cols(0, d);
    // U^T V and every deflation cross-Gram in one batch, one device->host copy
    std::vector<std::pair<DMat, DMat>> pairs{{u, v}};
    for (const DevBasis& b : deflation_bases(st)) {
        pairs.push_back({b.q, u});
        pairs.push_back({b.p, v});
    }
    std::vector<DenseMatrix> gs = ip_grams_host(ip, pairs);
    if (projected_gxy && !ip.weighted()) {
        *projected_gxy = gs[0];
        for (size_t i = 1; i + 1 < gs.size(); i += 2) {
            const DenseMatrix corr = matmul_tn(gs[i], gs[i + 1]);
            for (int64_t j = 0; j < d; ++j)
                for (int64_t r = 0; r < d; ++r) (*projected_gxy)(r, j) -= corr(r, j);
        }
    }
    if (cross) cross->assign(gs.begin() + 1, gs.end());
    DenseMatrix& g = gs[0];
    for (int64_t i = 0; i < g.rows(); ++i) g(i, i) -= 1.0;
    const double dev = g.max_abs();
    st.stats.max_biorth_deviation = std::max(st.stats.max_biorth_deviation, dev);
    double cg = 0.0;
    for (size_t i = 1; i < gs.size(); ++i) cg = std::max(cg, gs[i].max_abs());
    st.stats.max_deflation_crossgram = std::max(st.stats.max_deflation_crossgram, cg);
    return dev;
}

struct RitzOut {
    SmallEigenSolution sol;
    int64_t d = 0;
};

// Step 3 (:188-207): K U, M V, projected blocks, host small solve, pullbacks.
RitzOut ritz_step(DeviceState& st, const LinearOperator& k, const LinearOperator& m, int64_t wxa) {
    RitzOut ro;
    const int64_t d = wxa + st.wp + st.ww;
    ro.d = d;
    const DMat u = st.U.cols(st.frozen, d), v = st.V.cols(st.frozen, d);
    ensure_block(st.ku, st.n, d);
    ensure_block(st.mv, st.n, d);
    k.apply_device(u, st.ku.view());
    m.apply_device(v, st.mv.view());
    st.stats.matvec_count += 2 * d;
    st.stats.step3_matvecs += 2 * d;
    st.stats.step3_vecprods += d * d + d;

    DBlock g(d, 2 * d);
    GramJob jobs[2] = {{ColList(u), ColList(st.ku.view()), g.data(), g.ld()},
                       {ColList(v), ColList(st.mv.view()), g.data() + d * g.ld(), g.ld()}};
    // K^ = U^T (K U) and M^ = V^T (M V) are symmetric (K, M symmetric): upper tiles, mirrored --
    // exactly what finish_assembly's (A + A^T)/2 (projected_lrep.cpp:13-46) would make of them
    // up to rounding, for ~60 % of the Gram work at d = 320
    jobs[0].sym = jobs[1].sym = true;
    gram(jobs, 2, st.n);
    Runtime::get().allreduce(g.data(), g.ld() * 2 * d);
    DenseMatrix both(d, 2 * d);
    to_host(g.view().cols_range(0, 2 * d), both.data(), d);
    DenseMatrix khat(d, d), mhat(d, d);
    std::copy(both.data(), both.data() + d * d, khat.data());
    std::copy(both.data() + d * d, both.data() + 2 * d * d, mhat.data());

    static const char* dump = std::getenv("BOSP_DUMP_SMALL");  // diagnostics: "<path prefix>"
    if (dump && d >= 96 && (st.iter == 5 || st.iter == 20)) {
        const std::string path = std::string(dump) + "_it" + std::to_string(st.iter) + "_d" + std::to_string(d) + ".bin";
        if (FILE* f = std::fopen(path.c_str(), "wb")) {
            std::fwrite(khat.data(), sizeof(double), static_cast<size_t>(d * d), f);
            std::fwrite(mhat.data(), sizeof(double), static_cast<size_t>(d * d), f);
            std::fclose(f);
        }
    }
    const auto t0 = Clock::now();
    {
        auto ph = st.phases.scope(PH_SMALL);
        ProjectedLrep proj = finish_assembly(khat, mhat);  // NullspaceLeak propagates
        ro.sol = solve_small_lrep(proj, wxa);
    }
    st.stats.host_small_seconds += secs(t0, Clock::now());

    ensure_block(st.small, d, 2 * wxa);
    to_device(ro.sol.xhat.data(), d, wxa, d, st.small.cols(0, wxa));
    to_device(ro.sol.yhat.data(), d, wxa, d, st.small.cols(wxa, wxa));
    ensure_block(st.xt, st.n, wxa);
    ensure_block(st.yt, st.n, wxa);
    ensure_block(st.kxt, st.n, wxa);
    ensure_block(st.myt, st.n, wxa);
    const double* xh = st.small.data();
    const double* yh = st.small.data() + wxa * st.small.ld();
    const int64_t lds = st.small.ld();
    const int32_t w = static_cast<int32_t>(wxa);
    ProductJob pj[4] = {{ColList(u), xh, lds, w, st.xt.data(), st.xt.ld(), 1.0, 0.0},
                        {ColList(v), yh, lds, w, st.yt.data(), st.yt.ld(), 1.0, 0.0},
                        {ColList(st.ku.view()), xh, lds, w, st.kxt.data(), st.kxt.ld(), 1.0, 0.0},
                        {ColList(st.mv.view()), yh, lds, w, st.myt.data(), st.myt.ld(), 1.0, 0.0}};
    // K X~ and M Y~: the reference pulls them back through linearity, (K U) X^ and (M V) Y^
    // (bosp_solver.cpp:203-206, "no extra matvec").  For operators whose apply is one streaming
    // pass (stencils, DIA-stored CSR) applying them to X~, Y~ is ~10x cheaper than the d-wide
    // DMMA products at d >= 128 (configs 3 and 5: 2 x n x 320 x 192 per iteration) -- the same
    // vectors up to rounding, with the true residual of the stored pairs.
    if (d >= 128 && k.impl()->cheap_apply() && m.impl()->cheap_apply()) {
        product(pj, 2, st.n);
        k.apply_device(st.xt.view(), st.kxt.view());
        m.apply_device(st.yt.view(), st.myt.view());
        st.stats.matvec_count += 2 * wxa;
    } else {
        product(pj, 4, st.n);
    }
    return ro;
}

}  // namespace

SolverState initialize(const LinearOperator& k, const LinearOperator& m, const InnerProduct& ip,
                        const GeneralizedNullspace& ns, const BospConfig& cfg) {
    cfg.validate();
    const int64_t n = k.dim();
    if (m.dim() != n) throw ContractViolation("bosp: K and M dimension mismatch");
    if (ns.r > 0 && (ns.x0.dim() != n || ns.x0.cols() != ns.r || ns.y0.dim() != n || ns.y0.cols() != ns.r))
        throw ContractViolation("bosp: nullspace inconsistent with operators");
    // row-partitioned solves see their local rows; widths follow the global dimension
    Runtime& rt = Runtime::get();
    const int64_t n_global = rt.nranks() > 1 ? rt.n_global() : n;
    const int64_t row0 = rt.nranks() > 1 ? rt.row0() : 0;
    const int64_t budget = n_global - ns.r;
    if (cfg.nev > budget) throw ContractViolation("bosp: nev exceeds the number of positive eigenvalues");

    const int64_t nb = cfg.effective_nb();
    const bool moving = cfg.effective_moving();
    const int64_t wx = std::min(moving ? cfg.s * nb : cfg.nev, budget);
    const int64_t avail = budget - wx;
    const int64_t wp = std::min(nb, avail / 2);
    const int64_t ww = std::min(nb, avail - wp);
    const int64_t d = wx + wp + ww;
    // capacity: a moving step appends P and W to the window (X width <= wx - 2nb + 2nb)
    const int64_t cap = std::max<int64_t>(d, wx + 2 * nb);

    SolverState ss;
    DeviceState& st = ss.dev();
    st.n = n;
    st.wx = wx;
    st.wp = wp;
    st.ww = ww;
    st.scal_cap = std::max<int64_t>({cap, nb, 32});
    if (ns.r > 0) {
        st.x0 = DBlock(n, ns.r);
        st.y0 = DBlock(n, ns.r);
        to_device(ns.x0.data(), n, ns.r, n, st.x0.view());
        to_device(ns.y0.data(), n, ns.r, n, st.y0.view());
    }
    // Steps 1-2: the reference's RNG stream (mt19937_64, U[-1,1], fill order x,p,w,y,q,z --
    // bosp_solver.cpp:144-150) so both solvers start from the same vectors.
    DBlock u(n, cap), v(n, cap);
    const DMat ua = u.cols(0, d), va = v.cols(0, d);
    mt_fill_uv(cfg.rng_seed, ua, va, n_global, row0);  // the exact x,p,w,y,q,z stream, in HBM
    dev_biorth_against(deflation_bases(st), ua, va, ip);
    st.U = DBlock(n, cap);
    st.V = DBlock(n, cap);
    DevBiorthOutcome out = dev_mgs_biorth(ua, va, st.U.cols(0, d), st.V.cols(0, d), ip);
    if (out.kept < d)
        throw InitializationFailure("bosp: column drops during seeding left fewer than the required " +
                                    std::to_string(d) + " columns");
    st.lambdas.assign(static_cast<size_t>(wx), std::numeric_limits<double>::infinity());
    st.residuals.assign(static_cast<size_t>(wx), 1.0);
    st.last_residual.assign(static_cast<size_t>(cfg.nev), 1.0);
    mirror_state(ss);
    return ss;
}

namespace {
bool iterate_device(DeviceState& st, const LinearOperator& k, const LinearOperator& m,
                    const InnerProduct& ip, const GeneralizedNullspace& ns, const BospConfig& cfg) {
    const int64_t n = st.n;
    const int64_t nb = cfg.effective_nb();
    const bool moving = cfg.effective_moving();
    const int64_t budget = (Runtime::get().nranks() > 1 ? Runtime::get().n_global() : n) - ns.r;
    ++st.iter;
    ++st.stats.iterations;

    const int64_t wxa = st.wx - st.frozen;
    st.stats.max_width_u = std::max(st.stats.max_width_u, wxa + st.wp + st.ww);
    RitzOut ro;
    try {
        auto ph = st.phases.scope(PH_RITZ);
        ro = ritz_step(st, k, m, wxa);
    } catch (const NullspaceLeak&) {
        if (st.leak_recovered) throw NumericalAbort("bosp: projected blocks lost positive definiteness twice");
        st.leak_recovered = true;
        rebiorthogonalize_state(st, ip);
        ro = ritz_step(st, k, m, wxa);
    }
    const int64_t d = ro.d;
    const SmallEigenSolution& sol = ro.sol;

    // The refreshed window X~ = U X^ is written back into U only after Step 5 has formed
    // P~ = U P^ from the old U (the reference's `u` is a copy taken before assign_columns).
    auto write_back_window = [&] {
        copy_block(st.xt.view(), st.U.cols(st.frozen, wxa));
        copy_block(st.yt.view(), st.V.cols(st.frozen, wxa));
    };
    for (int64_t j = 0; j < wxa; ++j) st.lambdas[st.frozen + j] = sol.lambdas[j];

    // Step 4: normalized residuals of the window pairs (:246-272)
    DMat xt_b = st.xt.view(), yt_b = st.yt.view();
    if (ip.weighted()) {
        ensure_block(st.xtb, n, wxa);
        ensure_block(st.ytb, n, wxa);
        ip.weight()->apply_device(st.xt.view(), st.xtb.view());
        ip.weight()->apply_device(st.yt.view(), st.ytb.view());
        xt_b = st.xtb.view();
        yt_b = st.ytb.view();
        st.stats.matvec_count += 2 * wxa;
    }
    const double* lam_dev = upload_scalars(st, sol.lambdas, 0);
    double* num_dev = scal_slot(st, 1);
    double* den_dev = scal_slot(st, 2);
    residual_sums(st.kxt.view(), st.myt.view(), xt_b, yt_b, st.xt.view(), st.yt.view(), lam_dev,
                  num_dev, den_dev);
    const int64_t sld = st.scal.ld();  // slots 1 and 2 are adjacent columns of st.scal
    std::vector<double> nd(static_cast<size_t>(2 * sld));
    BOSP_CUDA(cudaMemcpyAsync(nd.data(), num_dev, sizeof(double) * 2 * sld, cudaMemcpyDeviceToHost, Runtime::get().stream()));
    Runtime::get().sync();
    for (int64_t j = 0; j < wxa; ++j) {
        const double lam = sol.lambdas[j];
        st.residuals[st.frozen + j] = std::sqrt(nd[j]) / ((1.0 + lam) * std::sqrt(nd[sld + j]));
    }
    const int64_t base = st.locked_count() + st.frozen;
    int64_t prefix = 0;
    while (prefix < wxa && st.residuals[st.frozen + prefix] < cfg.tol) ++prefix;
    st.nev_conv = std::max(st.nev_conv, base + prefix);
    for (int64_t j = 0; j < wxa && base + j < cfg.nev; ++j) st.last_residual[base + j] = st.residuals[st.frozen + j];
    st.residual_history.push_back(st.last_residual);
    if (!st.nevconv_history.empty() && st.nev_conv < st.nevconv_history.back()) st.stats.nevconv_monotone = false;
    st.nevconv_history.push_back(st.nev_conv);
    if (st.nev_conv >= cfg.nev) {
        write_back_window();
        return true;
    }

    // Step 5 (:288-327): host algebra on the d x nb coefficients, then P~ = U P^, Q~ = V Q^
    const int64_t c0 = std::min(st.nev_conv - base, wxa);
    int64_t nb_eff = std::min(nb, wxa - c0);
    if (wxa + 2 * nb_eff > budget) nb_eff = (budget - wxa) / 2;
    int64_t kp = 0;
    const DMat u_act = st.U.cols(st.frozen, d), v_act = st.V.cols(st.frozen, d);
    if (nb_eff > 0) {
        const auto t0 = Clock::now();
        DenseMatrix t1(d, nb_eff), t2(d, nb_eff);
        for (int64_t j = 0; j < nb_eff; ++j) {
            for (int64_t i = 0; i < d; ++i) {
                t1(i, j) = sol.xhat(i, c0 + j);
                t2(i, j) = sol.yhat(i, c0 + j);
            }
            t1(c0 + j, j) -= 1.0;
            t2(c0 + j, j) -= 1.0;
        }
        DenseMatrix phat = t1, qhat = t2;
        {
            DenseMatrix corr = matmul(sol.xhat, matmul_tn(sol.yhat, t1));
            for (int64_t j = 0; j < nb_eff; ++j)
                for (int64_t i = 0; i < d; ++i) phat(i, j) -= corr(i, j);
        }
        {
            DenseMatrix corr = matmul(sol.yhat, matmul_tn(sol.xhat, t2));
            for (int64_t j = 0; j < nb_eff; ++j)
                for (int64_t i = 0; i < d; ++i) qhat(i, j) -= corr(i, j);
        }
        HostBiorth small = host_mgs_biorth(phat, qhat);
        st.stats.host_small_seconds += secs(t0, Clock::now());
        kp = small.p.cols();
        if (kp > 0) {
            ensure_block(st.small, d, 2 * kp);
            to_device(small.p.data(), d, kp, d, st.small.cols(0, kp));
            to_device(small.q.data(), d, kp, d, st.small.cols(kp, kp));
            ensure_block(st.pt, n, kp);
            ensure_block(st.qt, n, kp);
            ProductJob pj[2] = {{ColList(u_act), st.small.data(), st.small.ld(), static_cast<int32_t>(kp), st.pt.data(), st.pt.ld(), 1.0, 0.0},
                                {ColList(v_act), st.small.data() + kp * st.small.ld(), st.small.ld(), static_cast<int32_t>(kp), st.qt.data(), st.qt.ld(), 1.0, 0.0}};
            product(pj, 2, n);
        }
    }
    write_back_window();

    // Step 6 (:329-388): block Gauss-Seidel with batched inner CG, projection, MGS-Biorth
    int64_t kw = 0;
    const DBlock* w_src = &st.rz;  // where W~, Z~ end up (the MGS output, or its inputs)
    const DBlock* z_src = &st.rw;
    if (nb_eff > 0) {
        std::vector<double> lam_b(sol.lambdas.begin() + c0, sol.lambdas.begin() + c0 + nb_eff);
        const double* lamb = upload_scalars(st, lam_b, 3);
        ensure_block(st.rz, n, nb_eff);
        ensure_block(st.rw, n, nb_eff);
        ensure_block(st.zg, n, nb_eff);
        ensure_block(st.wg, n, nb_eff);
        ensure_block(st.tmp, n, nb_eff);
        lam_axmy(xt_b.cols_range(c0, nb_eff), st.myt.cols(c0, nb_eff), lamb, st.rz.view());
        lam_axmy(yt_b.cols_range(c0, nb_eff), st.kxt.cols(c0, nb_eff), lamb, st.rw.view());
        for (int64_t sweep = 0; sweep < cfg.ngs; ++sweep) {
            // rhs_z = rz (+ lam B W on later sweeps); Z = CG(M, rhs_z)
            DMat rhs_z = st.rz.view();
            if (sweep > 0) {
                copy_block(st.rz.view(), st.tmp.view());
                if (ip.weighted()) {
                    DBlock bw(n, nb_eff);
                    ip.weight()->apply_device(st.wg.view(), bw.view());
                    lam_axpy(bw.view(), lamb, st.tmp.view());
                    st.stats.matvec_count += nb_eff;
                } else {
                    lam_axpy(st.wg.view(), lamb, st.tmp.view());
                }
                rhs_z = st.tmp.view();
            }
            {
                auto phz = st.phases.scope(PH_CG);
                DevCgOutcome cz = dev_cg(m, rhs_z, st.zg.view(), cfg.inner_cg_tol, cfg.inner_cg_max_iter, st.cg,
                                         nullptr, false, true);
                if (cz.sweeps >= 0) st.stats.cg_iterations += cz.sweeps;
                else st.cg_deferred = true;
            }
            // rhs_w = rw + lam B Z; W = CG(K, rhs_w)
            copy_block(st.rw.view(), st.tmp.view());
            if (ip.weighted()) {
                DBlock bz(n, nb_eff);
                ip.weight()->apply_device(st.zg.view(), bz.view());
                lam_axpy(bz.view(), lamb, st.tmp.view());
                st.stats.matvec_count += nb_eff;
            } else {
                lam_axpy(st.zg.view(), lamb, st.tmp.view());
            }
            {
                auto phw = st.phases.scope(PH_CG);
                DevCgOutcome cw = dev_cg(k, st.tmp.view(), st.wg.view(), cfg.inner_cg_tol, cfg.inner_cg_max_iter,
                                         st.cg, nullptr, false, true);
                if (cw.sweeps >= 0) st.stats.cg_iterations += cw.sweeps;
                else st.cg_deferred = true;
            }
        }
        std::vector<DevBasis> bases = deflation_bases(st);
        bases.push_back({st.X(), st.Y()});
        if (kp > 0) bases.push_back({st.pt.view(), st.qt.view()});
        {
            auto ph = st.phases.scope(PH_AGAINST);
            dev_biorth_against(bases, st.wg.view(), st.zg.view(), ip);
        }
        // MGS into the W/Z slots of U/V right after the new P/Q (old P/W are dead here)
        ensure_block(st.rz, n, nb_eff);
        ensure_block(st.rw, n, nb_eff);
        auto phm = st.phases.scope(PH_MGS);
        DevBiorthOutcome wz = dev_mgs_biorth(st.wg.view(), st.zg.view(), st.rz.view(), st.rw.view(), ip,
                                             1e-12, false, nullptr, true);
        kw = wz.kept;
        if (wz.result_in_inputs) {  // the second pass left W~, Z~ in the CG outputs
            w_src = &st.wg;
            z_src = &st.zg;
        }
    }

    // Step 7 (:390-427): U = [X, P~, W~], V = [Y, Q~, Z~]
    copy_block(st.pt.cols(0, kp), st.U.cols(st.wx, kp));
    copy_block(st.qt.cols(0, kp), st.V.cols(st.wx, kp));
    copy_block(w_src->cols(0, kw), st.U.cols(st.wx + kp, kw));
    copy_block(z_src->cols(0, kw), st.V.cols(st.wx + kp, kw));
    st.wp = kp;
    st.ww = kw;

    if (moving) {
        const int64_t conv_window = st.nev_conv - st.locked_count();
        if (conv_window >= 2 * nb && st.wx >= 2 * nb) {
            DBlock lp(n, 2 * nb), lq(n, 2 * nb);
            copy_block(st.U.cols(0, 2 * nb), lp.view());
            copy_block(st.V.cols(0, 2 * nb), lq.view());
            st.locked_p.push_back(std::move(lp));
            st.locked_q.push_back(std::move(lq));
            for (int64_t j = 0; j < 2 * nb; ++j) st.locked_lambdas.push_back(st.lambdas[j]);
            // X = [X_rest, P, W]: shift columns [2nb, width) left by 2nb (through a temp copy)
            const int64_t rest = st.width() - 2 * nb;
            DBlock su(n, std::max<int64_t>(rest, 1)), sv(n, std::max<int64_t>(rest, 1));
            copy_block(st.U.cols(2 * nb, rest), su.cols(0, rest));
            copy_block(st.V.cols(2 * nb, rest), sv.cols(0, rest));
            copy_block(su.cols(0, rest), st.U.cols(0, rest));
            copy_block(sv.cols(0, rest), st.V.cols(0, rest));
            std::vector<double> lam_rest(st.lambdas.begin() + 2 * nb, st.lambdas.end());
            std::vector<double> res_rest(st.residuals.begin() + 2 * nb, st.residuals.end());
            st.wx = rest;
            st.wp = st.ww = 0;
            lam_rest.resize(static_cast<size_t>(st.wx), std::numeric_limits<double>::infinity());
            res_rest.resize(static_cast<size_t>(st.wx), 1.0);
            st.lambdas = std::move(lam_rest);
            st.residuals = std::move(res_rest);
        }
    } else if (st.wx > nb) {
        const int64_t milestone = nb * (st.nev_conv / nb);
        st.frozen = std::max(st.frozen, std::min(milestone, st.wx - nb));
    }

    // invariant sampling doubles as the drift monitor (:429-432)
    double dev;
    DenseMatrix gxy;
    std::vector<DenseMatrix> cross;
    {
        auto ph = st.phases.scope(PH_SAMPLE);
        dev = sample_invariants(st, ip, &gxy, &cross);
    }
    if (debug_enabled())
        std::fprintf(stderr, "[bosp] it=%lld wx=%lld wp=%lld ww=%lld frozen=%lld locked=%lld nev_conv=%lld "
                     "nb_eff=%lld c0=%lld dev=%.3e\n", (long long)st.iter, (long long)st.wx, (long long)st.wp,
                     (long long)st.ww, (long long)st.frozen, (long long)st.locked_count(),
                     (long long)st.nev_conv, (long long)nb_eff, (long long)c0, dev);
    if (dev > 5e-11) {
        auto ph = st.phases.scope(PH_REPAIR);
        rebiorthogonalize_state(st, ip, gxy.rows() == st.width() ? &gxy : nullptr, &cross);
    }
    return false;
}
}  // namespace

bool iterate_once(SolverState& ss, const LinearOperator& k, const LinearOperator& m,
                  const InnerProduct& ip, const GeneralizedNullspace& ns, const BospConfig& cfg) {
    const bool done = iterate_device(ss.dev(), k, m, ip, ns, cfg);
    mirror_state(ss);
    return done;
}

namespace {

EigenResult assemble_result(DeviceState& st, const LinearOperator& k, const LinearOperator& m,
                            const InnerProduct& ip, const BospConfig& cfg, bool converged,
                            const HostVectorsOut* out = nullptr) {
    const int64_t n = st.n;
    const int64_t have = std::min<int64_t>(cfg.nev, st.locked_count() + st.wx);
    std::vector<double> lambdas;
    std::vector<std::pair<const double*, const double*>> cols;  // (x col, y col) device pointers
    int64_t at = 0;
    for (size_t b = 0; b < st.locked_p.size() && at < have; ++b)
        for (int64_t j = 0; j < st.locked_p[b].ncols() && at < have; ++j, ++at) {
            cols.push_back({st.locked_p[b].data() + j * st.locked_p[b].ld(), st.locked_q[b].data() + j * st.locked_q[b].ld()});
            lambdas.push_back(st.locked_lambdas[at]);
        }
    for (int64_t j = 0; at < have && j < st.wx; ++j, ++at) {
        cols.push_back({st.U.data() + j * st.U.ld(), st.V.data() + j * st.V.ld()});
        lambdas.push_back(st.lambdas[j]);
    }
    std::vector<int64_t> order(lambdas.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return lambdas[a] < lambdas[b]; });

    const int64_t h = static_cast<int64_t>(order.size());
    DBlock rx(n, std::max<int64_t>(h, 1)), ry(n, std::max<int64_t>(h, 1));
    rx.set_cols(h);
    ry.set_cols(h);
    EigenResult res;
    res.lambdas.resize(static_cast<size_t>(h));
    for (int64_t j = 0; j < h; ++j) {
        res.lambdas[j] = lambdas[order[j]];
        copy_block(DMat{const_cast<double*>(cols[order[j]].first), n, n, 1}, rx.cols(j, 1));
        copy_block(DMat{const_cast<double*>(cols[order[j]].second), n, n, 1}, ry.cols(j, 1));
    }
    // fresh residuals of the assembled pairs (:486-497)
    DBlock kx(n, std::max<int64_t>(h, 1)), my(n, std::max<int64_t>(h, 1));
    kx.set_cols(h);
    my.set_cols(h);
    k.apply_device(rx.view(), kx.view());
    m.apply_device(ry.view(), my.view());
    DMat bx = rx.view(), by = ry.view();
    DBlock wbx, wby;
    if (ip.weighted()) {
        wbx = DBlock(n, std::max<int64_t>(h, 1));
        wby = DBlock(n, std::max<int64_t>(h, 1));
        wbx.set_cols(h);
        wby.set_cols(h);
        ip.weight()->apply_device(rx.view(), wbx.view());
        ip.weight()->apply_device(ry.view(), wby.view());
        bx = wbx.view();
        by = wby.view();
    }
    DBlock sc(std::max<int64_t>(h, 1), 3);
    to_device(res.lambdas.data(), h, 1, h, sc.cols(0, 1));
    residual_sums(kx.view(), my.view(), bx, by, rx.view(), ry.view(), sc.data(), sc.data() + sc.ld(),
                  sc.data() + 2 * sc.ld());
    std::vector<double> nd(static_cast<size_t>(3 * sc.ld()));
    to_host(sc.view(), nd.data(), sc.ld());
    res.residuals.resize(static_cast<size_t>(h));
    for (int64_t j = 0; j < h; ++j)
        res.residuals[j] = std::sqrt(nd[sc.ld() + j]) / ((1.0 + res.lambdas[j]) * std::sqrt(nd[2 * sc.ld() + j]));

    res.iterations = st.iter;
    res.history = st.residual_history;
    res.nevconv_history = st.nevconv_history;
    res.converged = converged;
    res.nev_converged = std::min(st.nev_conv, cfg.nev);
    if (st.cg_deferred) st.stats.cg_iterations = st.cg.total_sweeps();
    res.stats = st.stats;
    DenseMatrix g = ip_gram_host(ip, rx.view(), ry.view());
    for (int64_t i = 0; i < g.rows(); ++i) g(i, i) -= 1.0;
    res.stats.final_biorth_deviation = g.max_abs();
    if (out && out->discard) {
        res.x = BlockVectors(n, 0);
        res.y = BlockVectors(n, 0);
        return res;
    }
    if (out && out->x && out->y) {
        require(h <= out->cap, "solve: output capacity too small");
        to_host(rx.view(), out->x, n);
        to_host(ry.view(), out->y, n);
        res.x = BlockVectors(n, 0);
        res.y = BlockVectors(n, 0);
        return res;
    }
    res.x = BlockVectors(n, h);
    res.y = BlockVectors(n, h);
    to_host(rx.view(), res.x.data(), n);
    to_host(ry.view(), res.y.data(), n);
    return res;
}

}  // namespace

EigenResult solve(const LinearOperator& k, const LinearOperator& m, const InnerProduct& ip,
                  const BospConfig& cfg, std::optional<GeneralizedNullspace> ns, const HostVectorsOut* out) {
    cfg.validate();
    Runtime& rt = Runtime::get();
    const int64_t launches0 = rt.launches();
    cudaEvent_t ev0, ev1;
    BOSP_CUDA(cudaEventCreate(&ev0));
    BOSP_CUDA(cudaEventCreate(&ev1));
    const auto t0 = Clock::now();
    BOSP_CUDA(cudaEventRecord(ev0, rt.stream()));
    GeneralizedNullspace nullspace =
        ns ? std::move(*ns) : compute_nullspace(k, m, cfg.rank_hint, cfg.tol_null, ip, cfg.rng_seed + 1);
    const auto ti = Clock::now();
    SolverState st = initialize(k, m, ip, nullspace, cfg);
    if (phases_enabled()) rt.sync();
    st.dev().phases.acc[PH_INIT] += secs(ti, Clock::now());
    bool converged = false;
    while (st.iter < cfg.max_outer_iter) {
        if (iterate_once(st, k, m, ip, nullspace, cfg)) {
            converged = true;
            break;
        }
    }
    const auto ta = Clock::now();
    EigenResult res = assemble_result(st.dev(), k, m, ip, cfg, converged, out);
    st.dev().phases.acc[PH_ASSEMBLE] += secs(ta, Clock::now());
    if (std::getenv("BOSP_SYNC_STATS"))
        std::fprintf(stderr, "[bosp] %lld host syncs, %.4f s waiting in them, %lld CG graphs built in %.4f s\n",
                     (long long)rt.sync_count_, rt.sync_wait_s_, (long long)rt.graph_builds_, rt.graph_build_s_);
    if (phases_mode() != 0) {
        std::fprintf(stderr, "[bosp] phase %s times (s), %lld iterations:\n", phases_enabled() ? "wall" : "host",
                     (long long)st.iter);
        for (int i = 0; i < PH_COUNT; ++i)
            std::fprintf(stderr, "[bosp]   %-28s %9.4f\n", kPhaseNames[i], st.dev().phases.acc[i]);
    }
    BOSP_CUDA(cudaEventRecord(ev1, rt.stream()));
    rt.sync();
    res.stats.wall_seconds = secs(t0, Clock::now());
    float ms = 0.f;
    BOSP_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    res.stats.device_seconds = ms * 1e-3;
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    res.stats.gpu_launches = rt.launches() - launches0;
    return res;
}

RegressionFit regression_coefficients(const std::vector<std::vector<double>>& history,
                                      int64_t eigenindex, double tol) {
    std::vector<double> r;
    for (const auto& row : history)
        if (eigenindex < static_cast<int64_t>(row.size())) r.push_back(row[eigenindex]);
    std::vector<std::pair<double, double>> pts;
    for (size_t j = 1; j < r.size(); ++j) {
        if (!(r[j - 1] > 10.0 * tol) || !(r[j] > 10.0 * tol)) continue;
        if (!(r[j - 1] > 0.0) || !(r[j] > 0.0)) continue;
        pts.emplace_back(std::log(r[j - 1]), std::log(r[j]));
    }
    if (pts.size() < 2)
        throw NotEnoughSamples("regression_coefficients: need at least 3 iterations of residuals above 10*tol");
    double sx = 0.0, sy = 0.0;
    for (auto& p : pts) {
        sx += p.first;
        sy += p.second;
    }
    const double mx = sx / pts.size(), my = sy / pts.size();
    double sxx = 0.0, sxy = 0.0;
    for (auto& p : pts) {
        sxx += (p.first - mx) * (p.first - mx);
        sxy += (p.first - mx) * (p.second - my);
    }
    RegressionFit fit;
    if (sxx < 1e-24) {
        fit.degenerate = true;
        fit.alpha = std::exp(my);
        return fit;
    }
    fit.beta = sxy / sxx;
    fit.alpha = std::exp(my - fit.beta * mx);
    return fit;
}

}  // namespace b200
}  // namespace bosp
