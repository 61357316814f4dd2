#include <chrono>
#include "runtime.hpp"

#include <algorithm>
#include <cstdio>
#include <cstring>

namespace bosp {
inline namespace b200 {

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    char buf[512];
    std::snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d in %s", cudaGetErrorName(e),
                  cudaGetErrorString(e), file, line, what);
    throw CudaError(buf);
}

Comm::~Comm() = default;

std::mutex& Runtime::setup_mutex() {
    static std::mutex mu;
    return mu;
}

Runtime& Runtime::get() {
    thread_local Runtime rt;
    return rt;
}

Runtime::Runtime() {
    BOSP_CUDA(cudaGetDevice(&device_));
    cudaDeviceProp prop{};
    BOSP_CUDA(cudaGetDeviceProperties(&prop, device_));
    sm_count_ = prop.multiProcessorCount;
    if (prop.major < 10)
        throw CudaError("bosp_b200: this library is built for sm_100a (B200); found sm_" +
                        std::to_string(prop.major) + std::to_string(prop.minor));
    BOSP_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    cudaMemPool_t pool;
    BOSP_CUDA(cudaDeviceGetDefaultMemPool(&pool, device_));
    uint64_t thresh = UINT64_MAX;
    BOSP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
}

Runtime::~Runtime() {
    // Process teardown: the driver reclaims everything; avoid CUDA calls after context death.
}

void* Runtime::alloc(size_t bytes) {
    if (bytes == 0) return nullptr;
    void* p = nullptr;
    BOSP_CUDA(cudaMallocAsync(&p, bytes, stream_));
    return p;
}

void Runtime::free(void* p) {
    if (p) cudaFreeAsync(p, stream_);
}

void Runtime::sync() {
    static const bool stats = std::getenv("BOSP_SYNC_STATS") != nullptr;
    if (!stats) {
        BOSP_CUDA(cudaStreamSynchronize(stream_));
        return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    BOSP_CUDA(cudaStreamSynchronize(stream_));
    sync_count_ += 1;
    sync_wait_s_ += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

double* Runtime::scratch(size_t doubles) {
    if (doubles > scratch_cap_) {
        if (scratch_) free(scratch_);
        scratch_cap_ = doubles + doubles / 2 + 4096;
        scratch_ = static_cast<double*>(alloc(scratch_cap_ * sizeof(double)));
        ++scratch_gen_;
    }
    return scratch_;
}

unsigned int* Runtime::tickets(size_t count) {
    if (count > tickets_cap_) {
        if (tickets_) free(tickets_);
        tickets_cap_ = count + 1024;
        tickets_ = static_cast<unsigned int*>(alloc(tickets_cap_ * sizeof(unsigned int)));
        ++scratch_gen_;
        BOSP_CUDA(cudaMemsetAsync(tickets_, 0, tickets_cap_ * sizeof(unsigned int), stream_));
    }
    return tickets_;
}

double* Runtime::pinned(size_t doubles) {
    if (doubles > pinned_cap_) {
        if (pinned_) {
            sync();
            cudaFreeHost(pinned_);
        }
        pinned_cap_ = doubles + doubles / 2 + 4096;
        BOSP_CUDA(cudaMallocHost(&pinned_, pinned_cap_ * sizeof(double)));
    }
    return pinned_;
}

double* Runtime::stage(int i) {
    if (!stage_[i]) {
        BOSP_CUDA(cudaMallocHost(&stage_[i], kStageDoubles * sizeof(double)));
        BOSP_CUDA(cudaEventCreateWithFlags(&stage_ev_[i], cudaEventDisableTiming));
    }
    return stage_[i];
}

cudaEvent_t Runtime::stage_event(int i) {
    stage(i);
    return stage_ev_[i];
}

void Runtime::count_launch(const char* family) {
    if (capture_sink_) {
        ++(*capture_sink_)[family];
        return;
    }
    ++launches_;
    ++family_launches_[family];
}

void Runtime::add_launches(const std::map<std::string, int64_t>& fam, int64_t times) {
    for (const auto& kv : fam) {
        launches_ += kv.second * times;
        family_launches_[kv.first] += kv.second * times;
    }
}

void Runtime::prof_enable(const std::string& family) {
    prof_family_ = family;
    prof_events_.clear();
    timer_pending_.clear();
    graph_samples_ = ProfReport{0, 0.0, 0.0, 0.0};
    region_depth_ = 0;
}

bool Runtime::prof_on(const char* family) const {
    return !prof_family_.empty() && (region_depth_ > 0 || prof_family_ == family || prof_family_ == "*");
}

bool Runtime::region_open(const char* name) {
    if (prof_family_.empty() || prof_family_ != name) return false;
    ++region_depth_;
    return true;
}

void Runtime::region_close(double algo_bytes, double algo_flops) {
    if (region_depth_ > 0) --region_depth_;
    if (region_depth_ == 0) {
        graph_samples_.region_calls += 1;
        graph_samples_.region_bytes += algo_bytes;
        graph_samples_.region_flops += algo_flops;
    }
}

cudaEvent_t Runtime::take_event() {
    if (!event_pool_.empty()) {
        cudaEvent_t e = event_pool_.back();
        event_pool_.pop_back();
        return e;
    }
    cudaEvent_t e;
    BOSP_CUDA(cudaEventCreate(&e));
    return e;
}

void Runtime::prof_begin(const char* family, double bytes, double flops) {
    if (capture_prof_) return;  // inside a graph only device-clock timers are possible
    Ev ev{take_event(), take_event(), bytes, flops, family};
    BOSP_CUDA(cudaEventRecord(ev.a, stream_));
    prof_events_.push_back(ev);
}

void Runtime::prof_end(const char* family) {
    (void)family;
    if (capture_prof_) return;
    BOSP_CUDA(cudaEventRecord(prof_events_.back().b, stream_));
}

unsigned long long* Runtime::timer_begin(const char* family, double bytes, double flops, double fixed_bytes,
                                         int64_t ncols) {
    if (!prof_on(family)) return nullptr;
    if (!timer_slots_) {
        BOSP_CUDA(cudaMalloc(&timer_slots_, sizeof(unsigned long long) * kSlotWords * kTimerSlots));
    }
    const int64_t slot = timer_next_++ % kTimerSlots;
    unsigned long long* p = timer_slots_ + kSlotWords * slot;
    if (timer_reserved_ > 0) --timer_reserved_;
    else BOSP_CUDA(cudaMemsetAsync(p, 0, kSlotWords * sizeof(unsigned long long), stream_));
    ProfPair pp{slot, bytes, flops, fixed_bytes, ncols, family};
    if (capture_prof_) capture_prof_->push_back(pp);
    else timer_pending_.push_back(pp);
    return p;
}

void Runtime::timer_reserve(int64_t count) {
    if (count <= 0) {
        timer_reserved_ = 0;  // end of a reserved section
        return;
    }
    if (prof_family_.empty()) return;
    if (!timer_slots_) BOSP_CUDA(cudaMalloc(&timer_slots_, sizeof(unsigned long long) * kSlotWords * kTimerSlots));
    count = std::min<int64_t>(count, kTimerSlots / 2);
    if (timer_next_ % kTimerSlots + count > kTimerSlots) timer_next_ += kTimerSlots - timer_next_ % kTimerSlots;
    BOSP_CUDA(cudaMemsetAsync(timer_slots_ + kSlotWords * (timer_next_ % kTimerSlots), 0,
                              sizeof(unsigned long long) * kSlotWords * count, stream_));
    timer_reserved_ = count;
}

void Runtime::read_timer_samples(const std::vector<ProfPair>& pairs) {
    if (pairs.empty()) return;
    // copy only the slot range these pairs use (they are allocated consecutively)
    int64_t lo = kTimerSlots, hi = -1;
    for (const ProfPair& p : pairs) {
        lo = std::min(lo, p.slot);
        hi = std::max(hi, p.slot);
    }
    const int64_t cnt = hi - lo + 1;
    if (static_cast<int64_t>(timer_host_.size()) < kSlotWords * cnt) timer_host_.resize(kSlotWords * cnt);
    BOSP_CUDA(cudaMemcpy(timer_host_.data(), timer_slots_ + kSlotWords * lo,
                         sizeof(unsigned long long) * kSlotWords * cnt, cudaMemcpyDeviceToHost));
    for (const ProfPair& p : pairs) {
        const unsigned long long* w = timer_host_.data() + kSlotWords * (p.slot - lo);
        const unsigned long long s = ~w[0], e = w[1];
        if (w[0] == 0 || e == 0 || e < s) continue;
        double frac = 1.0;
        if (p.ncols > 0) {  // the kernel reports how many columns it applied
            const int64_t act = static_cast<int64_t>(w[2]);
            if (act == 0) continue;  // nothing to do (converged columns): not a real apply
            frac = static_cast<double>(act) / static_cast<double>(p.ncols);
        }
        const double ms = (e - s) * 1e-6, by = p.fixed_bytes + (p.bytes - p.fixed_bytes) * frac;
        graph_samples_.launches += 1;
        graph_samples_.ms += ms;
        graph_samples_.bytes += by;
        graph_samples_.flops += p.flops * frac;
        ProfReport& f = by_family_[p.family ? p.family : "?"];
        f.launches += 1;
        f.ms += ms;
        f.bytes += by;
        f.flops += p.flops * frac;
    }
}

void Runtime::add_prof_samples(const std::vector<ProfPair>& pairs) {
    sync();
    read_timer_samples(pairs);
}

Runtime::ProfReport Runtime::prof_collect() {
    sync();
    read_timer_samples(timer_pending_);
    timer_pending_.clear();
    ProfReport r = graph_samples_;
    last_regions_ = ProfReport{r.region_calls, 0.0, r.region_bytes, r.region_flops};
    graph_samples_ = ProfReport{0, 0.0, 0.0, 0.0};
    for (auto& e : prof_events_) {
        float ms = 0.f;
        BOSP_CUDA(cudaEventElapsedTime(&ms, e.a, e.b));
        r.ms += ms;
        r.bytes += e.bytes;
        r.flops += e.flops;
        ++r.launches;
        ProfReport& f = by_family_[e.family ? e.family : "?"];
        f.launches += 1;
        f.ms += ms;
        f.bytes += e.bytes;
        f.flops += e.flops;
        event_pool_.push_back(e.a);
        event_pool_.push_back(e.b);
    }
    prof_events_.clear();
    last_by_family_ = std::move(by_family_);
    by_family_.clear();
    return r;
}

FamilyScope::FamilyScope(const char* fam) : prev(Runtime::get().family_override) {
    Runtime::get().family_override = fam;
}
FamilyScope::~FamilyScope() { Runtime::get().family_override = prev; }

LaunchScope::LaunchScope(const char* fam, double bytes, double flops, bool events) : family(fam) {
    Runtime& rt = Runtime::get();
    if (rt.family_override) family = fam = rt.family_override;
    rt.count_launch(fam);
    timed = events && rt.prof_on(fam);
    if (timed) rt.prof_begin(fam, bytes, flops);
}

LaunchScope::~LaunchScope() {
    if (timed) Runtime::get().prof_end(family);
}

DBlock::DBlock(int64_t rows, int64_t cols) : rows_(rows), cols_(cols), cap_(cols), ld_(ld_for(rows)) {
    if (rows > 0 && cols > 0)
        p_ = static_cast<double*>(Runtime::get().alloc(sizeof(double) * ld_ * cols));
}

DBlock::~DBlock() {
    if (p_) Runtime::get().free(p_);
}

DBlock::DBlock(DBlock&& o) noexcept
    : p_(o.p_), rows_(o.rows_), cols_(o.cols_), cap_(o.cap_), ld_(o.ld_) {
    o.p_ = nullptr;
    o.rows_ = o.cols_ = o.cap_ = 0;
}

DBlock& DBlock::operator=(DBlock&& o) noexcept {
    if (this != &o) {
        if (p_) Runtime::get().free(p_);
        p_ = o.p_;
        rows_ = o.rows_;
        cols_ = o.cols_;
        cap_ = o.cap_;
        ld_ = o.ld_;
        o.p_ = nullptr;
        o.rows_ = o.cols_ = o.cap_ = 0;
    }
    return *this;
}

void DBlock::set_cols(int64_t c) {
    if (c > cap_) throw ContractViolation("DBlock::set_cols: exceeds capacity");
    cols_ = c;
}

void DBlock::zero() {
    if (p_) BOSP_CUDA(cudaMemsetAsync(p_, 0, sizeof(double) * ld_ * cap_, Runtime::get().stream()));
}

namespace {

// Large pageable transfers go through the pinned ring in chunks: the DMA of chunk i+1 overlaps
// the (OpenMP-parallel) host copy of chunk i, instead of the driver's serial pageable path.
constexpr size_t kStagedMin = size_t(4) << 20;  // bytes; smaller copies go direct

struct Chunk {
    int64_t c0, nc, r0, nr;  // columns [c0, c0+nc), rows [r0, r0+nr)
};

std::vector<Chunk> chunks_of(int64_t rows, int64_t cols) {
    std::vector<Chunk> out;
    const int64_t cap = static_cast<int64_t>(Runtime::kStageDoubles);
    if (rows >= cap / 2) {  // tall: split every column into row pieces
        for (int64_t c = 0; c < cols; ++c)
            for (int64_t r = 0; r < rows; r += cap) out.push_back({c, 1, r, std::min(cap, rows - r)});
    } else {
        const int64_t per = std::max<int64_t>(1, cap / rows);
        for (int64_t c = 0; c < cols; c += per) out.push_back({c, std::min(per, cols - c), 0, rows});
    }
    return out;
}

void host_scatter(const double* stage, const Chunk& ch, double* host, int64_t ld_host, bool to_host_dir) {
    // stage holds the chunk as nr x nc, ld = nr
#pragma omp parallel for schedule(static) if (ch.nr * ch.nc > (1 << 16))
    for (int64_t q = 0; q < ch.nc * 8; ++q) {
        const int64_t c = q / 8, part = q % 8;
        const int64_t lo = ch.nr * part / 8, hi = ch.nr * (part + 1) / 8;
        if (hi <= lo) continue;
        double* h = host + (ch.c0 + c) * ld_host + ch.r0 + lo;
        double* st = const_cast<double*>(stage) + c * ch.nr + lo;
        if (to_host_dir) std::memcpy(h, st, sizeof(double) * (hi - lo));
        else std::memcpy(st, h, sizeof(double) * (hi - lo));
    }
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

void to_device(const double* host, int64_t rows, int64_t cols, int64_t ld_host, const DMat& dst) {
    if (rows == 0 || cols == 0) return;
    Runtime& rt = Runtime::get();
    if (static_cast<size_t>(rows * cols) * sizeof(double) < kStagedMin || is_pinned(host)) {
        BOSP_CUDA(cudaMemcpy2DAsync(dst.p, dst.ld * sizeof(double), host, ld_host * sizeof(double),
                                    rows * sizeof(double), cols, cudaMemcpyHostToDevice, rt.stream()));
        return;
    }
    const std::vector<Chunk> ch = chunks_of(rows, cols);
    for (size_t i = 0; i < ch.size(); ++i) {
        const int b = static_cast<int>(i & 1);
        double* st = rt.stage(b);
        if (i >= 2) BOSP_CUDA(cudaEventSynchronize(rt.stage_event(b)));  // buffer's previous DMA done
        host_scatter(st, ch[i], const_cast<double*>(host), ld_host, false);
        BOSP_CUDA(cudaMemcpy2DAsync(dst.p + ch[i].c0 * dst.ld + ch[i].r0, dst.ld * sizeof(double), st,
                                    ch[i].nr * sizeof(double), ch[i].nr * sizeof(double), ch[i].nc,
                                    cudaMemcpyHostToDevice, rt.stream()));
        BOSP_CUDA(cudaEventRecord(rt.stage_event(b), rt.stream()));
    }
    // the ring is reused by the next transfer only after these events
    BOSP_CUDA(cudaEventSynchronize(rt.stage_event(static_cast<int>((ch.size() - 1) & 1))));
}

void h2d_bytes(void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return;
    if (bytes >= kStagedMin && bytes % sizeof(double) == 0 && !is_pinned(src)) {
        const int64_t nd = static_cast<int64_t>(bytes / sizeof(double));
        to_device(static_cast<const double*>(src), nd, 1, nd, DMat{static_cast<double*>(dst), nd, nd, 1});
        return;
    }
    BOSP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, Runtime::get().stream()));
}

void to_host(const DMat& src, double* host, int64_t ld_host) {
    if (src.rows == 0 || src.cols == 0) return;
    Runtime& rt = Runtime::get();
    if (static_cast<size_t>(src.rows * src.cols) * sizeof(double) < kStagedMin || is_pinned(host)) {
        BOSP_CUDA(cudaMemcpy2DAsync(host, ld_host * sizeof(double), src.p, src.ld * sizeof(double),
                                    src.rows * sizeof(double), src.cols, cudaMemcpyDeviceToHost,
                                    rt.stream()));
        rt.sync();
        return;
    }
    const std::vector<Chunk> ch = chunks_of(src.rows, src.cols);
    auto issue = [&](size_t i) {
        const int b = static_cast<int>(i & 1);
        BOSP_CUDA(cudaMemcpy2DAsync(rt.stage(b), ch[i].nr * sizeof(double), src.p + ch[i].c0 * src.ld + ch[i].r0,
                                    src.ld * sizeof(double), ch[i].nr * sizeof(double), ch[i].nc,
                                    cudaMemcpyDeviceToHost, rt.stream()));
        BOSP_CUDA(cudaEventRecord(rt.stage_event(b), rt.stream()));
    };
    issue(0);
    for (size_t i = 0; i < ch.size(); ++i) {
        const int b = static_cast<int>(i & 1);
        BOSP_CUDA(cudaEventSynchronize(rt.stage_event(b)));
        if (i + 1 < ch.size()) issue(i + 1);  // DMA of the next chunk overlaps this host copy
        host_scatter(rt.stage(b), ch[i], host, ld_host, true);
    }
}

void copy_block(const DMat& src, const DMat& dst) {
    if (src.rows == 0 || src.cols == 0) return;
    if (src.p == dst.p && src.ld == dst.ld) return;
    BOSP_CUDA(cudaMemcpy2DAsync(dst.p, dst.ld * sizeof(double), src.p, src.ld * sizeof(double),
                                src.rows * sizeof(double), src.cols, cudaMemcpyDeviceToDevice,
                                Runtime::get().stream()));
}

}  // namespace b200
}  // namespace bosp
