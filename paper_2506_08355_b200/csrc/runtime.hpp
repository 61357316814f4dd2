// Device runtime for the B200 BOSP core: one stream per process/device, a stream-ordered memory
// pool (cudaMallocAsync, release threshold = unlimited so HBM stays cached across solves), a
// grow-only scratch arena for split-K partials and reduction tickets, pinned staging for the
// small host<->device matrices, launch counting and per-kernel-family CUDA-event timing.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"

namespace bosp {
inline namespace b200 {

// Row-partition communicator: every n-length block of the solve is split by rows across ranks;
// Grams, dots and residual sums are partial per rank and summed by allreduce_sum (which must give
// bit-identical results on every rank so all ranks take the same host decisions).  Halo rows of
// the sparse operators move with sendrecv, dense operators allgather x.
struct HaloMsg {
    int peer;
    double* ptr;    // device buffer (read for sends, written for receives)
    int64_t count;  // doubles
};

class Comm {
public:
    virtual ~Comm();
    virtual int rank() const = 0;
    virtual int size() const = 0;
    // in place over `count` doubles in device memory, ordered on `stream`; identical result on
    // every rank
    virtual void allreduce_sum(double* dev, int64_t count, cudaStream_t stream) = 0;
    // point-to-point halo exchange: every send must be matched by the peer's receive
    virtual void exchange(const std::vector<HaloMsg>& sends, const std::vector<HaloMsg>& recvs,
                          cudaStream_t stream) = 0;
    // every rank contributes `count` doubles; recv holds size()*count, rank-major
    virtual void allgather(const double* sdev, int64_t count, double* rdev, cudaStream_t stream) = 0;
    // Every call only enqueues work on `stream` (no host synchronisation), so it can be recorded
    // into a CUDA graph: NCCL (collectives and grouped send/recv are capturable), not ThreadComm
    // (its ranks meet at host barriers).
    virtual bool stream_capturable() const { return false; }
};

class Runtime {
public:
    // One runtime per host thread: its own stream, pool, scratch and communicator, so that
    // several ranks (one thread per GPU, or several virtual ranks on one GPU) never share state.
    static Runtime& get();
    void set_comm(std::shared_ptr<Comm> c) { comm_ = std::move(c); }
    Comm* comm() const { return comm_.get(); }
    int nranks() const { return comm_ ? comm_->size() : 1; }
    int rank() const { return comm_ ? comm_->rank() : 0; }
    // Global row window of this rank (row-partitioned solve): rows [row0, row0 + local) of
    // n_global.  Defaults describe an unpartitioned solve (set by solve()).
    void set_rows(int64_t n_global, int64_t row0) { n_global_ = n_global; row0_ = row0; }
    int64_t n_global() const { return n_global_; }
    int64_t row0() const { return row0_; }
    // Sum a per-rank partial result across ranks (no-op on one rank).
    void allreduce(double* dev, int64_t count) {
        if (comm_ && comm_->size() > 1) comm_->allreduce_sum(dev, count, stream_);
    }
    // Per-device one-time kernel attribute setup (bit per device id).
    // Per-device one-time setup (kernel attributes), thread-safe: ranks sharing a device (one
    // thread each) wait until the first caller's setup is done -- publishing the bit before the
    // attribute call let a second rank launch without it (cudaErrorInvalidValue).
    template <class F>
    void once_per_device(unsigned& mask, F&& setup) {
        const unsigned bit = 1u << (device_ & 31);
        if (__atomic_load_n(&mask, __ATOMIC_ACQUIRE) & bit) return;
        std::lock_guard<std::mutex> lk(setup_mutex());
        if (mask & bit) return;
        setup();
        __atomic_fetch_or(&mask, bit, __ATOMIC_RELEASE);
    }
    static std::mutex& setup_mutex();

    cudaStream_t stream() const { return stream_; }
    int device() const { return device_; }
    int sm_count() const { return sm_count_; }

    void* alloc(size_t bytes);
    void free(void* p);
    void sync();
    // BOSP_SYNC_STATS=1: host synchronisations and the host time spent waiting in them
    int64_t sync_count_ = 0;
    int64_t graph_builds_ = 0;
    double graph_build_s_ = 0.0;
    double sync_wait_s_ = 0.0;

    // Scratch for split-K partials (fp64) -- valid until the next call; stream-ordered reuse is
    // safe because every consumer runs on stream().
    double* scratch(size_t doubles);
    // Zero-initialised uint32 tickets; each kernel that takes tickets leaves them at zero.
    unsigned int* tickets(size_t count);
    // Bumped whenever scratch() or tickets() reallocates: a CUDA graph that captured the old
    // pointers must not be replayed after that (dev_cg keys its graph cache on it).
    uint64_t scratch_generation() const { return scratch_gen_; }
    // Pinned host staging (grow-only).
    double* pinned(size_t doubles);
    // Double-buffered pinned ring for large pageable host<->device copies (to_host/to_device):
    // buffer i of kStageDoubles doubles and its completion event.
    static constexpr size_t kStageDoubles = size_t(1) << 20;  // 8 MB
    double* stage(int i);
    cudaEvent_t stage_event(int i);

    // Kernel accounting (gpu_launches) and optional CUDA-event timing of one kernel family.
    void count_launch(const char* family);
    // While set, every launch is attributed to this family (an operator's apply: "dense_apply")
    const char* family_override = nullptr;
    int64_t launches() const { return launches_; }
    void reset_launches() { launches_ = 0; family_launches_.clear(); }
    const std::map<std::string, int64_t>& family_launches() const { return family_launches_; }

    // Launches issued while a stream capture is recorded are tallied into `sink` (per family)
    // instead of the live counters; graph replays add them back per execution.
    void set_capture_sink(std::map<std::string, int64_t>* sink) { capture_sink_ = sink; }
    void add_launches(const std::map<std::string, int64_t>& fam, int64_t times);

    void prof_enable(const std::string& family);  // "" disables
    bool prof_on(const char* family) const;
    bool prof_active() const { return !prof_family_.empty(); }
    void prof_begin(const char* family, double algo_bytes, double algo_flops);
    void prof_end(const char* family);
    // launches/ms/bytes/flops: the timed kernels (each with its own operand bytes);
    // region_calls/region_bytes: composite operations (ProfRegion) and their algorithmic bytes.
    struct ProfReport {
        int64_t launches; double ms; double bytes; double flops;
        int64_t region_calls = 0; double region_bytes = 0.0; double region_flops = 0.0;
    };
    ProfReport prof_collect();  // synchronises, sums elapsed times, resets
    // prof_enable("*") times every launch; the last prof_collect() split by kernel family
    const std::map<std::string, ProfReport>& prof_by_family() const { return last_by_family_; }
    // Composite-operation profiling: while a region named like the profiled family is open,
    // every launch inside it is timed (whatever its own family); at close the region credits
    // its algorithmic bytes once.  Nested regions of the same name count once (outermost).
    bool region_open(const char* name);
    void region_close(double algo_bytes, double algo_flops = 0.0);
    // the last prof_collect()'s composite-operation totals (calls, bytes, flops)
    ProfReport last_regions_{0, 0.0, 0.0, 0.0};
    // Device-clock timing for kernels that may run inside CUDA graphs (event nodes are not
    // allowed in conditional bodies): the kernel writes (max of ~start, max of end) %globaltimer
    // into a 2-word slot that a memset resets before each launch.  A launch recorded into a
    // graph keeps its slot; after each replay the slot holds that launch's last execution.
    // Slot words: [~earliest start, latest end, columns the launch actually applied (0 = none
    // reported)].  bytes/flops are the launch's algorithmic totals for all `ncols` columns; a
    // launch that reports fewer active columns is credited proportionally (fixed part kept).
    struct ProfPair { int64_t slot; double bytes, flops, fixed_bytes; int64_t ncols; const char* family; };
    static constexpr int kSlotWords = 4;
    unsigned long long* timer_begin(const char* family, double bytes, double flops, double fixed_bytes = 0.0,
                                    int64_t ncols = 0);
    // Zero `count` consecutive slots with one memset; the next `count` timer_begin calls take
    // them without their own memset (one memset node per recorded graph instead of one per
    // timed launch).  No-op unless a family is being profiled.
    void timer_reserve(int64_t count);
    void set_capture_prof(std::vector<ProfPair>* sink) { capture_prof_ = sink; }
    void add_prof_samples(const std::vector<ProfPair>& pairs);  // after the replay finished
    const std::string& prof_family() const { return prof_family_; }

private:
    Runtime();
    ~Runtime();
    int device_ = 0;
    int sm_count_ = 148;
    cudaStream_t stream_ = nullptr;
    std::shared_ptr<Comm> comm_;
    int64_t n_global_ = 0, row0_ = 0;
    double* scratch_ = nullptr;
    size_t scratch_cap_ = 0;
    uint64_t scratch_gen_ = 0;
    unsigned int* tickets_ = nullptr;
    size_t tickets_cap_ = 0;
    double* pinned_ = nullptr;
    size_t pinned_cap_ = 0;
    double* stage_[2] = {nullptr, nullptr};
    cudaEvent_t stage_ev_[2] = {nullptr, nullptr};
    int64_t launches_ = 0;
    std::map<std::string, int64_t> family_launches_;
    std::map<std::string, int64_t>* capture_sink_ = nullptr;
    std::string prof_family_;
    struct Ev { cudaEvent_t a, b; double bytes, flops; const char* family; };
    // per-family split of the last prof_collect() (family names are string literals)
    std::map<std::string, ProfReport> by_family_, last_by_family_;
    std::vector<Ev> prof_events_;
    std::vector<ProfPair>* capture_prof_ = nullptr;
    std::vector<ProfPair> timer_pending_;
    unsigned long long* timer_slots_ = nullptr;
    std::vector<unsigned long long> timer_host_;
    int64_t timer_reserved_ = 0;
    int64_t timer_next_ = 0;
    static constexpr int64_t kTimerSlots = 1 << 15;
    ProfReport graph_samples_{0, 0.0, 0.0, 0.0};
    int region_depth_ = 0;
    void read_timer_samples(const std::vector<ProfPair>& pairs);
    std::vector<cudaEvent_t> event_pool_;
    cudaEvent_t take_event();
};

// RAII: times one launch of `family` when profiling is on for it; always counts the launch.
// RAII: attribute the launches of a scope (e.g. one operator apply) to one family.
struct FamilyScope {
    const char* prev;
    explicit FamilyScope(const char* fam);
    ~FamilyScope();
};

struct LaunchScope {
    const char* family;
    bool timed;
    // events = false: the kernel times itself with a device-clock slot (Runtime::timer_begin)
    LaunchScope(const char* fam, double bytes = 0.0, double flops = 0.0, bool events = true);
    ~LaunchScope();
};

// RAII: a composite operation (e.g. one MGS-Biorth call) profiled as a unit when its name is the
// profiled family; `algo_bytes` is the operation's algorithmic traffic.
struct ProfRegion {
    bool open;
    double algo_bytes, algo_flops;
    ProfRegion(const char* name, double bytes, double flops = 0.0)
        : open(Runtime::get().region_open(name)), algo_bytes(bytes), algo_flops(flops) {}
    ~ProfRegion() {
        if (open) Runtime::get().region_close(algo_bytes, algo_flops);
    }
};

// Owning device block: rows x capacity columns, column stride ld = rows rounded up to 32
// doubles (256 B) so every column starts on a 256-byte boundary.
class DBlock {
public:
    DBlock() = default;
    DBlock(int64_t rows, int64_t cols);
    ~DBlock();
    DBlock(const DBlock&) = delete;
    DBlock& operator=(const DBlock&) = delete;
    DBlock(DBlock&& o) noexcept;
    DBlock& operator=(DBlock&& o) noexcept;

    DMat view() const { return DMat{p_, ld_, rows_, cols_}; }
    DMat cols(int64_t c0, int64_t nc) const { return view().cols_range(c0, nc); }
    int64_t rows() const { return rows_; }
    int64_t ncols() const { return cols_; }
    int64_t ld() const { return ld_; }
    double* data() const { return p_; }
    // Reshape the logical width within capacity (no data movement).
    void set_cols(int64_t c);
    int64_t capacity() const { return cap_; }
    void zero();

    static int64_t ld_for(int64_t rows) { return ((rows + 31) / 32) * 32; }

private:
    double* p_ = nullptr;
    int64_t rows_ = 0, cols_ = 0, cap_ = 0, ld_ = 0;
};

// Device copies of small host matrices (column-major) and back.
void to_device(const double* host, int64_t rows, int64_t cols, int64_t ld_host, const DMat& dst);
void to_host(const DMat& src, double* host, int64_t ld_host);
// Flat host -> device copy (stream-ordered; large 8-byte-multiple copies use the pinned ring).
void h2d_bytes(void* dst, const void* src, size_t bytes);
// D2D copy of a column range (handles differing ld).
void copy_block(const DMat& src, const DMat& dst);

}  // namespace b200
}  // namespace bosp
