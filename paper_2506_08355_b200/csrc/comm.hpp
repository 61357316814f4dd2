// Communicators for the row-partitioned solve.
//
//  * ThreadComm -- ranks are host threads of one process (one thread per GPU, or several
//    virtual ranks sharing one GPU).  Buffers are exchanged through device pointers published
//    in a shared table: same-device reads, or peer reads over NVLink (cudaDeviceEnablePeerAccess).
//    allreduce sums the ranks' buffers in rank order on every rank -> bit-identical results.
//  * NcclComm   -- one process per GPU (torchrun): ncclAllReduce / grouped ncclSend+ncclRecv /
//    ncclAllGather on the solver stream.  libnccl is dlopen'ed on first use so the library
//    loads without it.
#pragma once

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

#include "runtime.hpp"

namespace bosp {
inline namespace b200 {

class ThreadGroup {
public:
    explicit ThreadGroup(int size);
    int size() const { return size_; }
    void barrier();  // throws if another rank aborted (so a failing rank cannot hang the rest)
    void abort();
    // published state (indexed by rank)
    std::vector<const double*> ptr;
    std::vector<int> device;
    std::vector<std::vector<HaloMsg>> sends;

private:
    int size_;
    std::mutex mu_;
    std::condition_variable cv_;
    int arrived_ = 0;
    int64_t generation_ = 0;
    bool aborted_ = false;
};

class ThreadComm final : public Comm {
public:
    ThreadComm(std::shared_ptr<ThreadGroup> g, int rank, int device);
    int rank() const override { return rank_; }
    int size() const override { return group_->size(); }
    void allreduce_sum(double* dev, int64_t count, cudaStream_t stream) override;
    void exchange(const std::vector<HaloMsg>& sends, const std::vector<HaloMsg>& recvs,
                  cudaStream_t stream) override;
    void allgather(const double* sdev, int64_t count, double* rdev, cudaStream_t stream) override;

private:
    std::shared_ptr<ThreadGroup> group_;
    int rank_, device_;
    double* tmp_ = nullptr;
    int64_t tmp_cap_ = 0;
};

class NcclComm final : public Comm {
public:
    static constexpr int kIdBytes = 128;
    static void unique_id(unsigned char out[kIdBytes]);
    NcclComm(const unsigned char id[kIdBytes], int nranks, int rank);
    ~NcclComm() override;
    int rank() const override { return rank_; }
    int size() const override { return size_; }
    void allreduce_sum(double* dev, int64_t count, cudaStream_t stream) override;
    void exchange(const std::vector<HaloMsg>& sends, const std::vector<HaloMsg>& recvs,
                  cudaStream_t stream) override;
    void allgather(const double* sdev, int64_t count, double* rdev, cudaStream_t stream) override;
    bool stream_capturable() const override { return true; }

private:
    void* comm_ = nullptr;
    int rank_, size_;
};

// device helpers (comm_kernels.cu)
constexpr int kMaxRanks = 16;
struct RankPtrs {
    const double* p[kMaxRanks];
    int n;
};
void sum_ranks(const RankPtrs& src, double* dst, int64_t count, cudaStream_t stream);
// out[i + j*ldo] = x[idx[i] + j*ldx] for i < cnt, j < m  (halo packing)
void gather_rows(const double* x, int64_t ldx, const int32_t* idx, int64_t cnt, int64_t m,
                 double* out, int64_t ldo, cudaStream_t stream);

}  // namespace b200
}  // namespace bosp
