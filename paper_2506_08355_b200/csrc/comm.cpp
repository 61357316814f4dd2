// ThreadComm (ranks = threads of one process) and NcclComm (ranks = processes, dlopen'ed NCCL).
#include "comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

namespace bosp {
inline namespace b200 {

// ---------------------------------------------------------------------------------------------
ThreadGroup::ThreadGroup(int size) : ptr(size, nullptr), device(size, -1), sends(size), size_(size) {
    require(size >= 1 && size <= kMaxRanks, "ThreadGroup: 1..16 ranks");
}

void ThreadGroup::barrier() {
    std::unique_lock<std::mutex> lk(mu_);
    if (aborted_) throw Error("ThreadGroup: another rank failed");
    const int64_t gen = generation_;
    if (++arrived_ == size_) {
        arrived_ = 0;
        ++generation_;
        cv_.notify_all();
        return;
    }
    cv_.wait(lk, [&] { return generation_ != gen || aborted_; });
    if (generation_ == gen) throw Error("ThreadGroup: another rank failed");
}

void ThreadGroup::abort() {
    std::lock_guard<std::mutex> lk(mu_);
    aborted_ = true;
    cv_.notify_all();
}

ThreadComm::ThreadComm(std::shared_ptr<ThreadGroup> g, int rank, int device)
    : group_(std::move(g)), rank_(rank), device_(device) {
    group_->device[rank_] = device_;
    group_->barrier();  // every rank registered its device
    for (int r = 0; r < group_->size(); ++r) {
        const int d = group_->device[r];
        if (d == device_) continue;
        const cudaError_t e = cudaDeviceEnablePeerAccess(d, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            throw CudaError(std::string("ThreadComm: peer access ") + cudaGetErrorString(e));
        cudaGetLastError();
    }
    group_->barrier();
}

void ThreadComm::allreduce_sum(double* dev, int64_t count, cudaStream_t stream) {
    if (count <= 0) return;
    BOSP_CUDA(cudaStreamSynchronize(stream));
    group_->ptr[rank_] = dev;
    group_->barrier();
    if (count > tmp_cap_) {
        if (tmp_) cudaFree(tmp_);
        tmp_cap_ = count;
        BOSP_CUDA(cudaMalloc(&tmp_, sizeof(double) * tmp_cap_));
    }
    RankPtrs rp{};
    rp.n = group_->size();
    for (int r = 0; r < rp.n; ++r) rp.p[r] = group_->ptr[r];
    sum_ranks(rp, tmp_, count, stream);
    BOSP_CUDA(cudaStreamSynchronize(stream));
    group_->barrier();  // every rank finished reading every buffer
    BOSP_CUDA(cudaMemcpyAsync(dev, tmp_, sizeof(double) * count, cudaMemcpyDeviceToDevice, stream));
}

void ThreadComm::exchange(const std::vector<HaloMsg>& sends, const std::vector<HaloMsg>& recvs,
                          cudaStream_t stream) {
    BOSP_CUDA(cudaStreamSynchronize(stream));
    group_->sends[rank_] = sends;
    group_->barrier();
    for (const HaloMsg& r : recvs) {
        const HaloMsg* s = nullptr;
        for (const HaloMsg& m : group_->sends[r.peer])
            if (m.peer == rank_) s = &m;
        require(s != nullptr && s->count == r.count, "ThreadComm::exchange: unmatched halo message");
        if (r.count > 0)
            BOSP_CUDA(cudaMemcpyPeerAsync(r.ptr, device_, s->ptr, group_->device[r.peer],
                                          sizeof(double) * r.count, stream));
    }
    BOSP_CUDA(cudaStreamSynchronize(stream));
    group_->barrier();
}

void ThreadComm::allgather(const double* sdev, int64_t count, double* rdev, cudaStream_t stream) {
    BOSP_CUDA(cudaStreamSynchronize(stream));
    group_->ptr[rank_] = sdev;
    group_->barrier();
    for (int r = 0; r < group_->size(); ++r)
        if (count > 0)
            BOSP_CUDA(cudaMemcpyPeerAsync(rdev + r * count, device_, group_->ptr[r], group_->device[r],
                                          sizeof(double) * count, stream));
    BOSP_CUDA(cudaStreamSynchronize(stream));
    group_->barrier();
}

// ---------------------------------------------------------------------------------------------
namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        // prefer an already-loaded libnccl (e.g. torch's), else the system one
        // Reuse an NCCL the process already loaded (e.g. torch's bundled one: loading the older
        // system libnccl.so.2 first would make a later `import torch` resolve its NCCL symbols
        // against it and fail); otherwise load it privately (RTLD_LOCAL).
        a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!a.h) a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!a.h) throw CudaError("NcclComm: cannot dlopen libnccl.so.2");
        auto sym = [&](const char* n) {
            void* s = dlsym(a.h, n);
            if (!s) throw CudaError(std::string("NcclComm: missing symbol ") + n);
            return s;
        };
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
        a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
        a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
        a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
        a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
        a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
        return a;
    }();
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaError(std::string("NCCL ") + what + ": " + nccl().GetErrorString(r));
}

}  // namespace

void NcclComm::unique_id(unsigned char out[kIdBytes]) {
    ncclUniqueId id;
    nccl_check(nccl().GetUniqueId(&id), "GetUniqueId");
    static_assert(sizeof(ncclUniqueId) == kIdBytes, "ncclUniqueId size");
    std::memcpy(out, &id, kIdBytes);
}

NcclComm::NcclComm(const unsigned char id[kIdBytes], int nranks, int rank) : rank_(rank), size_(nranks) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, kIdBytes);
    ncclComm_t c = nullptr;
    nccl_check(nccl().CommInitRank(&c, nranks, uid, rank), "CommInitRank");
    comm_ = c;
}

NcclComm::~NcclComm() {
    if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
}

void NcclComm::allreduce_sum(double* dev, int64_t count, cudaStream_t stream) {
    if (count <= 0) return;
    nccl_check(nccl().AllReduce(dev, dev, static_cast<size_t>(count), ncclFloat64, ncclSum,
                                static_cast<ncclComm_t>(comm_), stream), "AllReduce");
}

void NcclComm::exchange(const std::vector<HaloMsg>& sends, const std::vector<HaloMsg>& recvs,
                        cudaStream_t stream) {
    nccl_check(nccl().GroupStart(), "GroupStart");
    for (const HaloMsg& s : sends)
        if (s.count > 0)
            nccl_check(nccl().Send(s.ptr, static_cast<size_t>(s.count), ncclFloat64, s.peer,
                                   static_cast<ncclComm_t>(comm_), stream), "Send");
    for (const HaloMsg& r : recvs)
        if (r.count > 0)
            nccl_check(nccl().Recv(r.ptr, static_cast<size_t>(r.count), ncclFloat64, r.peer,
                                   static_cast<ncclComm_t>(comm_), stream), "Recv");
    nccl_check(nccl().GroupEnd(), "GroupEnd");
}

void NcclComm::allgather(const double* sdev, int64_t count, double* rdev, cudaStream_t stream) {
    nccl_check(nccl().AllGather(sdev, rdev, static_cast<size_t>(count), ncclFloat64,
                                static_cast<ncclComm_t>(comm_), stream), "AllGather");
}

}  // namespace b200
}  // namespace bosp
