// stabkit/nccl_exchange.hpp -- the ShardExchange of stabkit/sharded.hpp over NCCL (north_star: "each measurement is a small NCCL
// allreduce for the pivot index plus a broadcast of the pivot row over NVLink").  One process per GPU.
//   allreduce_min  ncclAllReduce(ncclMin, int32)   pivot candidates of a window, 4 bytes per pending measurement
//   broadcast      ncclBroadcast(uint64)           the pivot row from the rank that owns it (16*Wp + 16 bytes)
//   allgather      ncclAllGather(uint64)           the shards' partial products of a run of deterministic measurements
// All three are enqueued on the library context's stream (sk_ctx_stream), so they are ordered with the sk_shard_* kernels without
// any host synchronisation; only the candidates come back to the host (the driver branches on them).
// Header only; the application links NCCL and the CUDA runtime itself (libstabkit_b200.so does not depend on NCCL).
// An NCCL failure is reported as stabkit::Error carrying the SK_ENCCL status text.
// The reference has no counterpart: it is a single-process CPU code (proj/CMakeLists.txt:11 links Threads only).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdio>
#include <string>
#include <vector>

#include "stabkit/sharded.hpp"

namespace stabkit {

class NcclExchange : public ShardExchange {
  public:
    // Joins the communicator described by `id` (made by rank 0 with NcclExchange::make_id() and handed to the others by the
    // launcher: file, MPI, torch.distributed store ...).  The device is the one of Device::instance() (STABKIT_DEVICE).
    NcclExchange(const ncclUniqueId& id, int rank, int world) : rank_(rank), world_(world) {
        Device& d = Device::instance();
        stream_ = static_cast<cudaStream_t>(sk_ctx_stream(d.ctx()));
        check(ncclCommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
        if (cudaMalloc(&d_cand_, cap_ * sizeof(int32_t)) != cudaSuccess) throw Error("NcclExchange: cudaMalloc failed");
    }
    ~NcclExchange() override {
        if (d_cand_) cudaFree(d_cand_);
        if (comm_) ncclCommDestroy(comm_);
    }
    NcclExchange(const NcclExchange&) = delete;
    NcclExchange& operator=(const NcclExchange&) = delete;
    static ncclUniqueId make_id() { ncclUniqueId id; check(ncclGetUniqueId(&id), "ncclGetUniqueId"); return id; }

    int rank() const override { return rank_; }
    int world() const override { return world_; }
    void allreduce_min(std::vector<int32_t>& cand) override {
        if (cand.empty()) return;
        if (cand.size() > cap_) {
            cudaFree(d_cand_); d_cand_ = nullptr; cap_ = 2 * cand.size();
            if (cudaMalloc(&d_cand_, cap_ * sizeof(int32_t)) != cudaSuccess) throw Error("NcclExchange: cudaMalloc failed");
        }
        cudaMemcpyAsync(d_cand_, cand.data(), cand.size() * 4, cudaMemcpyHostToDevice, stream_);
        check(ncclAllReduce(d_cand_, d_cand_, cand.size(), ncclInt32, ncclMin, comm_, stream_), "ncclAllReduce(min)");
        cudaMemcpyAsync(cand.data(), d_cand_, cand.size() * 4, cudaMemcpyDeviceToHost, stream_);
        if (cudaStreamSynchronize(stream_) != cudaSuccess) throw Error("NcclExchange: stream error after ncclAllReduce");
        ++calls_[0]; bytes_ += cand.size() * 4;
    }
    void allgather(sk_ctx* /*ctx*/, const uint64_t* d_in, uint64_t* d_out, size_t words_per_rank) override {
        check(ncclAllGather(d_in, d_out, words_per_rank, ncclUint64, comm_, stream_), "ncclAllGather");
        ++calls_[1]; bytes_ += words_per_rank * 8 * size_t(world_);
    }
    void broadcast(sk_ctx* /*ctx*/, uint64_t* d_row, size_t words, int root_rank) override {
        check(ncclBroadcast(d_row, d_row, words, ncclUint64, root_rank, comm_, stream_), "ncclBroadcast");
        ++calls_[2]; bytes_ += words * 8;
    }
    // collectives issued so far: allreduce-min, allgather, broadcast; and the payload bytes
    const size_t* calls() const { return calls_; }
    size_t bytes() const { return bytes_; }

  private:
    static void check(ncclResult_t r, const char* what) {
        if (r != ncclSuccess) throw_status(SK_ENCCL, std::string(what) + ": " + ncclGetErrorString(r));
    }
    int rank_, world_;
    ncclComm_t comm_ = nullptr;
    cudaStream_t stream_ = nullptr;
    int32_t* d_cand_ = nullptr; size_t cap_ = 8192;
    size_t calls_[3] = {0, 0, 0}, bytes_ = 0;
};

}  // namespace stabkit
