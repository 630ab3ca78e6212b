// comm.cpp -- NCCL and loopback implementations of ciq::Comm (see comm.h).
#include "comm.h"

#include <string>

#include "nccl_dl.h"

namespace ciq {

namespace {

class NcclComm final : public Comm {
 public:
  NcclComm(int rank, int world, void* comm) : rank_(rank), world_(world), comm_(comm) {}
  ~NcclComm() override { nccl_comm_destroy(comm_); }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  bool allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    // ncclInt8 = 0: byte-exact transport of fp32 rows / fp64 partials
    if (!nccl_allgather(send, recv, bytes, /*ncclInt8*/ 0, comm_, s)) {
      err_ = nccl_error();
      return false;
    }
    return true;
  }
  const char* error() const override { return err_.c_str(); }
  bool capturable() const override { return true; }

 private:
  int rank_, world_;
  void* comm_;
  std::string err_;
};

class LoopbackComm final : public Comm {
 public:
  LoopbackComm(LoopbackGroup* g, int rank) : g_(g), rank_(rank) {
    cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&done_, cudaEventDisableTiming);
  }
  ~LoopbackComm() override {
    cudaEventDestroy(ready_);
    cudaEventDestroy(done_);
  }
  int rank() const override { return rank_; }
  int world() const override { return g_->world(); }
  bool allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    const int w = g_->world();
    // 1. publish our send buffer once its producer work is enqueued
    if (cudaEventRecord(ready_, s) != cudaSuccess) return fail("event record");
    g_->slots[rank_].send = send;
    g_->slots[rank_].ready = ready_;
    g_->slots[rank_].done = done_;
    g_->barrier();
    // 2. pull every rank's block (device-to-device on our stream, after its producer)
    for (int p = 0; p < w; ++p) {
      const auto& sl = g_->slots[p];
      char* dst = static_cast<char*>(recv) + (size_t)p * bytes;
      if (sl.send == dst) continue;
      if (p != rank_ && cudaStreamWaitEvent(s, sl.ready, 0) != cudaSuccess) return fail("wait ready");
      if (cudaMemcpyAsync(dst, sl.send, bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess) return fail("copy");
    }
    if (cudaEventRecord(done_, s) != cudaSuccess) return fail("event record");
    g_->barrier();
    // 3. nobody may overwrite its send buffer before every peer has copied from it
    for (int p = 0; p < w; ++p)
      if (p != rank_ && cudaStreamWaitEvent(s, g_->slots[p].done, 0) != cudaSuccess) return fail("wait done");
    g_->barrier();
    return true;
  }
  const char* error() const override { return err_.c_str(); }
  bool capturable() const override { return false; }

 private:
  bool fail(const char* what) {
    err_ = std::string("loopback allgather: ") + what + ": " + cudaGetErrorString(cudaGetLastError());
    return false;
  }
  LoopbackGroup* g_;
  int rank_;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
  std::string err_;
};

}  // namespace

LoopbackGroup::LoopbackGroup(int world) : slots(world), world_(world) {}

void LoopbackGroup::barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  const long gen = generation_;
  if (++arrived_ == world_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
  } else {
    cv_.wait(lk, [&] { return generation_ != gen; });
  }
}

Comm* make_nccl_comm(int rank, int world, const void* id128) {
  void* c = nccl_comm_init(world, rank, id128);
  if (!c) return nullptr;
  return new NcclComm(rank, world, c);
}

Comm* make_loopback_comm(LoopbackGroup* g, int rank) { return new LoopbackComm(g, rank); }

}  // namespace ciq
