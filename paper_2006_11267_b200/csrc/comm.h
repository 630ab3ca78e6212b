// comm.h -- the two collectives of the row-sharded msMINRES-CIQ loop:
//   allgather: every rank contributes `bytes` (its row block of the next Lanczos vector, or its
//              T fp64 partial sums) and receives all ranks' blocks in rank order;
// cross-rank sums are an allgather followed by a fixed-order (rank 0, 1, ...) device sum, so the
// scalar recurrence state is bit-identical on all ranks without relying on NCCL's reduction order.
//
// Backends: NCCL (one process per GPU, NVLink/NVSwitch) and Loopback (G ranks as threads of one
// process sharing one GPU: device copies + host barriers) -- the latter exercises the sharded
// code path on a single GPU in tests.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

#include <condition_variable>
#include <mutex>
#include <vector>

namespace ciq {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // recv[r * bytes .. (r+1) * bytes) <- rank r's send (send may alias recv + rank * bytes)
  virtual bool allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  virtual const char* error() const = 0;
  virtual bool capturable() const = 0;  // may the collective be captured in a CUDA graph?
};

Comm* make_nccl_comm(int rank, int world, const void* id128);

// Host-side rendezvous shared by the loopback ranks.
class LoopbackGroup {
 public:
  explicit LoopbackGroup(int world);
  int world() const { return world_; }
  void barrier();
  struct Slot {
    const void* send = nullptr;
    cudaEvent_t ready = nullptr;
    cudaEvent_t done = nullptr;
  };
  std::vector<Slot> slots;

 private:
  int world_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  long generation_ = 0;
};

Comm* make_loopback_comm(LoopbackGroup* g, int rank);

}  // namespace ciq
