// hostcomm.h -- node-local shared-memory collective of a multi-process engine
// (see hostcomm.cu).  Host code only.
#pragma once

#include <stdint.h>

#include <functional>
#include <memory>
#include <vector>

namespace tg {

class HostComm {
 public:
  // Collective over the `world` ranks: rank 0 creates a segment, its name is
  // shared through `allgather(send, recv, bytes)` (recv = world x bytes),
  // every rank maps it, `barrier()` follows.  nullptr (every rank) if any
  // rank could not map it: the caller keeps using its callbacks.
  static std::unique_ptr<HostComm> create(
      int rank, int world, const std::function<void(const void*, void*, uint64_t)>& allgather,
      const std::function<void()>& barrier);
  ~HostComm();
  // In-place allreduce of n <= 16 values, ops[i] 0 = sum, 1 = min.  Collective
  // (SPMD: every rank calls with the same n and ops).  false on timeout.
  bool allreduce(uint64_t* data, int n, const int* ops, double timeout_s = 600.0);
  int rank() const { return rank_; }
  int world() const { return world_; }

 private:
  HostComm() = default;
  int rank_ = 0, world_ = 1;
  void* base_ = nullptr;
  size_t bytes_ = 0;
  uint64_t epoch_ = 0;
};

}  // namespace tg
