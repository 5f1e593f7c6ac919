// NCCL collectives of the FSDP path: per-unit all-gather of the working
// parameters, per-unit reduce-scatter (sum) of gradients, and the small fp64 all-reduces of the
// Lanczos scalars.  All calls are stream-ordered on the caller's stream.
#pragma once

#include <stddef.h>
#include <stdint.h>

#include <cuda_runtime.h>

namespace slq {

enum CommType { COMM_F32 = 0, COMM_F64 = 1 };

struct CommCounts {
  int64_t allgather = 0, reduce_scatter = 0, allreduce = 0;
  double ag_bytes = 0, rs_bytes = 0, ar_bytes = 0;
};

class Comm {
 public:
  Comm(const void* unique_id128, int rank, int world, int device);
  ~Comm();
  void allgather(const void* send, void* recv, size_t count_per_rank, CommType t, cudaStream_t s);
  void reduce_scatter(const void* send, void* recv, size_t count_per_rank, CommType t, cudaStream_t s);
  void allreduce_sum_f64(double* buf, size_t count, cudaStream_t s);
  void abort();
  int rank() const { return rank_; }
  int world() const { return world_; }
  CommCounts counts;

 private:
  void* comm_ = nullptr;  // ncclComm_t
  int rank_, world_;
};

void nccl_unique_id(void* out128);

}  // namespace slq
