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
  bool aborted() const { return comm_ == nullptr; }
  void check_async();  // throws SLQ_ENCCL (after aborting) on an asynchronous NCCL error
  int rank() const { return rank_; }
  int world() const { return world_; }
  CommCounts counts;

 private:
  void* comm_ = nullptr;  // ncclComm_t
  int rank_, world_;
};

void nccl_unique_id(void* out128);

// Collective watchdog: wait for `s` to drain, polling the stream and, when `comm`
// is given, the communicator's asynchronous error state.  A NCCL error (e.g. a peer that died)
// aborts the communicator and throws SLQ_ENCCL; no completion within `timeout_s` seconds
// (<= 0: wait forever) aborts it and throws SLQ_ETIMEOUT.  Without a communicator (world size 1)
// only the timeout applies.  After an abort every later collective throws SLQ_ENCCL.
void watchdog_wait(cudaStream_t s, Comm* comm, double timeout_s);
// SLQ_TIMEOUT_S from the environment (default 1800 s; 0 disables the timeout)
double watchdog_timeout_s();
// diagnostic: a one-thread kernel that keeps `s` busy for `ms` milliseconds (diag.cu)
void diag_stall(cudaStream_t s, int ms);

}  // namespace slq
