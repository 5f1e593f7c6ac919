// Collectives of the FSDP path: per-unit all-gather of the working parameters,
// per-unit reduce-scatter (sum) of gradients, and the small fp64 all-reduces of the Lanczos
// scalars.  All calls are stream-ordered on the caller's stream.
//
// Two backends behind one interface: NCCL (the product path, one process per GPU) and LOOPBACK
// (test only, SLQ_COMM_LOOPBACK in slq.h): the ranks are contexts of one process on one GPU, one
// host thread each, and every collective is host-synchronous -- the caller's stream is drained, the
// ranks meet at a host barrier, the data moves by device copies / a fixed rank-order sum kernel,
// and a second barrier releases the send buffers.  No kernel ever waits on another rank's kernel.
#pragma once

#include <stddef.h>
#include <stdint.h>

#include <memory>
#include <vector>

#include <cuda_runtime.h>

namespace slq {

enum CommType { COMM_F32 = 0, COMM_F64 = 1 };

struct CommCounts {
  int64_t allgather = 0, reduce_scatter = 0, allreduce = 0;
  double ag_bytes = 0, rs_bytes = 0, ar_bytes = 0;
};

class Comm {
 public:
  virtual ~Comm() {}
  virtual void allgather(const void* send, void* recv, size_t count_per_rank, CommType t, cudaStream_t s) = 0;
  virtual void reduce_scatter(const void* send, void* recv, size_t count_per_rank, CommType t, cudaStream_t s) = 0;
  virtual void allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) = 0;
  // abort this communicator and every communicator split from it
  virtual void abort() = 0;
  virtual bool aborted() const = 0;
  // throws SLQ_ENCCL (after aborting) on an asynchronous error of this or a split communicator
  virtual void check_async() = 0;
  // collective: a new communicator over the same ranks (one per concurrent gradient pass), owned
  // by this one (aborted with it, counted in total_counts)
  virtual Comm* split(int color) = 0;
  // true: collectives block the host (loopback) -- they cannot be captured into CUDA graphs
  virtual bool host_sync() const { return false; }
  int rank() const { return rank_; }
  int world() const { return world_; }
  CommCounts counts;
  CommCounts total_counts() const;  // this communicator plus its splits

 protected:
  int rank_ = 0, world_ = 1;
  std::vector<std::unique_ptr<Comm>> children_;
};

std::unique_ptr<Comm> make_nccl_comm(const void* unique_id128, int rank, int world, int device);
std::unique_ptr<Comm> make_loopback_comm(const void* key128, int rank, int world, int device);

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
