#include "comm.h"

#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <string>
#include <thread>

#include "common.h"

namespace slq {

#define SLQ_NCCL(expr)                                                                                  \
  do {                                                                                                  \
    ncclResult_t r_ = (expr);                                                                           \
    if (r_ != ncclSuccess) throw Error(SLQ_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(r_)); \
  } while (0)

static ncclDataType_t nt(CommType t) { return t == COMM_F64 ? ncclFloat64 : ncclFloat32; }
static size_t nsize(CommType t) { return t == COMM_F64 ? 8 : 4; }

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  SLQ_NCCL(ncclGetUniqueId(&id));
  memcpy(out128, &id, sizeof(id));
}

Comm::Comm(const void* uid, int rank, int world, int device) : rank_(rank), world_(world) {
  SLQ_CHECK_ARG(uid != nullptr, "nccl_unique_id required for world_size > 1");
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  SLQ_CUDA(cudaSetDevice(device));
  ncclComm_t c;
  SLQ_NCCL(ncclCommInitRank(&c, world, id, rank));
  comm_ = c;
}

Comm::~Comm() {
  if (comm_) ncclCommDestroy((ncclComm_t)comm_);
}

void Comm::abort() {
  if (comm_) ncclCommAbort((ncclComm_t)comm_);
  comm_ = nullptr;
}

#define SLQ_LIVE() \
  if (!comm_) throw Error(SLQ_ENCCL, "the NCCL communicator was aborted (watchdog or peer failure)")

void Comm::allgather(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) {
  SLQ_LIVE();
  SLQ_NCCL(ncclAllGather(send, recv, count, nt(t), (ncclComm_t)comm_, s));
  counts.allgather++;
  counts.ag_bytes += (double)count * nsize(t) * world_;
}

void Comm::reduce_scatter(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) {
  SLQ_LIVE();
  SLQ_NCCL(ncclReduceScatter(send, recv, count, nt(t), ncclSum, (ncclComm_t)comm_, s));
  counts.reduce_scatter++;
  counts.rs_bytes += (double)count * nsize(t) * world_;
}

void Comm::allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) {
  SLQ_LIVE();
  SLQ_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)comm_, s));
  counts.allreduce++;
  counts.ar_bytes += 8.0 * count;
}

double watchdog_timeout_s() {
  static const double t = getenv("SLQ_TIMEOUT_S") ? atof(getenv("SLQ_TIMEOUT_S")) : 1800.0;
  return t;
}

void watchdog_wait(cudaStream_t s, Comm* comm, double timeout_s) {
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  for (int polls = 0;; ++polls) {
    const cudaError_t e = cudaStreamQuery(s);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) throw Error(SLQ_ECUDA, std::string("stream: ") + cudaGetErrorString(e));
    if (comm && !comm->aborted()) comm->check_async();
    const double dt = std::chrono::duration<double>(clk::now() - t0).count();
    if (timeout_s > 0 && dt > timeout_s) {
      if (comm) comm->abort();
      throw Error(SLQ_ETIMEOUT, "watchdog: the stream did not drain within " + std::to_string(timeout_s) +
                                    " s (communicator aborted)");
    }
    // spin briefly (short kernels), then back off to 50 us sleeps
    if (polls > 200) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

void Comm::check_async() {
  ncclResult_t ae = ncclSuccess;
  if (ncclCommGetAsyncError((ncclComm_t)comm_, &ae) != ncclSuccess) ae = ncclSystemError;
  if (ae != ncclSuccess && ae != ncclInProgress) {
    abort();
    throw Error(SLQ_ENCCL, std::string("NCCL asynchronous error (peer failure?): ") + ncclGetErrorString(ae));
  }
}

}  // namespace slq
