#include "comm.h"

#include <nccl.h>
#include <string.h>

#include <string>

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

void Comm::allgather(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) {
  SLQ_NCCL(ncclAllGather(send, recv, count, nt(t), (ncclComm_t)comm_, s));
  counts.allgather++;
  counts.ag_bytes += (double)count * nsize(t) * world_;
}

void Comm::reduce_scatter(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) {
  SLQ_NCCL(ncclReduceScatter(send, recv, count, nt(t), ncclSum, (ncclComm_t)comm_, s));
  counts.reduce_scatter++;
  counts.rs_bytes += (double)count * nsize(t) * world_;
}

void Comm::allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) {
  SLQ_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, (ncclComm_t)comm_, s));
  counts.allreduce++;
  counts.ar_bytes += 8.0 * count;
}

}  // namespace slq
