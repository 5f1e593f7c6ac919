#include "comm.h"

#include <nccl.h>
#include <stdlib.h>
#include <string.h>

#include <chrono>
#include <condition_variable>
#include <map>
#include <mutex>
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

CommCounts Comm::total_counts() const {
  CommCounts c = counts;
  for (const auto& ch : children_) {
    const CommCounts d = ch->total_counts();
    c.allgather += d.allgather; c.reduce_scatter += d.reduce_scatter; c.allreduce += d.allreduce;
    c.ag_bytes += d.ag_bytes; c.rs_bytes += d.rs_bytes; c.ar_bytes += d.ar_bytes;
  }
  return c;
}

// ------------------------------------------------------------------------------------------------
// NCCL
class NcclComm : public Comm {
 public:
  NcclComm(ncclComm_t c, int rank, int world) : comm_(c) {
    rank_ = rank;
    world_ = world;
  }
  ~NcclComm() override {
    children_.clear();
    if (comm_) ncclCommDestroy(comm_);
  }
  void live() const {
    if (!comm_) throw Error(SLQ_ENCCL, "the NCCL communicator was aborted (watchdog or peer failure)");
  }
  void allgather(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) override {
    live();
    SLQ_NCCL(ncclAllGather(send, recv, count, nt(t), comm_, s));
    counts.allgather++;
    counts.ag_bytes += (double)count * nsize(t) * world_;
  }
  void reduce_scatter(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) override {
    live();
    SLQ_NCCL(ncclReduceScatter(send, recv, count, nt(t), ncclSum, comm_, s));
    counts.reduce_scatter++;
    counts.rs_bytes += (double)count * nsize(t) * world_;
  }
  void allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) override {
    live();
    SLQ_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, comm_, s));
    counts.allreduce++;
    counts.ar_bytes += 8.0 * count;
  }
  void abort() override {
    for (auto& ch : children_) ch->abort();
    if (comm_) ncclCommAbort(comm_);
    comm_ = nullptr;
  }
  bool aborted() const override { return comm_ == nullptr; }
  void check_async() override {
    ncclResult_t ae = ncclSuccess;
    if (comm_ && ncclCommGetAsyncError(comm_, &ae) != ncclSuccess) ae = ncclSystemError;
    for (auto& ch : children_)
      if (ae == ncclSuccess || ae == ncclInProgress) {
        try {
          ch->check_async();
        } catch (const Error&) {
          ae = ncclSystemError;
        }
      }
    if (ae != ncclSuccess && ae != ncclInProgress) {
      abort();
      throw Error(SLQ_ENCCL, std::string("NCCL asynchronous error (peer failure?): ") + ncclGetErrorString(ae));
    }
  }
  Comm* split(int color) override {
    live();
    ncclComm_t nc = nullptr;
    SLQ_NCCL(ncclCommSplit(comm_, color, rank_, &nc, nullptr));
    children_.emplace_back(new NcclComm(nc, rank_, world_));
    return children_.back().get();
  }

 private:
  ncclComm_t comm_ = nullptr;
};

std::unique_ptr<Comm> make_nccl_comm(const void* uid, int rank, int world, int device) {
  SLQ_CHECK_ARG(uid != nullptr, "nccl_unique_id required for world_size > 1");
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  SLQ_CUDA(cudaSetDevice(device));
  ncclComm_t c;
  SLQ_NCCL(ncclCommInitRank(&c, world, id, rank));
  return std::unique_ptr<Comm>(new NcclComm(c, rank, world));
}

// ------------------------------------------------------------------------------------------------
// LOOPBACK (test only): in-process ranks on one GPU, host-synchronous collectives
namespace {

struct LoopGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;
  std::vector<const void*> ptrs;
  // every rank meets here; SLQ_ETIMEOUT after timeout_s (<= 0: forever), SLQ_ENCCL if a peer aborted
  void barrier(double timeout_s) {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) throw Error(SLQ_ENCCL, "loopback group aborted by a peer");
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    auto done = [&] { return gen != g || broken; };
    if (timeout_s > 0) {
      if (!cv.wait_for(lk, std::chrono::duration<double>(timeout_s), done)) {
        broken = true;
        cv.notify_all();
        throw Error(SLQ_ETIMEOUT, "loopback barrier: a peer did not arrive within the watchdog timeout");
      }
    } else {
      cv.wait(lk, done);
    }
    if (broken) throw Error(SLQ_ENCCL, "loopback group aborted by a peer");
  }
  void publish(int rank, const void* p) {
    std::lock_guard<std::mutex> lk(mu);
    ptrs[rank] = p;
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

std::mutex g_reg_mu;
std::map<std::string, std::weak_ptr<LoopGroup>> g_reg;

std::shared_ptr<LoopGroup> join_group(const std::string& key, int world) {
  std::lock_guard<std::mutex> lk(g_reg_mu);
  auto it = g_reg.find(key);
  if (it != g_reg.end())
    if (auto g = it->second.lock()) {
      SLQ_CHECK_ARG(g->world == world, "loopback group: world_size differs between ranks");
      return g;
    }
  auto g = std::make_shared<LoopGroup>();
  g->world = world;
  g->ptrs.assign(world, nullptr);
  g_reg[key] = g;
  return g;
}

constexpr int kMaxLoopRanks = 8;
struct RankPtrs {
  const void* p[kMaxLoopRanks];
};

// out[i] = sum_{r = 0..R-1} src_r[off + i], ranks summed in order 0, 1, ..., R-1
template <class T>
__global__ void k_sum_ranks(RankPtrs src, int R, int64_t off, T* out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    T acc = reinterpret_cast<const T*>(src.p[0])[off + i];
    for (int r = 1; r < R; ++r) acc += reinterpret_cast<const T*>(src.p[r])[off + i];
    out[i] = acc;
  }
}

}  // namespace

class LoopbackComm : public Comm {
 public:
  LoopbackComm(const std::string& key, int rank, int world, int device) : key_(key), device_(device) {
    SLQ_CHECK_ARG(world >= 1 && world <= kMaxLoopRanks, "loopback: 1 <= world_size <= 8");
    rank_ = rank;
    world_ = world;
    g_ = join_group(key, world);
  }
  ~LoopbackComm() override {
    children_.clear();
    if (tmp_) cudaFree(tmp_);
  }
  bool host_sync() const override { return true; }
  void live() const {
    if (aborted_) throw Error(SLQ_ENCCL, "the loopback communicator was aborted");
  }
  void allgather(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) override {
    live();
    const size_t b = count * nsize(t);
    enter(send, s);
    for (int r = 0; r < world_; ++r)
      SLQ_CUDA(cudaMemcpyAsync((char*)recv + r * b, g_->ptrs[r], b, cudaMemcpyDeviceToDevice, s));
    leave(s);
    counts.allgather++;
    counts.ag_bytes += (double)b * world_;
  }
  void reduce_scatter(const void* send, void* recv, size_t count, CommType t, cudaStream_t s) override {
    live();
    enter(send, s);
    sum(t, (int64_t)rank_ * (int64_t)count, recv, count, s);
    leave(s);
    counts.reduce_scatter++;
    counts.rs_bytes += (double)count * nsize(t) * world_;
  }
  void allreduce_sum_f64(double* buf, size_t count, cudaStream_t s) override {
    live();
    if (tmp_bytes_ < 8 * count) {
      if (tmp_) SLQ_CUDA(cudaFree(tmp_));
      tmp_ = nullptr;
      SLQ_CUDA(cudaMalloc(&tmp_, 8 * count));
      tmp_bytes_ = 8 * count;
    }
    enter(buf, s);
    sum(COMM_F64, 0, tmp_, count, s);
    leave(s);  // every rank has read every buf
    SLQ_CUDA(cudaMemcpyAsync(buf, tmp_, 8 * count, cudaMemcpyDeviceToDevice, s));
    counts.allreduce++;
    counts.ar_bytes += 8.0 * count;
  }
  void abort() override {
    for (auto& ch : children_) ch->abort();
    aborted_ = true;
    g_->abort();
  }
  bool aborted() const override { return aborted_; }
  void check_async() override {}
  Comm* split(int color) override {
    live();
    const std::string k = key_ + "/split" + std::to_string(nsplit_++) + "." + std::to_string(color);
    children_.emplace_back(new LoopbackComm(k, rank_, world_, device_));
    return children_.back().get();
  }

 private:
  void enter(const void* mine, cudaStream_t s) {
    SLQ_CUDA(cudaStreamSynchronize(s));  // `mine` is complete
    g_->publish(rank_, mine);
    barrier();
  }
  void leave(cudaStream_t s) {
    SLQ_CUDA(cudaStreamSynchronize(s));  // this rank is done reading the peers' buffers
    barrier();
  }
  void barrier() {
    try {
      g_->barrier(watchdog_timeout_s());
    } catch (...) {
      aborted_ = true;
      throw;
    }
  }
  void sum(CommType t, int64_t off, void* out, size_t count, cudaStream_t s) {
    if (count == 0) return;
    RankPtrs rp;
    for (int r = 0; r < kMaxLoopRanks; ++r) rp.p[r] = r < world_ ? g_->ptrs[r] : nullptr;
    const int blocks = (int)std::min<int64_t>(((int64_t)count + 255) / 256, 148 * 8);
    if (t == COMM_F64)
      k_sum_ranks<double><<<blocks, 256, 0, s>>>(rp, world_, off, (double*)out, (int64_t)count);
    else
      k_sum_ranks<float><<<blocks, 256, 0, s>>>(rp, world_, off, (float*)out, (int64_t)count);
    SLQ_CUDA(cudaGetLastError());
  }
  std::string key_;
  int device_;
  std::shared_ptr<LoopGroup> g_;
  bool aborted_ = false;
  int nsplit_ = 0;
  void* tmp_ = nullptr;
  size_t tmp_bytes_ = 0;
};

std::unique_ptr<Comm> make_loopback_comm(const void* key128, int rank, int world, int device) {
  SLQ_CHECK_ARG(key128 != nullptr, "loopback: a 128-byte group key in nccl_unique_id");
  std::string key((const char*)key128, 128);
  SLQ_CUDA(cudaSetDevice(device));
  return std::unique_ptr<Comm>(new LoopbackComm(key, rank, world, device));
}

// ------------------------------------------------------------------------------------------------
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

}  // namespace slq
