// C-ABI of libslq.so (include/slq.h): argument checking, context lifetime, host/device buffer
// marshalling, the per-kernel-class CUDA-event profiler.  No torch types cross this boundary.
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "comm.h"
#include "common.h"
#include "engine.h"
#include "kernels.h"
#include "layout.h"

namespace slq {
void tridiag_gauss(const double* alpha, const double* beta, int m, double* nodes, double* weights);
void ghost_clusters(const double* nodes, int m, double tol, int32_t* cluster_id, int32_t* n_ghost, double* max_split);
void slq_average(const double* nodes, const double* weights, const int32_t* mc, int np, int jmax, double* mom,
                 const double* grid, int ng, double sigma, double* dens);

const char* kernel_class_name(int c) {
  static const char* names[KC_COUNT] = {"gemm", "attention", "norm", "cross_entropy", "embedding",
                                        "elementwise", "perturb", "fd_lanczos", "reorth", "vector", "gemm_i8",
                                        "oz_slice", "attn_i8"};
  return (c >= 0 && c < KC_COUNT) ? names[c] : "?";
}

// Per-kernel-class CUDA-event profiler.  Mode 1 (serial): the library runs every launch of a pass
// on one stream (no side stream, no concurrent passes), so each launch's event duration is its
// own.  Mode 2 (overlap-aware): the execution keeps its concurrency (two passes, side streams),
// and besides the summed durations each class gets its BUSY time -- the length of the union of its
// launches' [start, end] intervals on the device timeline (events are timed against one reference
// event), i.e. the wall time during which at least one kernel of that class ran.  Busy time never
// exceeds the profiled region, so a class's share of a step is busy / step time.
struct Profiler {
  bool on = false;
  int mode = 1;
  struct Rec {
    cudaEvent_t a, b;
    int cls;
    double flops, bytes;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t open = nullptr;
  cudaEvent_t t0 = nullptr;  // reference of the interval timeline (mode 2)
  double ms[KC_COUNT] = {}, flops[KC_COUNT] = {}, bytes[KC_COUNT] = {};
  int64_t count[KC_COUNT] = {};
  std::vector<std::pair<float, float>> iv[KC_COUNT];
  cudaEvent_t take() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  void flush() {
    for (Rec& r : pending) {
      cudaEventSynchronize(r.b);
      float t = 0;
      cudaEventElapsedTime(&t, r.a, r.b);
      ms[r.cls] += t;
      flops[r.cls] += r.flops;
      bytes[r.cls] += r.bytes;
      count[r.cls]++;
      if (t0) {
        float s = 0, e = 0;
        cudaEventElapsedTime(&s, t0, r.a);
        cudaEventElapsedTime(&e, t0, r.b);
        iv[r.cls].push_back({s, e});
      }
      pool.push_back(r.a);
      pool.push_back(r.b);
    }
    pending.clear();
  }
  // union length of the intervals of class c (c < 0: of every class)
  double busy(int c) {
    flush();
    std::vector<std::pair<float, float>> v;
    for (int i = 0; i < KC_COUNT; ++i)
      if (c < 0 || c == i) v.insert(v.end(), iv[i].begin(), iv[i].end());
    std::sort(v.begin(), v.end());
    double tot = 0, cs = 0, ce = -1e30;
    for (auto& x : v) {
      if (x.first > ce) {
        if (ce > cs) tot += ce - cs;
        cs = x.first;
        ce = x.second;
      } else {
        ce = std::max(ce, (double)x.second);
      }
    }
    if (ce > cs) tot += ce - cs;
    return tot;
  }
  void reset(cudaStream_t s) {
    flush();
    for (int i = 0; i < KC_COUNT; ++i) ms[i] = flops[i] = bytes[i] = 0, count[i] = 0, iv[i].clear();
    if (!t0) cudaEventCreate(&t0);
    cudaEventRecord(t0, s);
  }
  ~Profiler() {
    flush();
    for (auto e : pool) cudaEventDestroy(e);
    if (t0) cudaEventDestroy(t0);
  }
};

bool prof_enabled(const Profiler* p) { return p && p->on; }
bool prof_serial(const Profiler* p) { return p && p->on && p->mode == 1; }

void prof_begin(Profiler* p, int, cudaStream_t s) {
  if (!p || !p->on) return;
  p->open = p->take();
  cudaEventRecord(p->open, s);
}
void prof_end(Profiler* p, int cls, cudaStream_t s, double flops, double bytes) {
  if (!p || !p->on || !p->open) return;
  cudaEvent_t e = p->take();
  cudaEventRecord(e, s);
  p->pending.push_back({p->open, e, cls, flops, bytes});
  p->open = nullptr;
  if (p->pending.size() > 200000) p->flush();
}

// A grown workspace keeps its previous buffers alive until destruction: captured CUDA graphs may
// still reference them (freeing them made later graph replays fault).
void* Workspace::get(size_t need, cudaStream_t) {
  if (need <= bytes) return ptr;
  if (ptr) retired.push_back(ptr);
  ptr = nullptr;
  bytes = 0;
  const size_t nb = need + need / 4 + 4096;
  SLQ_CUDA(cudaMalloc(&ptr, nb));
  bytes = nb;
  return ptr;
}
void Workspace::reserve(size_t need) {
  if (need <= bytes) return;
  if (ptr) retired.push_back(ptr);
  ptr = nullptr;
  bytes = 0;
  SLQ_CUDA(cudaMalloc(&ptr, need));
  bytes = need;
}
unsigned* Workspace::counters(size_t n) {
  if (n > kCounters) return nullptr;
  if (!cnt) {
    SLQ_CUDA(cudaMalloc(&cnt, sizeof(unsigned) * kCounters));
    SLQ_CUDA(cudaMemset(cnt, 0, sizeof(unsigned) * kCounters));
  }
  return cnt;
}
Workspace::~Workspace() {
  if (!ptr && !cnt && retired.empty()) return;
  cudaDeviceSynchronize();
  if (ptr) cudaFree(ptr);
  if (cnt) cudaFree(cnt);
  for (void* p : retired) cudaFree(p);
}

}  // namespace slq

using namespace slq;

struct slq_ctx {
  slq_model_desc desc;
  slq_world world;
  LayoutPlan plan;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::unique_ptr<Comm> comm;
  Profiler prof;
  Workspace ws;
  int64_t launches = 0;
  std::unique_ptr<Engine> engine;
  std::string err;
  float* stage_in = nullptr;  // device staging for host-pointer calls
  float* stage_out = nullptr;
  cudaEvent_t ev_entry = nullptr;  // library-owned stream: orders each call after the legacy stream
  Launch launch() { return Launch{stream, &prof, &ws, &launches}; }
  ~slq_ctx() {
    if (stream) cudaStreamSynchronize(stream);
    engine.reset();
    if (stage_in) cudaFree(stage_in);
    if (stage_out) cudaFree(stage_out);
    if (ev_entry) cudaEventDestroy(ev_entry);
    comm.reset();
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

namespace {
thread_local std::string g_err;

slq_status fail(slq_ctx* ctx, slq_status s, const std::string& msg) {
  if (ctx) ctx->err = msg;
  g_err = msg;
  return s;
}

template <class F>
slq_status guarded(slq_ctx* ctx, F&& f) {
  try {
    f();
    return SLQ_OK;
  } catch (const Error& e) {
    return fail(ctx, e.status, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ctx, SLQ_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, SLQ_ECUDA, e.what());
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// entry check of every call that runs the engine: the device, and a communicator that a watchdog
// or an asynchronous NCCL error aborted (its captured graphs reference it: never replay them)
// A library-owned stream is non-blocking (the library's internal streams synchronise with it by
// events only), so each entry point makes it wait for the work already queued on the legacy
// default stream, where callers (e.g. torch's default stream) write the device shards they pass.
void check_device(slq_ctx* ctx) {
  SLQ_CUDA(cudaSetDevice(ctx->world.device));
  if (ctx->comm && ctx->comm->aborted())
    throw Error(SLQ_ENCCL, "the NCCL communicator was aborted (watchdog or peer failure); destroy the context");
  if (ctx->own_stream && ctx->ev_entry) {
    SLQ_CUDA(cudaEventRecord(ctx->ev_entry, cudaStreamLegacy));
    SLQ_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_entry, 0));
  }
}

void ensure_stage(slq_ctx* ctx) {
  if (!ctx->stage_in) {
    SLQ_CUDA(cudaMalloc(&ctx->stage_in, sizeof(float) * (size_t)ctx->plan.P_loc));
    SLQ_CUDA(cudaMalloc(&ctx->stage_out, sizeof(float) * (size_t)ctx->plan.P_loc));
  }
}

// float4 paths need 16-byte aligned shards; stage misaligned device pointers
bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
}  // namespace

extern "C" {

const char* slq_last_error(const slq_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

slq_status slq_plan_layout(const slq_model_desc* desc, int32_t world, int64_t* P, int64_t* P_loc, int32_t* n_units,
                           int64_t* table) {
  return guarded(nullptr, [&] {
    SLQ_CHECK_ARG(desc != nullptr, "desc");
    LayoutPlan p = plan_layout(*desc, world);
    if (P) *P = p.P;
    if (P_loc) *P_loc = p.P_loc;
    if (n_units) *n_units = (int32_t)p.units.size();
    if (table)
      for (size_t u = 0; u < p.units.size(); ++u) {
        table[4 * u + 0] = p.units[u].global_offset;
        table[4 * u + 1] = p.units[u].numel;
        table[4 * u + 2] = p.units[u].local_offset;
        table[4 * u + 3] = p.units[u].chunk;
      }
  });
}

slq_status slq_plan_memory(const slq_model_desc* desc, int32_t world_size, int32_t n_local, int64_t* bytes) {
  return guarded(nullptr, [&] {
    SLQ_CHECK_ARG(desc != nullptr && bytes != nullptr, "desc / bytes");
    plan_memory(*desc, world_size, n_local, bytes);
  });
}

slq_status slq_nccl_unique_id(void* out128) {
  return guarded(nullptr, [&] {
    SLQ_CHECK_ARG(out128 != nullptr, "out");
    nccl_unique_id(out128);
  });
}

slq_status slq_init(const slq_model_desc* desc, const slq_batch* batch, const slq_world* world, slq_ctx** out) {
  if (out) *out = nullptr;
  std::unique_ptr<slq_ctx> ctx(new slq_ctx());
  slq_status st = guarded(nullptr, [&] {
    SLQ_CHECK_ARG(desc && batch && world && out, "null argument");
    SLQ_CHECK_ARG(world->world_size >= 1 && world->rank >= 0 && world->rank < world->world_size, "rank/world");
    ctx->desc = *desc;
    ctx->world = *world;
    ctx->plan = plan_layout(*desc, world->world_size);
    SLQ_CHECK_ARG(batch->params_host != nullptr, "params_host");
    HostBatch hb;
    if (desc->arch == SLQ_ARCH_MLP) {
      SLQ_CHECK_ARG(batch->n_rows_local >= 1 && batch->n_rows_global >= batch->n_rows_local, "n_rows");
      SLQ_CHECK_ARG(batch->x && batch->y, "x / y");
      hb.n_rows = batch->n_rows_local;
      hb.n_rows_global = batch->n_rows_global;
      hb.x.assign(batch->x, batch->x + (size_t)hb.n_rows * desc->d_in);
      hb.y.assign(batch->y, batch->y + hb.n_rows);
      for (int32_t v : hb.y) SLQ_CHECK_ARG(v >= 0 && v < desc->n_classes, "label out of range");
    } else {
      SLQ_CHECK_ARG(batch->n_seq_local >= 1 && batch->n_seq_global >= batch->n_seq_local, "n_seq");
      SLQ_CHECK_ARG(batch->tokens, "tokens");
      hb.n_seq = batch->n_seq_local;
      hb.n_seq_global = batch->n_seq_global;
      hb.tokens.assign(batch->tokens, batch->tokens + (size_t)hb.n_seq * (desc->seq_len + 1));
      for (int32_t v : hb.tokens) SLQ_CHECK_ARG(v >= 0 && v < desc->vocab, "token id out of range");
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(SLQ_ECUDA, "no CUDA device: the CUDA path is required (no CPU fallback exists)");
    SLQ_CHECK_ARG(world->device >= 0 && world->device < ndev, "device");
    check_device(ctx.get());
    if (world->cuda_stream) {
      ctx->stream = (cudaStream_t)world->cuda_stream;
    } else {
      SLQ_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
      ctx->own_stream = true;
      SLQ_CUDA(cudaEventCreateWithFlags(&ctx->ev_entry, cudaEventDisableTiming));
    }
    SLQ_CHECK_ARG(world->comm_backend == SLQ_COMM_NCCL || world->comm_backend == SLQ_COMM_LOOPBACK, "comm_backend");
    {  // the device-memory plan against the free memory, before allocating anything
      int64_t mem[SLQ_MEM_COUNT];
      plan_memory(*desc, world->world_size,
                  desc->arch == SLQ_ARCH_MLP ? batch->n_rows_local : batch->n_seq_local, mem);
      size_t free_b = 0, total_b = 0;
      SLQ_CUDA(cudaMemGetInfo(&free_b, &total_b));
      static const char* names[SLQ_MEM_COUNT] = {"theta", "points", "grads", "lanczos", "fsdp", "activations",
                                                 "logits", "scratch", "workspace", "total"};
      std::string m;
      for (int i = 0; i < SLQ_MEM_COUNT; ++i) m += std::string(" ") + names[i] + "=" + std::to_string(mem[i] >> 20) + "MiB";
      // SLQ_VERBOSE=1: print the plan of every context (rank, world size, free memory)
      if (getenv("SLQ_VERBOSE") && atoi(getenv("SLQ_VERBOSE")) > 0)
        fprintf(stderr, "[slq] rank %d/%d device memory plan:%s (free %zu MiB)\n", world->rank, world->world_size,
                m.c_str(), free_b >> 20);
      if ((size_t)mem[SLQ_MEM_TOTAL] > free_b)
        throw Error(SLQ_ENOMEM, "device memory plan exceeds the free memory (" + std::to_string(free_b >> 20) +
                                    " MiB):" + m + " (try act_ckpt = 1, a larger world_size or a smaller batch)");
    }
    if (world->world_size > 1) {
      if (world->comm_backend == SLQ_COMM_LOOPBACK)
        ctx->comm = make_loopback_comm(world->nccl_unique_id, world->rank, world->world_size, world->device);
      else
        ctx->comm = make_nccl_comm(world->nccl_unique_id, world->rank, world->world_size, world->device);
    } else if (getenv("SLQ_FORCE_NCCL") && atoi(getenv("SLQ_FORCE_NCCL")) != 0) {
      // diagnostic: a one-rank NCCL communicator, so the FSDP path (per-unit all-gather /
      // reduce-scatter, scalar all-reduces) runs on a single GPU (tests/test_gpu_fsdp1.py)
      char uid[128];
      nccl_unique_id(uid);
      ctx->comm = make_nccl_comm(uid, 0, 1, world->device);
    }
    ctx->engine = make_engine(*desc, ctx->plan, hb, batch->params_host, world->rank, ctx->comm.get(),
                              ctx->launch());
  });
  if (st == SLQ_OK) *out = ctx.release();
  return st;
}

slq_status slq_destroy(slq_ctx* ctx) {
  delete ctx;
  return SLQ_OK;
}

int64_t slq_local_len(const slq_ctx* ctx) { return ctx ? ctx->plan.P_loc : -1; }
int64_t slq_global_len(const slq_ctx* ctx) { return ctx ? ctx->plan.P : -1; }
int32_t slq_num_units(const slq_ctx* ctx) { return ctx ? (int32_t)ctx->plan.units.size() : -1; }

slq_status slq_unit_info(const slq_ctx* ctx, int32_t u, int64_t* g, int64_t* numel, int64_t* l, int64_t* chunk) {
  if (!ctx || u < 0 || u >= (int32_t)ctx->plan.units.size()) return fail(nullptr, SLQ_EINVAL, "unit index");
  const UnitPlan& p = ctx->plan.units[u];
  if (g) *g = p.global_offset;
  if (numel) *numel = p.numel;
  if (l) *l = p.local_offset;
  if (chunk) *chunk = p.chunk;
  return SLQ_OK;
}

slq_status slq_hvp(slq_ctx* ctx, const float* v, float* out, double eps) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    SLQ_CHECK_ARG(v && out, "null v/out");
    SLQ_CHECK_ARG(eps > 0, "eps > 0");
    SLQ_CHECK_ARG(v != out, "v and out must not alias");
    check_device(ctx);
    const size_t bytes = sizeof(float) * (size_t)ctx->plan.P_loc;
    const bool vdev = is_device_ptr(v), odev = is_device_ptr(out);
    const float* vd = v;
    float* od = out;
    if (!vdev || !aligned16(v)) {
      ensure_stage(ctx);
      SLQ_CUDA(cudaMemcpyAsync(ctx->stage_in, v, bytes, vdev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                               ctx->stream));
      vd = ctx->stage_in;
    }
    if (!odev) {
      ensure_stage(ctx);
      od = ctx->stage_out;
    }
    ctx->engine->hvp(vd, od, eps);
    if (!odev) {
      SLQ_CUDA(cudaMemcpyAsync(out, od, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      SLQ_CUDA(cudaStreamSynchronize(ctx->stream));
    }
  });
}

slq_status slq_diag_watchdog(slq_ctx* ctx, int32_t stall_ms, double timeout_s) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  if (stall_ms < 0 || stall_ms > 10000) return fail(ctx, SLQ_EINVAL, "stall_ms must be in [0, 10000]");
  return guarded(ctx, [&] {
    check_device(ctx);
    diag_stall(ctx->stream, stall_ms);
    watchdog_wait(ctx->stream, ctx->comm.get(), timeout_s);
  });
}

slq_status slq_grad(slq_ctx* ctx, float* g, double* loss) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    check_device(ctx);
    const size_t bytes = sizeof(float) * (size_t)ctx->plan.P_loc;
    const bool gdev = g ? is_device_ptr(g) : true;
    float* gd = g;
    if (g && !gdev) {
      ensure_stage(ctx);
      gd = ctx->stage_out;
    }
    const double l = ctx->engine->grad(gd);
    if (g && !gdev) {
      SLQ_CUDA(cudaMemcpyAsync(g, gd, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      SLQ_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (loss) *loss = l;
  });
}

slq_status slq_lanczos(slq_ctx* ctx, uint64_t seed, int32_t m, double* alpha, double* beta) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    SLQ_CHECK_ARG(alpha != nullptr && (m == 1 || beta != nullptr), "alpha / beta");
    check_device(ctx);
    std::vector<double> b(std::max(m - 1, 1));
    ctx->engine->lanczos(seed, m, alpha, b.data());
    for (int i = 0; i + 1 < m; ++i) beta[i] = b[i];
  });
}

slq_status slq_lanczos_start(slq_ctx* ctx, uint64_t seed, int32_t m) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    check_device(ctx);
    ctx->engine->start(seed, m);
  });
}

slq_status slq_lanczos_step(slq_ctx* ctx, int32_t n_steps) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    check_device(ctx);
    ctx->engine->step(n_steps);
  });
}

slq_status slq_lanczos_result(slq_ctx* ctx, double* alpha, double* beta) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    SLQ_CHECK_ARG(alpha != nullptr && beta != nullptr, "alpha / beta");
    check_device(ctx);
    ctx->engine->result(alpha, beta);
  });
}

slq_status slq_slq(slq_ctx* ctx, const uint64_t* seeds, int32_t n_probes, int32_t m, double* alpha, double* beta,
                   int32_t* m_done) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    SLQ_CHECK_ARG(seeds && n_probes >= 1 && m >= 1 && alpha && (m == 1 || beta), "seeds / n_probes / m / outputs");
    check_device(ctx);
    std::vector<double> b(std::max(m - 1, 1));
    for (int p = 0; p < n_probes; ++p) {
      ctx->engine->lanczos(seeds[p], m, alpha + (int64_t)p * m, b.data());
      for (int i = 0; i + 1 < m; ++i) beta[(int64_t)p * (m - 1) + i] = b[i];
      if (m_done) m_done[p] = ctx->engine->last_info.m_done;
    }
  });
}

slq_status slq_nonfinite_seq(const slq_ctx* ctx, int32_t* seq) {
  if (!ctx || !seq) return fail(nullptr, SLQ_EINVAL, "ctx / seq");
  *seq = ctx->engine->nonfinite_seq;
  return SLQ_OK;
}

slq_status slq_lanczos_info(const slq_ctx* ctx, int32_t* m_done, double* beta_next, int32_t* nonfinite) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  const LanczosInfo& i = ctx->engine->last_info;
  if (m_done) *m_done = i.m_done;
  if (beta_next) *beta_next = i.beta_next;
  if (nonfinite) *nonfinite = i.nonfinite;
  return SLQ_OK;
}

slq_status slq_quadrature(const double* alpha, const double* beta, int32_t m, double* nodes, double* weights) {
  return guarded(nullptr, [&] { tridiag_gauss(alpha, beta, m, nodes, weights); });
}

slq_status slq_density(const double* nodes, const double* weights, const int32_t* m_counts, int32_t n_probes,
                       int32_t jmax, double* moments, const double* grid, int32_t n_grid, double sigma,
                       double* density) {
  return guarded(nullptr, [&] {
    slq_average(nodes, weights, m_counts, n_probes, jmax, moments, grid, n_grid, sigma, density);
  });
}

slq_status slq_ghost_clusters(const double* nodes, int32_t m, double tol, int32_t* cluster_id, int32_t* n_ghost,
                              double* max_split) {
  return guarded(nullptr, [&] { ghost_clusters(nodes, m, tol, cluster_id, n_ghost, max_split); });
}

slq_status slq_probe(slq_ctx* ctx, uint64_t seed, float* q) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    SLQ_CHECK_ARG(q != nullptr, "q");
    check_device(ctx);
    if (is_device_ptr(q)) {
      ctx->engine->probe(seed, q);
    } else {
      ensure_stage(ctx);
      ctx->engine->probe(seed, ctx->stage_out);
      SLQ_CUDA(cudaMemcpy(q, ctx->stage_out, sizeof(float) * (size_t)ctx->plan.P_loc, cudaMemcpyDeviceToHost));
    }
  });
}

slq_status slq_cg(slq_ctx* ctx, const float* b, float* x, double damping, int32_t max_iter, double tol,
                  int32_t* iters, double* rel_residual) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    SLQ_CHECK_ARG(b && x && b != x, "b / x (non-aliasing)");
    SLQ_CHECK_ARG(max_iter >= 1 && damping >= 0 && tol >= 0, "max_iter >= 1, damping >= 0, tol >= 0");
    check_device(ctx);
    const size_t bytes = sizeof(float) * (size_t)ctx->plan.P_loc;
    const bool bdev = is_device_ptr(b), xdev = is_device_ptr(x);
    ensure_stage(ctx);
    const float* bd = b;
    float* xd = x;
    if (!bdev) {
      SLQ_CUDA(cudaMemcpyAsync(ctx->stage_in, b, bytes, cudaMemcpyHostToDevice, ctx->stream));
      bd = ctx->stage_in;
    }
    if (!xdev) xd = ctx->stage_out;
    double rr = 0;
    const int it = ctx->engine->cg(bd, xd, damping, max_iter, tol, &rr);
    if (!xdev) {
      SLQ_CUDA(cudaMemcpyAsync(x, xd, bytes, cudaMemcpyDeviceToHost, ctx->stream));
      SLQ_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    if (iters) *iters = it;
    if (rel_residual) *rel_residual = rr;
  });
}

slq_status slq_blockdiag(slq_ctx* ctx, uint64_t probe_seed, double* rel_err, double* cosine) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    SLQ_CHECK_ARG(rel_err && cosine, "rel_err / cosine");
    check_device(ctx);
    ctx->engine->blockdiag(probe_seed, rel_err, cosine);
  });
}

slq_status slq_profile(slq_ctx* ctx, int32_t enable, int32_t reset) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  return guarded(ctx, [&] {
    SLQ_CHECK_ARG(enable >= 0 && enable <= 2, "enable: 0 off, 1 serial, 2 overlap-aware");
    if (reset) {
      check_device(ctx);
      ctx->prof.reset(ctx->stream);
    }
    ctx->prof.on = enable != 0;
    if (enable) ctx->prof.mode = enable;
  });
}

slq_status slq_kernel_busy(const slq_ctx* ctx, int32_t cls, double* busy_ms) {
  if (!ctx || cls < -1 || cls >= KC_COUNT || !busy_ms) return fail(nullptr, SLQ_EINVAL, "ctx / class / busy_ms");
  *busy_ms = const_cast<slq_ctx*>(ctx)->prof.busy(cls);
  return SLQ_OK;
}

int32_t slq_num_kernel_classes(void) { return KC_COUNT; }
const char* slq_kernel_class_name(int32_t c) { return kernel_class_name(c); }

slq_status slq_kernel_stats(const slq_ctx* ctx, int32_t cls, double* ms, int64_t* launches, double* flops,
                            double* bytes) {
  if (!ctx || cls < 0 || cls >= KC_COUNT) return fail(nullptr, SLQ_EINVAL, "ctx / class");
  slq_ctx* c = const_cast<slq_ctx*>(ctx);
  c->prof.flush();
  if (ms) *ms = c->prof.ms[cls];
  if (launches) *launches = c->prof.count[cls];
  if (flops) *flops = c->prof.flops[cls];
  if (bytes) *bytes = c->prof.bytes[cls];
  return SLQ_OK;
}

int64_t slq_launch_count(const slq_ctx* ctx) { return ctx ? ctx->launches : -1; }
void* slq_stream(const slq_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

slq_status slq_collective_counts(const slq_ctx* ctx, int64_t* ag, int64_t* rs, int64_t* ar) {
  if (!ctx) return fail(nullptr, SLQ_EINVAL, "ctx");
  CommCounts c;
  if (ctx->comm) c = ctx->comm->total_counts();
  if (ag) *ag = c.allgather;
  if (rs) *rs = c.reduce_scatter;
  if (ar) *ar = c.allreduce;
  return SLQ_OK;
}

}  // extern "C"
