// FD-HVP (Eq. (1), Alg. 1) and Lanczos (§4, App. C) orchestration on device-resident shards.
//
// Per HVP (done out of place):  theta+- = fmaf(+-eta, v, theta)  ->  pass(theta+) ->
// g+ ; pass(theta-) -> g- ; out = (g+ - g-)/(2 eta).  theta is never written.
// Per Lanczos step (P:307-311 in A(2,7) order; reading SURVEY §8(c2) #2, #5):
//   w = H q_k - beta_k q_{k-1};  alpha_k = <w, q_k>;  w -= alpha_k q_k;
//   [full: CGS over q_1..q_k, twice];  beta_{k+1} = ||w||;  q_{k+1} = w / beta_{k+1}
// All dot products are fp64 partials reduced in a fixed order, then (R > 1) one small fp64
// all-reduce.  Vectors are fp32 shards in the FSDP layout.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "engine.h"
#include "paired.h"

namespace slq {

namespace {

template <class T>
struct LocalIO : PassIO<T> {
  const LayoutPlan* plan;
  const T* shard = nullptr;
  T* gshard = nullptr;
  const T* params(int u) override { return shard + plan->units[u].local_offset; }
  T* grads(int u) override { return gshard + plan->units[u].local_offset; }
  void grads_done(int) override {}
};

// ZeRO-3: gather a unit's parameters before its forward and again before its backward; reduce-
// scatter its gradient after its backward.  Every NCCL call of a pass is issued on
// ONE communication stream (so all ranks execute them in the same order), linked to the compute
// stream by events: the runner's prefetch(u) hint starts unit u's all-gather into the free buffer
// of a ping-pong pair while the current unit computes; grads_done(u) reduce-scatters from one of
// two gradient buffers while the next unit's backward fills the other.  Unit 0 (embedding) has its
// own parameter and gradient buffers so it can stay live with any other unit (tied head).
template <class T>
struct FsdpIO : PassIO<T> {
  const LayoutPlan* plan;
  Comm* comm;
  cudaStream_t s = nullptr;   // compute stream
  cudaStream_t cs = nullptr;  // communication stream
  const T* shard = nullptr;
  T* gshard = nullptr;
  T *pbuf0, *gbuf0;
  T *pb[2], *gb[2];
  int holder[2] = {-1, -1};  // unit whose gather was issued into pb[i]
  int cur = -1;              // pb index of the unit returned last
  int gcur = 0;              // gb index for the next grads(u >= 1)
  bool gather0 = false;      // unit 0 gather issued and not yet consumed
  cudaEvent_t ev_main = nullptr, ev_ready[3] = {}, ev_gfree[3] = {}, ev_comm = nullptr;
  bool gpending[3] = {false, false, false};
  CommType ct() const { return sizeof(T) == 8 ? COMM_F64 : COMM_F32; }
  void init() {
    SLQ_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    SLQ_CUDA(cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming));
    SLQ_CUDA(cudaEventCreateWithFlags(&ev_comm, cudaEventDisableTiming));
    for (int i = 0; i < 3; ++i) {
      SLQ_CUDA(cudaEventCreateWithFlags(&ev_ready[i], cudaEventDisableTiming));
      SLQ_CUDA(cudaEventCreateWithFlags(&ev_gfree[i], cudaEventDisableTiming));
    }
  }
  ~FsdpIO() {
    if (cs) cudaStreamSynchronize(cs);
    if (ev_main) cudaEventDestroy(ev_main);
    if (ev_comm) cudaEventDestroy(ev_comm);
    for (int i = 0; i < 3; ++i) {
      if (ev_ready[i]) cudaEventDestroy(ev_ready[i]);
      if (ev_gfree[i]) cudaEventDestroy(ev_gfree[i]);
    }
    if (cs) cudaStreamDestroy(cs);
  }
  void begin_pass() {
    holder[0] = holder[1] = -1;
    cur = -1;
    gather0 = false;
  }
  // the comm stream waits for everything issued so far on the compute stream
  void comm_after_main() {
    SLQ_CUDA(cudaEventRecord(ev_main, s));
    SLQ_CUDA(cudaStreamWaitEvent(cs, ev_main, 0));
  }
  void gather(int u, T* dst, cudaEvent_t done) {
    const UnitPlan& up = plan->units[u];
    comm_after_main();  // dst's previous contents are no longer read
    comm->allgather(shard + up.local_offset, dst, (size_t)up.chunk, ct(), cs);
    SLQ_CUDA(cudaEventRecord(done, cs));
  }
  void prefetch(int u) override {
    if (u < 0 || u >= (int)plan->units.size()) return;
    if (u == 0) {
      if (!gather0) gather(0, pbuf0, ev_ready[2]);
      gather0 = true;
      return;
    }
    if (holder[0] == u || holder[1] == u) return;
    const int i = cur == 0 ? 1 : 0;  // never the buffer of the unit in use
    holder[i] = u;
    gather(u, pb[i], ev_ready[i]);
  }
  const T* params(int u) override {
    if (u == 0) {
      prefetch(0);
      gather0 = false;
      SLQ_CUDA(cudaStreamWaitEvent(s, ev_ready[2], 0));
      return pbuf0;
    }
    prefetch(u);
    const int i = holder[0] == u ? 0 : 1;
    SLQ_CUDA(cudaStreamWaitEvent(s, ev_ready[i], 0));
    cur = i;
    return pb[i];
  }
  T* grads(int u) override {
    const int i = u == 0 ? 2 : gcur;
    if (gpending[i]) SLQ_CUDA(cudaStreamWaitEvent(s, ev_gfree[i], 0));  // its reduce-scatter has read it
    gpending[i] = false;
    return u == 0 ? gbuf0 : gb[i];
  }
  bool collective() const override { return true; }
  void grads_done(int u) override {
    const UnitPlan& up = plan->units[u];
    const int i = u == 0 ? 2 : gcur;
    T* g = u == 0 ? gbuf0 : gb[i];
    comm_after_main();
    if (up.padded > up.numel)
      SLQ_CUDA(cudaMemsetAsync(g + up.numel, 0, sizeof(T) * (size_t)(up.padded - up.numel), cs));
    comm->reduce_scatter(g, gshard + up.local_offset, (size_t)up.chunk, ct(), cs);
    SLQ_CUDA(cudaEventRecord(ev_gfree[i], cs));
    gpending[i] = true;
    if (u != 0) gcur ^= 1;
  }
  // the compute stream waits for every collective of the pass (the reduce-scattered gradient)
  void end_pass() {
    SLQ_CUDA(cudaEventRecord(ev_comm, cs));
    SLQ_CUDA(cudaStreamWaitEvent(s, ev_comm, 0));
    gpending[0] = gpending[1] = gpending[2] = false;  // every buffer's reduce-scatter is behind us
  }
};

// One gradient-pass executor: a runner (its own activation buffers) bound to a stream.  After a
// first eager run (which sizes every workspace) the ~400 launches of a pass are captured once per
// (theta, grad) buffer pair into a CUDA graph and replayed; profiling runs stay eager because the
// per-class profiler records events around individual launches.
template <class T>
struct PassExec {
  Launch L;
  Workspace own_ws;
  cudaStream_t own_stream = nullptr;
  std::unique_ptr<Runner<T>> runner;
  LocalIO<T> lio;
  FsdpIO<T>* fio = nullptr;
  FsdpIO<T>* fio2 = nullptr;  // paired evaluation with FSDP: the half-difference (thetatil, gtil)
  struct Graph {
    const void* th;
    void* g;
    cudaGraphExec_t exec;
    int64_t launches;
    int eager_runs;
  };
  std::vector<Graph> graphs;
  bool use_graphs = getenv("SLQ_NO_GRAPHS") == nullptr;

  LocalIO<T> lio2;  // paired evaluation: (thetatil, gtil)

  PassExec(const slq_model_desc& d, const LayoutPlan& plan, const HostBatch& b, const Launch& base, bool own,
           bool paired = false) {
    L = base;
    if (own) {
      SLQ_CUDA(cudaStreamCreateWithFlags(&own_stream, cudaStreamNonBlocking));
      L.stream = own_stream;
      L.ws = &own_ws;
    }
    if constexpr (sizeof(T) == 4) {
      if (paired) {
        runner = make_paired_runner(d, plan, b, L);
        if (!runner) throw Error(SLQ_EUNSUPPORTED, "paired evaluation is implemented for the GPT arch only");
      }
    }
    if (!runner) runner = make_runner<T>(d, plan, b, L);
    lio.plan = &plan;
    lio2.plan = &plan;
  }
  // FSDP: this executor's collectives go through f (host-synchronous loopback collectives cannot
  // be captured, so such a pass stays eager)
  void attach(FsdpIO<T>* f, FsdpIO<T>* f2 = nullptr) {
    fio = f;
    fio2 = f2;
    if (f->comm->host_sync()) use_graphs = false;
  }
  ~PassExec() {
    if (L.stream) cudaStreamSynchronize(L.stream);
    for (auto& x : graphs)
      if (x.exec) cudaGraphExecDestroy(x.exec);
    runner.reset();
    if (own_stream) cudaStreamDestroy(own_stream);
  }

  void eager(const T* th, T* g, double* loss_dev) {
    if (runner->paired()) {
      if (fio) {
        fio->shard = th;
        fio->gshard = g;
        fio2->shard = lio2.shard;
        fio2->gshard = lio2.gshard;
        fio->begin_pass();
        fio2->begin_pass();
        runner->fwd_bwd_pair(*fio, *fio2, loss_dev);
        fio->end_pass();
        fio2->end_pass();
        return;
      }
      lio.shard = th;
      lio.gshard = g;
      runner->fwd_bwd_pair(lio, lio2, loss_dev);
      return;
    }
    if (fio) {
      fio->shard = th;
      fio->gshard = g;
      fio->begin_pass();
      runner->fwd_bwd(*fio, loss_dev);
      fio->end_pass();
    } else {
      lio.shard = th;
      lio.gshard = g;
      runner->fwd_bwd(lio, loss_dev);
    }
  }

  // paired: (th, g) = (theta, gbar) and (th2, g2) = (thetatil, gtil)
  void run_pair(const T* th, T* g, const T* th2, T* g2, double* loss_dev) {
    lio2.shard = th2;
    lio2.gshard = g2;
    run(th, g, loss_dev);
  }

  void run(const T* th, T* g, double* loss_dev) {
    if (!use_graphs || prof_enabled(L.prof)) {
      eager(th, g, loss_dev);
      return;
    }
    Graph* pg = nullptr;
    for (auto& x : graphs)
      if (x.th == th && x.g == g) pg = &x;
    if (!pg) {
      graphs.push_back(Graph{th, g, nullptr, 0, 0});
      pg = &graphs.back();
    }
    if (pg->exec) {
      SLQ_CUDA(cudaGraphLaunch(pg->exec, L.stream));
      *L.launches += pg->launches;
      return;
    }
    if (pg->eager_runs++ == 0) {
      eager(th, g, loss_dev);
      return;
    }
    const int64_t l0 = *L.launches;
    cudaGraph_t graph = nullptr;
    SLQ_CUDA(cudaStreamBeginCapture(L.stream, cudaStreamCaptureModeThreadLocal));
    try {
      eager(th, g, loss_dev);
    } catch (...) {
      cudaStreamEndCapture(L.stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    SLQ_CUDA(cudaStreamEndCapture(L.stream, &graph));
    SLQ_CUDA(cudaGraphInstantiate(&pg->exec, graph, 0));
    SLQ_CUDA(cudaGraphDestroy(graph));
    pg->launches = *L.launches - l0;
    SLQ_CUDA(cudaGraphLaunch(pg->exec, L.stream));
  }
};

template <class T>
struct EngineT : Engine {
  slq_model_desc d;
  const LayoutPlan& plan;
  Launch L;
  Comm* comm;
  int rank;
  int64_t n;  // P_loc
  std::vector<void*> allocs;
  float* theta;
  T *thp, *thm, *gp, *gm;
  // Krylov basis (reorth FULL: max_steps + 1 rows; WINDOW: a ring of r rows, q_j in row j % r):
  // fp32 rows, or bf16 rows plus two fp32 working copies of q_k, q_{k-1} (qf[k % 2])
  float *basis = nullptr, *w = nullptr, *vq[3] = {nullptr, nullptr, nullptr};
  __nv_bfloat16* basis16 = nullptr;
  float* qf[2] = {nullptr, nullptr};
  double* dscal;      // [0] sumsq, [1] beta_k, [2] loss, [3..] alpha / reorth coefficients
  double* gram = nullptr;  // Gram matrix of the stored basis rows (two-pass CGS2), ldg x ldg
  int ldg = 0;
  bool cgs3 = getenv("SLQ_CGS_3PASS") != nullptr;  // the explicit three-pass CGS2 (diagnostic)
  double* partials;
  int* dflag;
  UnitDev* units_dev;
  int max_steps;
  // pe[0] runs on the context stream; a second executor on its own stream evaluates the theta-
  // pass concurrently with the theta+ pass (the two gradient evaluations of Eq. (1) are independent
  // until the FD difference).  With FSDP each executor has its own FsdpIO (ping-pong buffers) and
  // its own communicator split from the context's, so the two passes' collectives never have to
  // be ordered against each other; the context communicator carries the scalar all-reduces.
  FsdpIO<T> fio[2];
  std::unique_ptr<PassExec<T>> pe[2];
  bool dual = false;
  // paired evaluation (SLQ_PASS_PAIRED*): thm holds thetatil = eta v, gp gets gbar, gm gets gtil;
  // the FD kernels then read gtil alone with scale 1/eta
  bool paired_ = false;
  const T* fd_a() const { return paired_ ? gm : gp; }
  const T* fd_b() const { return paired_ ? nullptr : gm; }
  double fd_scale(double inv2eta) const { return paired_ ? 2.0 * inv2eta : inv2eta; }
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  double* hstage;  // pinned host scalars

  template <class U>
  U* dalloc(int64_t cnt) {
    void* p = nullptr;
    SLQ_CUDA(cudaMalloc(&p, sizeof(U) * (size_t)std::max<int64_t>(cnt, 1)));
    allocs.push_back(p);
    return (U*)p;
  }

  EngineT(const slq_model_desc& d_, const LayoutPlan& plan_, const HostBatch& b, const float* theta_host, int rank_,
          Comm* comm_, const Launch& L_)
      : d(d_), plan(plan_), L(L_), comm(comm_), rank(rank_) {
    n = plan.P_loc;
    max_steps = d.max_steps;
    theta = dalloc<float>(n);
    {  // this rank's chunk of every unit; padding zero
      std::vector<float> h((size_t)n, 0.0f);
      for (const UnitPlan& u : plan.units) {
        const int64_t start = (int64_t)rank * u.chunk;
        for (int64_t j = 0; j < u.chunk; ++j) {
          const int64_t p = start + j;
          if (p < u.numel) h[(size_t)(u.local_offset + j)] = theta_host[u.global_offset + p];
        }
      }
      SLQ_CUDA(cudaMemcpy(theta, h.data(), sizeof(float) * (size_t)n, cudaMemcpyHostToDevice));
    }
    thp = dalloc<T>(n); thm = dalloc<T>(n); gp = dalloc<T>(n); gm = dalloc<T>(n);
    SLQ_CUDA(cudaMemset(gp, 0, sizeof(T) * (size_t)n));
    SLQ_CUDA(cudaMemset(gm, 0, sizeof(T) * (size_t)n));
    w = dalloc<float>(n);
    if (d.reorth == SLQ_REORTH_FULL || d.reorth == SLQ_REORTH_WINDOW) {
      const int64_t rows = d.reorth == SLQ_REORTH_FULL ? max_steps + 1 : d.reorth_window;
      if (d.basis_dtype == SLQ_BASIS_BF16) {
        basis16 = dalloc<__nv_bfloat16>(rows * n);
        qf[0] = dalloc<float>(n);
        qf[1] = dalloc<float>(n);
      } else {
        basis = dalloc<float>(rows * n);
      }
    } else {
      for (int i = 0; i < 3; ++i) vq[i] = dalloc<float>(n);
    }
    dscal = dalloc<double>(8 + 5 * (int64_t)(max_steps + 1));
    const int64_t np = std::max<int64_t>(vec_nblocks(n), (int64_t)reorth_nblocks(n) * 2 * (max_steps + 1));
    if (d.reorth != SLQ_REORTH_NONE) {
      ldg = d.reorth == SLQ_REORTH_FULL ? max_steps + 1 : d.reorth_window;
      gram = dalloc<double>((int64_t)ldg * ldg);
    }
    partials = dalloc<double>(np);
    dflag = dalloc<int>(1);
    {
      std::vector<UnitDev> ud;
      for (const UnitPlan& u : plan.units)
        ud.push_back(UnitDev{u.local_offset, u.chunk, u.global_offset, u.numel, (int64_t)rank * u.chunk});
      units_dev = dalloc<UnitDev>((int64_t)ud.size());
      SLQ_CUDA(cudaMemcpy(units_dev, ud.data(), sizeof(UnitDev) * ud.size(), cudaMemcpyHostToDevice));
    }
    SLQ_CUDA(cudaMallocHost(&hstage, (64 + 2 * (size_t)(max_steps + 1)) * sizeof(double)));
    paired_ = d.pass_numerics == SLQ_PASS_PAIRED || d.pass_numerics == SLQ_PASS_PAIRED_FP32;
    // one pass evaluates both points in the paired modes: nothing to run concurrently
    dual = !paired_ && getenv("SLQ_SERIAL_PASSES") == nullptr;
    const int nexec = dual ? 2 : 1;
    auto make_fio = [&](FsdpIO<T>& f, int color, cudaStream_t s) {
      f.plan = &plan;
      f.comm = comm->split(color);
      f.s = s;
      int64_t mx = 0;
      for (const UnitPlan& u : plan.units) mx = std::max(mx, u.padded);
      f.pbuf0 = dalloc<T>(plan.units[0].padded);
      f.gbuf0 = dalloc<T>(plan.units[0].padded);
      for (int k = 0; k < 2; ++k) {
        f.pb[k] = dalloc<T>(mx);
        f.gb[k] = dalloc<T>(mx);
      }
      f.init();
    };
    for (int i = 0; i < nexec; ++i) {
      pe[i].reset(new PassExec<T>(d, plan, b, L, i > 0, paired_));
      if (!comm) continue;
      // paired: one executor, two FSDP streams of collectives -- the mean (theta, gbar) and the
      // half-difference (thetatil = eta v, gtil), each with its own buffers and communicator
      make_fio(fio[i], i, pe[i]->L.stream);
      if (paired_) make_fio(fio[1], 1, pe[i]->L.stream);
      pe[i]->attach(&fio[i], paired_ ? &fio[1] : nullptr);
    }
    if (dual) {
      SLQ_CUDA(cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming));
      SLQ_CUDA(cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming));
    }
    SLQ_CUDA(cudaDeviceSynchronize());
  }
  ~EngineT() override {
    cudaStreamSynchronize(L.stream);
    pe[1].reset();
    pe[0].reset();
    if (ev_a) cudaEventDestroy(ev_a);
    if (ev_b) cudaEventDestroy(ev_b);
    for (void* p : allocs) cudaFree(p);
    if (hstage) cudaFreeHost(hstage);
  }

  // g+ = grad L(theta+), g- = grad L(theta-): concurrently on two streams when dual
  void two_passes() {
    if (paired_) {
      pe[0]->run_pair(reinterpret_cast<const T*>(theta), gp, thm, gm, dscal + 2);
      return;
    }
    if (!dual || prof_serial(L.prof)) {  // serial profile: per-launch durations stay honest
      pe[0]->run(thp, gp, dscal + 2);
      pe[0]->run(thm, gm, dscal + 3);
      return;
    }
    SLQ_CUDA(cudaEventRecord(ev_a, L.stream));
    SLQ_CUDA(cudaStreamWaitEvent(pe[1]->L.stream, ev_a, 0));
    pe[0]->run(thp, gp, dscal + 2);
    pe[1]->run(thm, gm, dscal + 3);
    SLQ_CUDA(cudaEventRecord(ev_b, pe[1]->L.stream));
    SLQ_CUDA(cudaStreamWaitEvent(L.stream, ev_b, 0));
  }

  double pass_flops() const override { return pe[0]->runner->flops_per_pass(); }

  // fixed-order reduction of `k` partial columns into out (device), then all-reduce
  void finish_reduce(int nb, int k, double* out) {
    reduce_partials(L, partials, nb, k, out);
    if (comm) comm->allreduce_sum_f64(out, (size_t)k, L.stream);
  }

  // host copy of `cnt` device doubles (synchronises the stream)
  // every host wait of the engine: with a communicator, through the collective watchdog
  // (asynchronous NCCL errors -> SLQ_ENCCL, no progress within SLQ_TIMEOUT_S -> SLQ_ETIMEOUT)
  void sync() {
    if (comm) watchdog_wait(L.stream, comm, watchdog_timeout_s());
    else SLQ_CUDA(cudaStreamSynchronize(L.stream));
  }
  void to_host(const double* dev, int cnt, double* host) {
    SLQ_CUDA(cudaMemcpyAsync(hstage, dev, sizeof(double) * cnt, cudaMemcpyDeviceToHost, L.stream));
    sync();
    memcpy(host, hstage, sizeof(double) * cnt);
  }

  // theta+- = theta +- eta v into thp / thm (reading R9); returns 1 / (2 eta_used)
  double form_points(const float* v, double eta) {
    if constexpr (sizeof(T) == 4) {
      if (paired_) {  // thetabar = theta (read in place), thetatil = eta v
        SLQ_CHECK_ARG(eta > 0 && std::isfinite(eta), "eps / ||v|| must be finite and > 0");
        pair_scale(L, v, eta, thm, n);
        return 1.0 / (2.0 * eta);
      }
    }
    if constexpr (sizeof(T) == 8) {
      if (d.perturb == SLQ_PERTURB_EXACT) {
        SLQ_CHECK_ARG(eta > 0 && std::isfinite(eta), "eps / ||v|| must be finite and > 0");
        perturb_exact(L, theta, v, eta, thp, thm, n);
        return 1.0 / (2.0 * eta);
      }
    }
    const float ef = (float)eta;
    SLQ_CHECK_ARG(ef > 0.0f && std::isfinite(ef), "eps / ||v|| not representable in fp32");
    perturb<T>(L, theta, v, ef, thp, thm, n);
    return 1.0 / (2.0 * (double)ef);
  }

  void hvp(const float* v, float* out, double eps) override {
    nonfinite_seq = -1;
    sumsq_partials(L, v, n, partials);
    finish_reduce(vec_nblocks(n), 1, dscal + 0);
    double ss;
    to_host(dscal, 1, &ss);
    if (!std::isfinite(ss)) throw Error(SLQ_ENUMERIC, "non-finite direction v");
    if (ss == 0.0) {
      SLQ_CUDA(cudaMemsetAsync(out, 0, sizeof(float) * (size_t)n, L.stream));
      sync();
      return;
    }
    const double inv2eta = form_points(v, eps / sqrt(ss));
    two_passes();
    SLQ_CUDA(cudaMemsetAsync(dflag, 0, sizeof(int), L.stream));
    fd_out<T>(L, fd_a(), fd_b(), fd_scale(inv2eta), out, n, dflag);
    int flag = 0;
    SLQ_CUDA(cudaMemcpyAsync(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost, L.stream));
    sync();
    if (flag) {
      for (auto& x : pe) {
        if (!x) continue;
        const int q = x->runner->first_nonfinite_seq();
        if (q >= 0 && (nonfinite_seq < 0 || q < nonfinite_seq)) nonfinite_seq = q;
      }
      throw Error(SLQ_ENUMERIC, "non-finite gradient in the FD-HVP" +
                                    (nonfinite_seq >= 0 ? " (local sequence " + std::to_string(nonfinite_seq) +
                                                              " has a non-finite loss)"
                                                        : std::string(" (all losses finite)")));
    }
  }

  double grad(float* g) override {
    if (paired_) {  // thetatil = 0: gbar is the gradient at theta
      SLQ_CUDA(cudaMemsetAsync(thm, 0, sizeof(T) * (size_t)n, L.stream));
      pe[0]->run_pair(reinterpret_cast<const T*>(theta), gp, thm, gm, dscal + 2);
    } else {
      convert_f32<T>(L, theta, thp, n);
      pe[0]->run(thp, gp, dscal + 2);
    }
    if (comm) comm->allreduce_sum_f64(dscal + 2, 1, L.stream);
    if (g) to_f32<T>(L, gp, g, n);
    double loss;
    to_host(dscal + 2, 1, &loss);
    return loss / pe[0]->runner->tokens_global();
  }

  // ---- vector helpers for the solvers built on the HVP primitive ----
  std::vector<float*> extra;  // lazily allocated P_loc vectors
  float* vec(int i) {
    while ((int)extra.size() <= i) extra.push_back(dalloc<float>(n));
    return extra[i];
  }
  double dot(const float* a, const float* b) {
    dot_partials(L, a, b, n, partials);
    finish_reduce(vec_nblocks(n), 1, dscal + 5);
    double h;
    to_host(dscal + 5, 1, &h);
    return h;
  }

  // Hestenes-Stiefel CG on (H + damping I) x = b, x_0 = 0; every H p is one FD-HVP (P:445, P:1164:
  // "repeated HVP calls plus scalar reductions and shard-local vector operations")
  int cg(const float* b, float* x, double damping, int max_iter, double tol, double* relres) override {
    float *r = vec(0), *p = vec(1), *ap = vec(2);
    SLQ_CUDA(cudaMemsetAsync(x, 0, sizeof(float) * (size_t)n, L.stream));
    SLQ_CUDA(cudaMemcpyAsync(r, b, sizeof(float) * (size_t)n, cudaMemcpyDeviceToDevice, L.stream));
    SLQ_CUDA(cudaMemcpyAsync(p, b, sizeof(float) * (size_t)n, cudaMemcpyDeviceToDevice, L.stream));
    double rr = dot(r, r);
    const double nb = sqrt(rr);
    *relres = nb > 0 ? 1.0 : 0.0;
    if (nb == 0) return 0;
    int it = 0;
    for (it = 1; it <= max_iter; ++it) {
      hvp(p, ap, d.eps_default);
      axpby(L, ap, p, damping, 1.0, n);
      const double pap = dot(p, ap);
      if (!(pap > 0)) throw Error(SLQ_ENUMERIC, "CG: p^T (H + damping I) p <= 0 (raise damping)");
      const double a = rr / pap;
      axpby(L, x, p, a, 1.0, n);
      axpby(L, r, ap, -a, 1.0, n);
      const double rr_new = dot(r, r);
      *relres = sqrt(rr_new) / nb;
      if (!std::isfinite(rr_new)) throw Error(SLQ_ENUMERIC, "CG: non-finite residual");
      if (*relres <= tol) break;
      axpby(L, p, r, 1.0, rr_new / rr, n);
      rr = rr_new;
    }
    sync();
    return std::min(it, max_iter);
  }

  // h_full = H v; per block b: h_b = H v^(b); compare restrictions to block b.  Blocks
  // are the FSDP units (each rank compares its chunk of every unit; partials are all-reduced).
  void blockdiag(uint64_t seed, double* rel_err, double* cosine) override {
    float *v = vec(0), *vb = vec(1), *hf = vec(2), *hb = vec(3);
    probe_fill(L, v, n, units_dev, (int)plan.units.size(), seed, 1.0 / sqrt((double)plan.P));
    hvp(v, hf, d.eps_default);
    for (size_t u = 0; u < plan.units.size(); ++u) {
      const UnitPlan& up = plan.units[u];
      const int64_t lo = up.local_offset, hi = up.local_offset + up.chunk;
      mask_range(L, v, vb, lo, hi, n);
      hvp(vb, hb, d.eps_default);
      const int nb = cmp4_partials(L, hf, hb, lo, hi, partials);
      finish_reduce(nb, 4, dscal + 4);  // dscal[4..7]
      double s[4];
      to_host(dscal + 4, 4, s);
      rel_err[u] = s[1] > 0 ? sqrt(s[0] / s[1]) : 0.0;
      cosine[u] = (s[1] > 0 && s[3] > 0) ? s[2] / sqrt(s[1] * s[3]) : 0.0;
    }
  }

  void probe(uint64_t seed, float* q) override {
    probe_fill(L, q, n, units_dev, (int)plan.units.size(), seed, 1.0 / sqrt((double)plan.P));
    sync();
  }

  // ---- resumable Lanczos: start(seed, m) / step(n) / result(...) (slq_lanczos_start / _step /
  // _result; slq_lanczos = all three).  State between calls: the step counter, the basis rows or
  // rotating vectors, the device recurrence scalars and (no-basis mode) the host-side alpha / beta.
  struct Probe {
    bool active = false;
    uint64_t seed = 0;
    int m = 0, k = 0;        // requested steps, steps done
    bool stopped = false;    // no-basis mode: breakdown seen on the host
    double a_prev = 0.0, b_k = 0.0, tmax = 0.0;
    std::vector<double> ha, hb;  // no-basis mode: alpha_k, beta_{k+1} as they are formed
    LanczosInfo info;
  } pr;

  void start(uint64_t seed, int m) override {
    SLQ_CHECK_ARG(m >= 1 && m <= max_steps, "1 <= m <= max_steps");
    pr = Probe();
    last_info = LanczosInfo();
    pr.active = true;
    pr.seed = seed;
    pr.m = m;
    pr.ha.assign((size_t)m, NAN);
    pr.hb.assign((size_t)m, NAN);
    const double inv_sqrt_P = 1.0 / sqrt((double)plan.P);
    if (d.reorth == SLQ_REORTH_NONE) {
      probe_fill(L, vq[0], n, units_dev, (int)plan.units.size(), seed, inv_sqrt_P);
    } else if (basis16) {  // q_1 = bf16(s / sqrt(P)): signs first, one rounding from fp64
      probe_fill(L, qf[0], n, units_dev, (int)plan.units.size(), seed, 1.0);
      store_bf16(L, qf[0], nullptr, inv_sqrt_P, basis16, qf[0], n);
    } else {
      probe_fill(L, basis, n, units_dev, (int)plan.units.size(), seed, inv_sqrt_P);
    }
  }

  void step(int nsteps) override {
    SLQ_CHECK_ARG(pr.active, "slq_lanczos_step before slq_lanczos_start");
    SLQ_CHECK_ARG(nsteps >= 0 && pr.k + nsteps <= pr.m, "steps beyond the m given to slq_lanczos_start");
    const int k1 = pr.k + nsteps;
    if (d.reorth == SLQ_REORTH_NONE) {
      for (; pr.k < k1; ++pr.k) nobasis_step(pr.k);
    } else {
      for (; pr.k < k1; ++pr.k) basis_step(pr.k);
    }
  }

  LanczosInfo result(double* alpha, double* beta) override {
    SLQ_CHECK_ARG(pr.active, "slq_lanczos_result before slq_lanczos_start");
    const int m = pr.m, mk = pr.k;
    for (int i = 0; i < m; ++i) alpha[i] = NAN;
    for (int i = 0; i + 1 < m; ++i) beta[i] = NAN;
    LanczosInfo info;
    if (d.reorth == SLQ_REORTH_NONE) {
      sync();
      info = pr.info;
      for (int k = 0; k < info.m_done; ++k) {
        alpha[k] = pr.ha[k];
        if (k + 1 < m && k + 1 < info.m_done) beta[k] = pr.hb[k];
      }
    } else {
      double* d_alpha = dscal + 8 + 3 * (max_steps + 1);
      double* d_bhist = dscal + 8 + 4 * (max_steps + 1);
      double* ha_pin = hstage + 64;
      double* hb_pin = hstage + 64 + (max_steps + 1);
      if (mk > 0) {
        SLQ_CUDA(cudaMemcpyAsync(ha_pin, d_alpha, sizeof(double) * mk, cudaMemcpyDeviceToHost, L.stream));
        SLQ_CUDA(cudaMemcpyAsync(hb_pin, d_bhist, sizeof(double) * mk, cudaMemcpyDeviceToHost, L.stream));
      }
      sync();
      // steps after a breakdown ran on a noise direction; they are discarded here
      double tmax = 0.0;
      for (int k = 0; k < mk; ++k) {
        const double a = ha_pin[k], bnext = hb_pin[k];
        if (!std::isfinite(a) || !std::isfinite(bnext)) {
          info.nonfinite = 1;
          info.m_done = k;
          last_info = info;
          pr.active = false;
          throw Error(SLQ_ENUMERIC, "non-finite Lanczos coefficient at step " + std::to_string(k + 1));
        }
        alpha[k] = a;
        if (k + 1 < m) beta[k] = bnext;
        tmax = std::max(tmax, fabs(a));
        if (k > 0) tmax = std::max(tmax, beta[k - 1]);
        info.m_done = k + 1;
        info.beta_next = bnext;
        if (k + 1 < m && bnext <= 1e-7 * tmax) {  // breakdown: invariant subspace (fp32 vectors)
          beta[k] = NAN;
          break;
        }
      }
      // the last step's beta_{k+1} is only an output if another step follows it
      if (mk < m && info.m_done == mk && mk >= 1) beta[mk - 1] = NAN;
    }
    last_info = info;
    pr.active = false;
    return info;
  }

  LanczosInfo lanczos(uint64_t seed, int m, double* alpha, double* beta) override {
    start(seed, m);
    step(m);
    return result(alpha, beta);
  }

  // Three-term recurrence without a stored basis (c5 mode; "only the essential Lanczos
  // vectors").  Per step two vector kernels and one 3-scalar reduction:
  //   perturb:  q_k = (w_raw - alpha_{k-1} q_{k-1}) / beta_k  (deferred normalisation) and theta+-
  //   passes:   g+, g-
  //   fd:       w_raw = (g+ - g-)/(2 eta) - beta_k q_{k-1};  s1 = <w_raw,q_k>, s2 = |w_raw|^2, s3 = |q_k|^2
  //   host:     alpha_k = s1;  beta_{k+1}^2 = |w_raw - alpha_k q_k|^2 = s2 - 2 alpha s1 + alpha^2 s3
  // If that Pythagorean form loses more than 3 digits to cancellation, the residual is formed
  // explicitly (one extra pass) and its norm taken directly.  After a breakdown (or a non-finite
  // coefficient) the remaining steps do nothing.
  void nobasis_step(int k) {
    if (pr.stopped) return;
    const bool exact = d.perturb == SLQ_PERTURB_EXACT && sizeof(T) == 8;
    const double eps = d.eps_default;
    const float eps_f = (float)eps;
    const double inv2eps = exact ? 1.0 / (2.0 * eps) : 1.0 / (2.0 * (double)eps_f);
    float* q[2] = {vq[0], vq[1]};  // q[k % 2] = q_k
    float* wr = vq[2];
    const int nb = vec_nblocks(n);
    float* qk = q[k % 2];
    const float* qprev = k > 0 ? q[(k + 1) % 2] : nullptr;
    if (k == 0) {
      form_points(qk, eps);
    } else {
      perturb_lanczos<T>(L, exact, theta, wr, q[(k + 1) % 2], pr.a_prev, pr.b_k, eps, qk, thp, thm, n);
    }
    two_passes();
    fd_partials3<T>(L, fd_a(), fd_b(), fd_scale(inv2eps), pr.b_k, qprev, qk, wr, n, partials);
    finish_reduce(nb, 3, dscal + 8);  // reduce_partials reads [nb x 3] row-major
    double s3[3];
    to_host(dscal + 8, 3, s3);
    const double a = s3[0];
    double b2 = s3[1] - 2.0 * a * s3[0] + a * a * s3[2];
    double a_carry = a;
    if (!(b2 > 1e-3 * s3[1])) {  // cancellation: form w = w_raw - alpha q_k explicitly
      SLQ_CUDA(cudaMemcpyAsync(dscal + 4, &a, sizeof(double), cudaMemcpyHostToDevice, L.stream));
      axpy_dev(L, wr, qk, dscal + 4, -1.0, n, partials);
      finish_reduce(nb, 1, dscal + 0);
      to_host(dscal + 0, 1, &b2);
      a_carry = 0.0;  // wr now holds the residual itself
    }
    if (!std::isfinite(a) || !std::isfinite(b2)) {
      pr.info.nonfinite = 1;
      pr.info.m_done = k;
      last_info = pr.info;
      pr.stopped = true;
      pr.active = false;
      throw Error(SLQ_ENUMERIC, "non-finite Lanczos coefficient at step " + std::to_string(k + 1));
    }
    const double bnext = sqrt(std::max(b2, 0.0));
    pr.ha[k] = a;
    pr.hb[k] = bnext;
    pr.tmax = std::max(pr.tmax, fabs(a));
    if (k > 0) pr.tmax = std::max(pr.tmax, pr.b_k);
    pr.info.m_done = k + 1;
    pr.info.beta_next = bnext;
    if (k + 1 < pr.m && bnext <= 1e-7 * pr.tmax) {
      pr.hb[k] = NAN;
      pr.stopped = true;
      return;
    }
    pr.a_prev = a_carry;
    pr.b_k = bnext;
  }

  // CGS2 over the `cnt` basis rows [0, cnt) (the window's ring holds exactly the last r vectors).
  // Two passes over the basis: (1) c1 = Q^T w together with the Gram row Q^T q_k of the newest
  // vector, (2) w -= Q (c1 + c2) fused with ||w||^2, where c2 = c1 - G c1 is the second classical
  // Gram-Schmidt pass's coefficient vector Q^T (w - Q c1) evaluated through the Gram matrix
  // G = Q^T Q (equal in exact arithmetic).  SLQ_CGS_3PASS runs the explicit passes.
  template <class B>
  void cgs2(const B* Q, int cnt, int kslot, const float* qk, double* d_coef, double* d_alpha_k) {
    const int nb = reorth_nblocks(n);
    if (cgs3) {
      reorth_dots<B>(L, Q, n, cnt, w, n, partials);
      finish_reduce(nb, cnt, d_coef);
      SLQ_CUDA(cudaMemcpyAsync(d_alpha_k, d_coef + kslot, sizeof(double), cudaMemcpyDeviceToDevice, L.stream));
      reorth_update<B>(L, Q, n, cnt, d_coef, w, n, partials, nullptr);
      finish_reduce(nb, cnt, d_coef);
      reorth_update<B>(L, Q, n, cnt, d_coef, w, n, nullptr, partials);
      finish_reduce(nb, 1, dscal + 0);
      return;
    }
    double* d_cg = d_coef + (max_steps + 1);  // [2 cnt]
    reorth_dots2<B>(L, Q, n, cnt, w, qk, n, partials);
    finish_reduce(nb, 2 * cnt, d_cg);
    gram_coef(L, d_cg, cnt, kslot, gram, ldg, d_coef, d_alpha_k);
    reorth_update<B>(L, Q, n, cnt, d_coef, w, n, nullptr, partials);
    finish_reduce(nb, 1, dscal + 0);
  }

  // step k with a stored basis (FULL / WINDOW): alpha / beta stay on the device (no host round
  // trip inside the recurrence); breakdown is detected in result()
  void basis_step(int k) {
    const bool window = d.reorth == SLQ_REORTH_WINDOW;
    const bool b16 = basis16 != nullptr;
    const int r = d.reorth_window;
    auto slot = [&](int j) { return window ? j % r : j; };
    // fp32 view of q_j: the basis row itself (fp32 basis) or the exact working copy (bf16 basis)
    auto qvec = [&](int j) -> float* { return b16 ? qf[j % 2] : basis + (int64_t)slot(j) * n; };
    double* d_beta = dscal + 1;
    double* d_coef = dscal + 8;                         // [max_steps + 1], then [2 (max_steps + 1)] dots
    double* d_alpha = dscal + 8 + 3 * (max_steps + 1);  // [max_steps + 1]
    double* d_bhist = dscal + 8 + 4 * (max_steps + 1);  // [max_steps + 1]: beta_{k+1}
    float* qk = qvec(k);
    const float* qprev = k > 0 ? qvec(k - 1) : nullptr;
    const double inv2eps = form_points(qk, d.eps_default);
    two_passes();
    fd_w<T>(L, fd_a(), fd_b(), fd_scale(inv2eps), k > 0 ? d_beta : nullptr, qprev, w, qk, n, nullptr);
    const int cnt = window ? std::min(k + 1, r) : k + 1;
    if (b16)
      cgs2<__nv_bfloat16>(basis16, cnt, slot(k), qk, d_coef, d_alpha + k);
    else
      cgs2<float>(basis, cnt, slot(k), qk, d_coef, d_alpha + k);
    // beta_{k+1} = ||w|| on the device (the next step's FD kernel reads it there)
    step_beta(L, dscal + 0, d_beta, d_bhist + k);
    if (k + 1 < pr.m) {
      if (b16)
        store_bf16(L, w, dscal + 0, 0.0, basis16 + (int64_t)slot(k + 1) * n, qf[(k + 1) % 2], n);
      else
        scale_by_inv_sqrt(L, w, dscal + 0, qvec(k + 1), n);
    }
  }
};

}  // namespace

// the pass-mode fields of a Launch (GEMM route, Ozaki settings) from the descriptor
Launch pass_launch(const slq_model_desc& d, const Launch& L) {
  Launch Lp = L;
  if (d.pass_numerics == SLQ_PASS_FP64 || d.pass_numerics == SLQ_PASS_FP64_OZ) {
    Lp.gemm_mode = d.pass_numerics == SLQ_PASS_FP64_OZ ? 2 : 0;
    // measured on B200 (c2 step, tools/exp_oz.sh): the int8 path wins on the 2e9-MNK head GEMMs and
    // breaks even below ~1e9, where the slicing launches and the fp64 epilogue dominate
    Lp.oz_min_mnk = d.oz_min_mnk > 0 ? d.oz_min_mnk : 1e9;
    // digit planes: S = 7 for the fp32 models (their fp32 alpha / beta gate needs it: S = 6 drifts
    // to 1.9e-4 by step 32 on c2), S = 5 for the bf16 models, whose gates are the bf16 ones
    // (moments <= 1e-2, extreme Ritz <= 2e-2; R27)
    // (eps < 5e-4 needs one more plane: the truncation enters the FD-HVP divided by 2 eps, and on c3
    // at eps = 1e-4 S = 5 leaves the extreme Ritz values at 1.8e-2 of the 2e-2 gate)
    Lp.oz_S = d.oz_slices > 0 ? d.oz_slices : (d.param_dtype == SLQ_PARAM_BF16 ? (d.eps_default >= 5e-4 ? 5 : 6) : 7);
    SLQ_CHECK_ARG(Lp.oz_S >= 4 && Lp.oz_S <= 7, "oz_slices must be 0 (default 7) or 4..7");
  } else {
    Lp.gemm_mode = (d.pass_numerics == SLQ_PASS_BF16X3 || d.pass_numerics == SLQ_PASS_PAIRED) ? 1
                   : d.pass_numerics == SLQ_PASS_BF16                                         ? 3
                                                                                              : 0;
  }
  return Lp;
}

std::unique_ptr<Engine> make_engine(const slq_model_desc& d, const LayoutPlan& plan, const HostBatch& b,
                                    const float* theta_host, int rank, Comm* comm, const Launch& L) {
  const Launch Lp = pass_launch(d, L);
  if (d.pass_numerics == SLQ_PASS_FP64 || d.pass_numerics == SLQ_PASS_FP64_OZ)
    return std::unique_ptr<Engine>(new EngineT<double>(d, plan, b, theta_host, rank, comm, Lp));
  return std::unique_ptr<Engine>(new EngineT<float>(d, plan, b, theta_host, rank, comm, Lp));
}

namespace {
template <class T>
void plan_runner(const slq_model_desc& d, const LayoutPlan& plan, const HostBatch& hb, const Launch& Lp,
                 int64_t* out, int nexec) {
  auto r = make_runner<T>(d, plan, hb, Lp, true);
  size_t wm = 0, wsd = 0;
  r->plan_ws(wm, wsd);
  out[SLQ_MEM_ACTIVATIONS] += nexec * (int64_t)r->arena_bytes(0);
  out[SLQ_MEM_LOGITS] += nexec * (int64_t)r->arena_bytes(1);
  out[SLQ_MEM_SCRATCH] += nexec * (int64_t)r->arena_bytes(2);
  const int64_t counters = (int64_t)(sizeof(unsigned) * Workspace::kCounters);
  out[SLQ_MEM_WORKSPACE] += nexec * ((int64_t)wm + (int64_t)wsd + 2 * counters);
}
}  // namespace

// Host-only mirror of the allocations of EngineT + its PassExecs + their runners (the runners are
// built in dry mode, so their byte counts are the real allocation code's)
void plan_memory(const slq_model_desc& d, int world, int n_local, int64_t* out) {
  SLQ_CHECK_ARG(world >= 1 && n_local >= 1, "world_size >= 1, n_local >= 1");
  for (int i = 0; i < SLQ_MEM_COUNT; ++i) out[i] = 0;
  const LayoutPlan plan = plan_layout(d, world);
  const bool f64 = d.pass_numerics == SLQ_PASS_FP64 || d.pass_numerics == SLQ_PASS_FP64_OZ;
  const bool paired = d.pass_numerics == SLQ_PASS_PAIRED || d.pass_numerics == SLQ_PASS_PAIRED_FP32;
  const int64_t esz = f64 ? 8 : 4, n = plan.P_loc, ms = d.max_steps;
  const int nexec = (paired || getenv("SLQ_SERIAL_PASSES")) ? 1 : 2;
  out[SLQ_MEM_THETA] = 4 * n;
  out[SLQ_MEM_POINTS] = 2 * esz * n;
  out[SLQ_MEM_GRADS] = 2 * esz * n;
  int64_t lz = 4 * n + 8 * (8 + 5 * (ms + 1));  // w, device scalars
  if (d.reorth == SLQ_REORTH_FULL || d.reorth == SLQ_REORTH_WINDOW) {
    const int64_t rows = d.reorth == SLQ_REORTH_FULL ? ms + 1 : d.reorth_window;
    lz += d.basis_dtype == SLQ_BASIS_BF16 ? rows * n * 2 + 2 * 4 * n : rows * n * 4;
    const int64_t ldg = d.reorth == SLQ_REORTH_FULL ? ms + 1 : d.reorth_window;
    lz += 8 * ldg * ldg;
  } else {
    lz += 3 * 4 * n;
  }
  lz += 8 * std::max<int64_t>(vec_nblocks(n), (int64_t)reorth_nblocks(n) * 2 * (ms + 1));
  out[SLQ_MEM_LANCZOS] = lz;
  if (world > 1) {
    int64_t mx = 0;
    for (const UnitPlan& u : plan.units) mx = std::max(mx, u.padded);
    out[SLQ_MEM_FSDP] = (paired ? 2 : nexec) * esz * (2 * plan.units[0].padded + 4 * mx);  // paired: mean + diff
  }
  HostBatch hb;
  if (d.arch == SLQ_ARCH_MLP) {
    hb.n_rows = n_local;
    hb.n_rows_global = n_local * world;
  } else {
    hb.n_seq = n_local;
    hb.n_seq_global = n_local * world;
  }
  const Launch Lp = pass_launch(d, Launch{nullptr, nullptr, nullptr, nullptr});
  if (f64) plan_runner<double>(d, plan, hb, Lp, out, nexec);
  else plan_runner<float>(d, plan, hb, Lp, out, nexec);
  out[SLQ_MEM_WORKSPACE] += 2 * 4 * n;  // staging of host-pointer calls (allocated on first use)
  for (int i = 0; i < SLQ_MEM_TOTAL; ++i) out[SLQ_MEM_TOTAL] += out[i];
}

}  // namespace slq
