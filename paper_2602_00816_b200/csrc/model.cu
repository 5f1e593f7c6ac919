// MLP / GPT / Llama gradient passes on the GPU (pass dtype T = double or float).
//
// The loss is the mean token cross-entropy over the GLOBAL batch (Alg. 1 sum_b w_b = 1, P:182;
// SURVEY.md §8(c2) #1, #14): each rank scales its dlogits by 1/N_global, so the reduce-scatter
// of the unit gradients sums to grad L.  Layer math follows the oracle's definitions
// (DESIGN.md "Readings" #11); the code is independent of oracle/.
#include <math.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "model.h"

namespace slq {

int first_nonfinite_group(const double* dev, int n, int per, cudaStream_t s) {
  if (n <= 0) return -1;
  std::vector<double> h((size_t)n);
  SLQ_CUDA(cudaMemcpyAsync(h.data(), dev, sizeof(double) * (size_t)n, cudaMemcpyDeviceToHost, s));
  SLQ_CUDA(cudaStreamSynchronize(s));
  for (int i = 0; i < n; ++i)
    if (!std::isfinite(h[i])) return i / std::max(per, 1);
  return -1;
}

namespace {

// Device allocations of one runner.  Every allocation is counted under the memory-plan category
// set in `cat`; a dry arena (slq_plan_memory) only counts and returns nullptr.
enum { AC_ACT = 0, AC_LOGITS, AC_SCRATCH, AC_COUNT };
struct Arena {
  std::vector<void*> ptrs;
  bool dry = false;
  int cat = AC_ACT;
  size_t bytes[AC_COUNT] = {};
  template <class T>
  T* alloc(int64_t n) {
    void* p = nullptr;
    bytes[cat] += sizeof(T) * (size_t)std::max<int64_t>(n, 0);
    if (dry) return nullptr;
    if (n > 0) SLQ_CUDA(cudaMalloc(&p, sizeof(T) * (size_t)n));
    ptrs.push_back(p);
    return (T*)p;
  }
  ~Arena() {
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};

// Upper bound of the embedding-backward chunk count (build_embed_csr): every vocabulary row that
// occurs gets ceil(count / kEmbedChunk) chunks, so <= N / kEmbedChunk + min(V, N) over all rows
inline int64_t embed_chunks_bound(int64_t N, int64_t V) { return N / kEmbedChunk + std::min(V, N) + 1; }

// workspace of the column reductions (colreduce in layers.cu) for [rows x cols]
template <class T>
size_t colreduce_ws_bytes(int rows, int cols) {
  const int cblocks = (int)ceil_div(cols, 32);
  int rblocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 64), ceil_div(2 * 148, cblocks)));
  const int rpb = (int)ceil_div(std::max(rows, 1), rblocks);
  rblocks = (int)ceil_div(std::max(rows, 1), rpb);
  return sizeof(T) * 2 * (size_t)rblocks * cols;
}

// shape-only GEMM descriptors for workspace planning (the plans depend on M, N, K, batch, tri)
template <class T>
GemmArgs<T> shape(int M, int N, int K) {
  GemmArgs<T> a;
  a.M = M; a.N = N; a.K = K;
  return a;
}
// the largest workspace the linear layer [out x in] over N rows asks for on the data-gradient
// lane (forward + dgrad) and on the weight-gradient lane (wgrad)
template <class T>
void linear_ws(const Launch& L, int out, int in, int N, size_t& main, size_t& side) {
  main = std::max(main, gemm_ws_bytes<T>(L, shape<T>(N, out, in)));
  main = std::max(main, gemm_ws_bytes<T>(L, shape<T>(N, in, out)));
  side = std::max(side, gemm_ws_bytes<T>(L, shape<T>(out, in, N)));
}

// y[N x out] = x[N x in] . W[out x in]^T (+ bias) (+ resid), optional activation
template <class T>
void linear_fwd(const Launch& L, const T* x, int64_t ldx, const T* W, int out, int in, int N, T* y, int64_t ldy,
                const T* bias, const T* resid = nullptr, int64_t ldr = 0, int act = ACT_NONE, T* C2 = nullptr,
                int64_t ldc2 = 0) {
  GemmArgs<T> a;
  a.M = N; a.N = out; a.K = in;
  a.A = x; a.sAm = ldx; a.sAk = 1;
  a.B = W; a.sBk = 1; a.sBn = in;
  a.C = y; a.ldc = ldy;
  a.bias = bias; a.resid = resid; a.ldr = ldr; a.act = act; a.C2 = C2; a.ldc2 = ldc2;
  gemm(L, a);
}

// dx[N x in] (+)= (dy[N x out] . W[out x in]) (* activation derivative at aux)
template <class T>
void linear_dgrad(const Launch& L, const T* dy, int64_t lddy, const T* W, int out, int in, int N, T* dx,
                  int64_t lddx, int act = ACT_NONE, const T* aux = nullptr, int64_t ldaux = 0, bool acc = false) {
  GemmArgs<T> a;
  a.M = N; a.N = in; a.K = out;
  a.A = dy; a.sAm = lddy; a.sAk = 1;
  a.B = W; a.sBk = in; a.sBn = 1;
  a.C = dx; a.ldc = lddx;
  a.act = act; a.aux = aux; a.ldaux = ldaux; a.accumulate = acc;
  gemm(L, a);
}

// dW[out x in] (+)= dy[N x out]^T . x[N x in]
template <class T>
void linear_wgrad(const Launch& L, const T* dy, int64_t lddy, const T* x, int64_t ldx, int out, int in, int N, T* dW,
                  bool acc = false) {
  GemmArgs<T> a;
  a.M = out; a.N = in; a.K = N;
  a.A = dy; a.sAm = 1; a.sAk = lddy;
  a.B = x; a.sBk = ldx; a.sBn = 1;
  a.C = dW; a.ldc = in;
  a.accumulate = acc;
  gemm(L, a);
}

// dW_z[out x in] = dy_z^T . x_z for z = 0..nb-1 (one batched launch; operand z at base + z * stride)
template <class T>
void linear_wgrad_batched(const Launch& L, const T* dy, int64_t lddy, int64_t sdy, const T* x, int64_t ldx,
                          int64_t sx, int out, int in, int N, T* dW, int64_t sdw, int nb) {
  GemmArgs<T> a;
  a.M = out; a.N = in; a.K = N; a.batch = nb;
  a.A = dy; a.sAm = 1; a.sAk = lddy; a.offA = BatchOff{sdy, 0, 1, 1};
  a.B = x; a.sBk = ldx; a.sBn = 1; a.offB = BatchOff{sx, 0, 1, 1};
  a.C = dW; a.ldc = in; a.offC = BatchOff{sdw, 0, 1, 1};
  gemm(L, a);
}

// Causal multi-head attention over a packed projection buffer.
//   qkv rows r = b*Tn + t (ld = W); q head h at column qo + h*hd, kv head g at ko/vo + g*hd;
//   q head h reads kv head h / rep (GQA).  P = probabilities [nseq*Hq][Tn][Tn].
template <class T>
struct AttnGeom {
  int nseq, Tn, Hq, Hkv, hd;
  int64_t W;           // ld of the qkv buffer
  int64_t qo, ko, vo;  // column offsets
  int64_t ldo;         // ld of the merged output o [N x Hq*hd]
  int rep() const { return Hq / Hkv; }
  BatchOff qoff() const { return BatchOff{Tn * W, hd, Hq, 1}; }
  BatchOff kvoff() const { return BatchOff{Tn * W, hd, Hq, rep()}; }
  BatchOff poff() const { return BatchOff{(int64_t)Tn * Tn, 0, 1, 1}; }
  BatchOff ooff() const { return BatchOff{Tn * ldo, hd, Hq, 1}; }
};

template <class T>
AttnShape shape_of(const AttnGeom<T>& g) {
  return AttnShape{g.nseq, g.Tn, g.Hq, g.Hkv, g.hd, g.W, g.qo, g.ko, g.vo, g.ldo};
}
// workspace of the Ozaki attention path (FP64_OZ passes, eligible shapes; 0 otherwise)
template <class T>
size_t attn_ws(const Launch& L, const AttnGeom<T>& g) {
  if constexpr (sizeof(T) == 8) return attn_oz_ws_bytes(L, shape_of(g));
  return 0;
}

template <class T>
void attention_fwd(const Launch& L, const AttnGeom<T>& g, const T* qkv, T* P, T* o) {
  if constexpr (sizeof(T) == 8) {
    if (attn_oz_eligible(L, shape_of(g))) {  // all six contractions on the INT8 tensor cores (oz_attn.cu)
      attention_fwd_oz(L, shape_of(g), qkv, P, o);
      return;
    }
  }
  const T scale = T(1.0 / sqrt((double)g.hd));
  {  // S = scale * Q K^T
    GemmArgs<T> a;
    a.M = g.Tn; a.N = g.Tn; a.K = g.hd; a.batch = g.nseq * g.Hq;
    a.A = qkv + g.qo; a.sAm = g.W; a.sAk = 1; a.offA = g.qoff();
    a.B = qkv + g.ko; a.sBk = 1; a.sBn = g.W; a.offB = g.kvoff();
    a.C = P; a.ldc = g.Tn; a.offC = g.poff();
    a.alpha = scale;
    a.tri = TRI_SKIP_UPPER;
    gemm(L, a);
  }
  softmax_causal_fwd(L, P, (int64_t)g.nseq * g.Hq * g.Tn, g.Tn);
  {  // O = P V
    GemmArgs<T> a;
    a.M = g.Tn; a.N = g.hd; a.K = g.Tn; a.batch = g.nseq * g.Hq;
    a.A = P; a.sAm = g.Tn; a.sAk = 1; a.offA = g.poff();
    a.B = qkv + g.vo; a.sBk = g.W; a.sBn = 1; a.offB = g.kvoff();
    a.C = o; a.ldc = g.ldo; a.offC = g.ooff();
    a.tri = TRI_K_LE_M;
    gemm(L, a);
  }
}

// gradients w.r.t. q, k, v (written into dqkv with the qkv geometry); dP is scratch [like P]
template <class T>
void attention_bwd(const Launch& L, const AttnGeom<T>& g, const T* qkv, const T* P, const T* dO, T* dP, T* dqkv) {
  if constexpr (sizeof(T) == 8) {
    if (attn_oz_eligible(L, shape_of(g))) {
      attention_bwd_oz(L, shape_of(g), qkv, P, dO, dP, dqkv);
      return;
    }
  }
  const T scale = T(1.0 / sqrt((double)g.hd));
  const int rep = g.rep();
  // dV[b, g] = sum_{r < rep} P[b, g*rep + r]^T dO[b, g*rep + r]
  for (int r = 0; r < rep; ++r) {
    GemmArgs<T> a;
    a.M = g.Tn; a.N = g.hd; a.K = g.Tn; a.batch = g.nseq * g.Hkv;
    a.A = P + (int64_t)r * g.Tn * g.Tn; a.sAm = 1; a.sAk = g.Tn;
    a.offA = BatchOff{(int64_t)g.Hq * g.Tn * g.Tn, (int64_t)rep * g.Tn * g.Tn, g.Hkv, 1};
    a.B = dO + (int64_t)r * g.hd; a.sBk = g.ldo; a.sBn = 1;
    a.offB = BatchOff{g.Tn * g.ldo, (int64_t)rep * g.hd, g.Hkv, 1};
    a.C = dqkv + g.vo; a.ldc = g.W; a.offC = BatchOff{g.Tn * g.W, g.hd, g.Hkv, 1};
    a.accumulate = r > 0;
    a.tri = TRI_K_GE_M;
    gemm(L, a);
  }
  {  // dP = dO V^T
    GemmArgs<T> a;
    a.M = g.Tn; a.N = g.Tn; a.K = g.hd; a.batch = g.nseq * g.Hq;
    a.A = dO; a.sAm = g.ldo; a.sAk = 1; a.offA = g.ooff();
    a.B = qkv + g.vo; a.sBk = 1; a.sBn = g.W; a.offB = g.kvoff();
    a.C = dP; a.ldc = g.Tn; a.offC = g.poff();
    a.tri = TRI_SKIP_UPPER;
    gemm(L, a);
  }
  softmax_bwd(L, P, dP, (int64_t)g.nseq * g.Hq * g.Tn, g.Tn);  // dP <- dS
  {  // dQ = scale * dS K
    GemmArgs<T> a;
    a.M = g.Tn; a.N = g.hd; a.K = g.Tn; a.batch = g.nseq * g.Hq;
    a.A = dP; a.sAm = g.Tn; a.sAk = 1; a.offA = g.poff();
    a.B = qkv + g.ko; a.sBk = g.W; a.sBn = 1; a.offB = g.kvoff();
    a.C = dqkv + g.qo; a.ldc = g.W; a.offC = g.qoff();
    a.alpha = scale;
    a.tri = TRI_K_LE_M;
    gemm(L, a);
  }
  // dK[b, g] = scale * sum_r dS[b, g*rep + r]^T Q[b, g*rep + r]
  for (int r = 0; r < rep; ++r) {
    GemmArgs<T> a;
    a.M = g.Tn; a.N = g.hd; a.K = g.Tn; a.batch = g.nseq * g.Hkv;
    a.A = dP + (int64_t)r * g.Tn * g.Tn; a.sAm = 1; a.sAk = g.Tn;
    a.offA = BatchOff{(int64_t)g.Hq * g.Tn * g.Tn, (int64_t)rep * g.Tn * g.Tn, g.Hkv, 1};
    a.B = qkv + g.qo + (int64_t)r * g.hd; a.sBk = g.W; a.sBn = 1;
    a.offB = BatchOff{g.Tn * g.W, (int64_t)rep * g.hd, g.Hkv, 1};
    a.C = dqkv + g.ko; a.ldc = g.W; a.offC = BatchOff{g.Tn * g.W, g.hd, g.Hkv, 1};
    a.alpha = scale;
    a.accumulate = r > 0;
    a.tri = TRI_K_GE_M;
    gemm(L, a);
  }
}

// A second stream for the backward work that nothing on the critical path consumes (weight /
// bias / norm-gain gradients): fork() makes the side stream wait for everything issued on the
// main stream so far; join() makes the main stream wait for the side stream.  Small GEMMs do not
// fill the 148 SMs, so the weight-gradient GEMMs overlap the data-gradient chain.
struct SideStream {
  Launch main, side;
  Workspace ws;
  cudaStream_t s = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void init(const Launch& L) {
    main = L;
    SLQ_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    SLQ_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    SLQ_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    side = L;
    side.stream = s;
    side.ws = &ws;
  }
  // While the per-class profiler is on in serial mode, everything runs on the main stream so that
  // each launch's event-timed duration is its own (concurrent kernels would inflate each other's
  // durations); the overlap-aware mode keeps the side stream.
  bool serial() const { return prof_serial(main.prof); }
  const Launch& lane() const { return serial() ? main : side; }
  void fork() {
    if (serial()) return;
    SLQ_CUDA(cudaEventRecord(ev_fork, main.stream));
    SLQ_CUDA(cudaStreamWaitEvent(side.stream, ev_fork, 0));
  }
  void join() {
    if (serial()) return;
    SLQ_CUDA(cudaEventRecord(ev_join, side.stream));
    SLQ_CUDA(cudaStreamWaitEvent(main.stream, ev_join, 0));
  }
  // Lag-1 pipelining of the backward: the side stream may run up to two layers behind the data-
  // gradient chain.  mark(k) records the side stream's progress after a layer that used scratch
  // set k; wait_mark(k) makes the main stream wait for it before set k is overwritten again.
  cudaEvent_t ev_mark[2] = {nullptr, nullptr};
  bool marked[2] = {false, false};
  void begin_pass() { marked[0] = marked[1] = false; }
  void mark(int k) {
    if (serial()) return;
    if (!ev_mark[k]) SLQ_CUDA(cudaEventCreateWithFlags(&ev_mark[k], cudaEventDisableTiming));
    SLQ_CUDA(cudaEventRecord(ev_mark[k], side.stream));
    marked[k] = true;
  }
  void wait_mark(int k) {
    if (serial() || !marked[k]) return;
    SLQ_CUDA(cudaStreamWaitEvent(main.stream, ev_mark[k], 0));
  }
  ~SideStream() {
    if (s) cudaStreamSynchronize(s);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    for (cudaEvent_t e : ev_mark)
      if (e) cudaEventDestroy(e);
    if (s) cudaStreamDestroy(s);
  }
};

template <class T>
T* upload(Arena& A, const void* host, int64_t n) {
  T* d = A.alloc<T>(n);
  if (n > 0 && !A.dry) SLQ_CUDA(cudaMemcpy(d, host, sizeof(T) * (size_t)n, cudaMemcpyHostToDevice));
  return d;
}

// ------------------------------------------------------------------------------------------
template <class T>
struct MlpRunner : Runner<T> {
  Arena A;
  Launch L;
  const UnitPlan* u;
  int n, din, H, C, n_glob;
  T *x, *h, *z2, *dh;
  int32_t* y;
  double* loss_rows;

  MlpRunner(const slq_model_desc& d, const LayoutPlan& plan, const HostBatch& b, const Launch& L_, bool dry = false)
      : L(L_) {
    A.dry = dry;
    u = &plan.units[0];
    n = b.n_rows; n_glob = b.n_rows_global; din = d.d_in; H = d.d_hidden; C = d.n_classes;
    float* xf = upload<float>(A, b.x.data(), (int64_t)n * din);
    x = A.alloc<T>((int64_t)n * din);
    if (!dry) convert_f32<T>(L, xf, x, (int64_t)n * din);
    y = upload<int32_t>(A, b.y.data(), n);
    h = A.alloc<T>((int64_t)n * H);
    A.cat = AC_LOGITS;
    z2 = A.alloc<T>((int64_t)n * C);
    A.cat = AC_SCRATCH;
    dh = A.alloc<T>((int64_t)n * H);
    A.cat = AC_ACT;
    loss_rows = A.alloc<double>(std::max(n, 1));
    if (!dry) {
      size_t wm = 0, wsd = 0;
      plan_ws(wm, wsd);
      L.ws->reserve(wm);
    }
  }
  size_t arena_bytes(int c) const override { return A.bytes[c]; }
  void plan_ws(size_t& main, size_t& side) const override {  // no side stream: every GEMM on main
    size_t s2 = 0;
    linear_ws<T>(L, H, din, n, main, s2);
    linear_ws<T>(L, C, H, n, main, s2);
    main = std::max(main, s2);
    main = std::max(main, colreduce_ws_bytes<T>(n, H));
  }
  double tokens_global() const override { return n_glob; }
  int first_nonfinite_seq() override { return first_nonfinite_group(loss_rows, n, 1, L.stream); }
  double flops_per_pass() const override { return 6.0 * n * ((double)din * H + (double)H * C); }

  void fwd_bwd(PassIO<T>& io, double* loss_sum) override {
    const T* P = io.params(0);
    const T* W1 = P + u->t("fc1.w").offset;
    const T* b1 = P + u->t("fc1.b").offset;
    const T* W2 = P + u->t("fc2.w").offset;
    const T* b2 = P + u->t("fc2.b").offset;
    linear_fwd<T>(L, x, din, W1, H, din, n, h, H, b1, nullptr, 0, ACT_TANH);
    linear_fwd<T>(L, h, H, W2, C, H, n, z2, C, b2);
    cross_entropy<T>(L, z2, y, 1, 1, loss_rows, n, C, 1.0 / n_glob);
    T* G = io.grads(0);
    linear_wgrad<T>(L, z2, C, h, H, C, H, n, G + u->t("fc2.w").offset);
    colreduce<T>(L, 0, z2, C, nullptr, nullptr, nullptr, G + u->t("fc2.b").offset, nullptr, n, C, false);
    linear_dgrad<T>(L, z2, C, W2, C, H, n, dh, H, ACT_DTANH, h, H);
    linear_wgrad<T>(L, dh, H, x, din, H, din, n, G + u->t("fc1.w").offset);
    colreduce<T>(L, 0, dh, H, nullptr, nullptr, nullptr, G + u->t("fc1.b").offset, nullptr, n, H, false);
    io.grads_done(0);
    sum_rows_f64(L, loss_rows, n, loss_sum);
  }
};

// ------------------------------------------------------------------------------------------
template <class T>
struct GptRunner : Runner<T> {
  Arena A;
  Launch L;
  const LayoutPlan* plan;
  int nseq, Tn, N, D, H, hd, F, V, Ly, nseq_glob;
  bool tied, ckpt;
  double eps;
  int32_t* tok;
  EmbedCSR csr;
  double* loss_rows;
  std::vector<T*> xs;  // L+1 residual streams
  struct Layer { T *mean1, *rstd1, *h1, *qkv, *P, *o, *x1, *mean2, *rstd2, *h2, *u, *gu; };
  // block activations: one set per layer, or (activation checkpointing) two sets that the
  // forward fills alternately and the backward refills by recomputing the block forward
  std::vector<Layer> ly;
  T *meanf, *rstdf, *xf, *logits;
  // backward scratch: two sets (the side stream lags by up to one layer) and three residual-
  // gradient buffers
  struct Bwd { T *dx1, *dh1, *dh2, *dqkv, *du; } bb[2];
  T *dxs[3], *dhf, *dP, *do_;
  SideStream ss;
  // deferred weight gradients (SLQ_DEFER_WGRAD=1, fp64 DMMA passes, no collective, no
  // checkpointing): every layer's output gradients stay in per-layer slabs and the four weight-
  // gradient contractions run as one batched launch each over the layers after the data-gradient
  // chain
  bool defer_ok = false;
  T *s_h1 = nullptr, *s_o = nullptr, *s_h2 = nullptr, *s_gu = nullptr;
  T *s_dx = nullptr, *s_du = nullptr, *s_dx1 = nullptr, *s_dqkv = nullptr;

  GptRunner(const slq_model_desc& d, const LayoutPlan& p, const HostBatch& b, const Launch& L_, bool dry = false)
      : L(L_), plan(&p) {
    A.dry = dry;
    if (!dry) ss.init(L);
    nseq = b.n_seq; nseq_glob = b.n_seq_global; Tn = d.seq_len; N = nseq * Tn; D = d.d_model; H = d.n_heads;
    hd = D / H; F = d.d_ff; V = d.vocab; Ly = d.n_layers; tied = d.tie_embeddings != 0; eps = d.norm_eps;
    ckpt = d.act_ckpt != 0 && Ly > 0;
    tok = upload<int32_t>(A, b.tokens.data(), (int64_t)nseq * (Tn + 1));
    if (dry) {
      A.alloc<int32_t>(V + 1); A.alloc<int32_t>(N); A.alloc<int32_t>(V + 1);
      A.alloc<int32_t>(embed_chunks_bound(N, V) + 1);
    } else {
      std::vector<int32_t> off, pos, coff, cbeg;
      build_embed_csr(b.tokens, nseq, Tn, V, off, pos, coff, cbeg);
      csr.off = upload<int32_t>(A, off.data(), V + 1);
      csr.pos = upload<int32_t>(A, pos.data(), (int64_t)N);
      csr.coff = upload<int32_t>(A, coff.data(), V + 1);
      csr.cbeg = upload<int32_t>(A, cbeg.data(), (int64_t)cbeg.size());
      csr.nchunks = (int)cbeg.size() - 1;
    }
    loss_rows = A.alloc<double>(std::max(N, 1));
    for (int l = 0; l <= Ly; ++l) xs.push_back(A.alloc<T>((int64_t)N * D));
    const int64_t PP = (int64_t)nseq * H * Tn * Tn;
    const int nsets = ckpt ? std::min(Ly, 2) : Ly;
    if (!ckpt) {  // the weight-gradient operands of all layers in slabs (constant stride for batched launches)
      s_h1 = A.alloc<T>((int64_t)Ly * N * D); s_o = A.alloc<T>((int64_t)Ly * N * D);
      s_h2 = A.alloc<T>((int64_t)Ly * N * D); s_gu = A.alloc<T>((int64_t)Ly * N * F);
    }
    for (int l = 0; l < nsets; ++l) {
      Layer a;
      a.mean1 = A.alloc<T>(N); a.rstd1 = A.alloc<T>(N);
      a.qkv = A.alloc<T>((int64_t)N * 3 * D); a.P = A.alloc<T>(PP);
      a.x1 = A.alloc<T>((int64_t)N * D); a.mean2 = A.alloc<T>(N); a.rstd2 = A.alloc<T>(N);
      a.u = A.alloc<T>((int64_t)N * F);
      if (ckpt) {
        a.h1 = A.alloc<T>((int64_t)N * D); a.o = A.alloc<T>((int64_t)N * D);
        a.h2 = A.alloc<T>((int64_t)N * D); a.gu = A.alloc<T>((int64_t)N * F);
      } else if (!dry) {
        a.h1 = s_h1 + (int64_t)l * N * D; a.o = s_o + (int64_t)l * N * D;
        a.h2 = s_h2 + (int64_t)l * N * D; a.gu = s_gu + (int64_t)l * N * F;
      }
      ly.push_back(a);
    }
    if (!dry) {
      const char* e = getenv("SLQ_DEFER_WGRAD");
      const double mnk = (double)std::max(F, 3 * D) * D * N;  // largest per-layer weight gradient
      defer_ok = sizeof(T) == 8 && e && atoi(e) == 1 && Ly > 1 && !ckpt && (L.gemm_mode != 2 || mnk < L.oz_min_mnk);
      if (defer_ok) {
        s_dx = A.alloc<T>((int64_t)Ly * N * D); s_du = A.alloc<T>((int64_t)Ly * N * F);
        s_dx1 = A.alloc<T>((int64_t)Ly * N * D); s_dqkv = A.alloc<T>((int64_t)Ly * N * 3 * D);
      }
    }
    meanf = A.alloc<T>(N); rstdf = A.alloc<T>(N); xf = A.alloc<T>((int64_t)N * D);
    A.cat = AC_LOGITS;
    logits = A.alloc<T>((int64_t)N * V);
    A.cat = AC_SCRATCH;
    for (int i = 0; i < 3; ++i) dxs[i] = A.alloc<T>((int64_t)N * D);
    for (Bwd& b2 : bb) {
      b2.dx1 = A.alloc<T>((int64_t)N * D); b2.dh1 = A.alloc<T>((int64_t)N * D); b2.dh2 = A.alloc<T>((int64_t)N * D);
      b2.dqkv = A.alloc<T>((int64_t)N * 3 * D); b2.du = A.alloc<T>((int64_t)N * F);
    }
    dhf = A.alloc<T>((int64_t)N * D); dP = A.alloc<T>(PP); do_ = A.alloc<T>((int64_t)N * D);
    if (!dry) {  // every workspace at its planned size up front (no growth inside a pass)
      size_t wm = 0, wsd = 0;
      plan_ws(wm, wsd);
      L.ws->reserve(wm);
      ss.ws.reserve(wsd);
    }
  }
  size_t arena_bytes(int c) const override { return A.bytes[c]; }
  void plan_ws(size_t& main, size_t& side) const override {
    linear_ws<T>(L, 3 * D, D, N, main, side);
    linear_ws<T>(L, D, D, N, main, side);
    linear_ws<T>(L, F, D, N, main, side);
    linear_ws<T>(L, D, F, N, main, side);
    linear_ws<T>(L, V, D, N, main, side);
    main = std::max(main, sizeof(T) * (size_t)embed_chunks_bound(N, V) * D);
    side = std::max(side, colreduce_ws_bytes<T>(N, F));
    side = std::max(side, colreduce_ws_bytes<T>(N, 3 * D));
    main = std::max(main, attn_ws<T>(L, geom()));
  }
  double tokens_global() const override { return (double)nseq_glob * Tn; }
  int first_nonfinite_seq() override { return first_nonfinite_group(loss_rows, N, Tn, L.stream); }
  double flops_per_pass() const override {
    const double lin = (double)Ly * (3.0 * D * D + D * D + 2.0 * D * F) + (double)V * D;
    const double attn = (double)Ly * 4.0 * Tn * Tn * D * nseq;  // S and PV (full square)
    return 3.0 * (2.0 * N * lin + attn);
  }
  AttnGeom<T> geom() const {
    AttnGeom<T> g;
    g.nseq = nseq; g.Tn = Tn; g.Hq = H; g.Hkv = H; g.hd = hd; g.W = 3 * D; g.qo = 0; g.ko = D; g.vo = 2 * D; g.ldo = D;
    return g;
  }
  // block activations of layer l (checkpointing: the set shared with layer l +- 2)
  Layer& act(int l) { return ckpt ? ly[(Ly - 1 - l) & 1] : ly[l]; }

  // block l's forward from xs[l] into act(l); `out` = also the last GEMM, xs[l + 1] = x1 + mproj(gu)
  // (the backward's recomputation does not need it)
  void block_fwd(const T* Pl, const UnitPlan& ub, int l, bool out) {
    auto w = [&](const char* n) { return Pl + ub.t(n).offset; };
    Layer& a = act(l);
    layernorm_fwd<T>(L, xs[l], w("ln1.g"), w("ln1.b"), a.h1, a.mean1, a.rstd1, N, D, eps);
    linear_fwd<T>(L, a.h1, D, w("qkv.w"), 3 * D, D, N, a.qkv, 3 * D, w("qkv.b"));
    attention_fwd<T>(L, geom(), a.qkv, a.P, a.o);
    linear_fwd<T>(L, a.o, D, w("proj.w"), D, D, N, a.x1, D, w("proj.b"), xs[l], D);
    layernorm_fwd<T>(L, a.x1, w("ln2.g"), w("ln2.b"), a.h2, a.mean2, a.rstd2, N, D, eps);
    linear_fwd<T>(L, a.h2, D, w("fc.w"), F, D, N, a.gu, F, w("fc.b"), nullptr, 0, ACT_GELU, a.u, F);
    if (out) linear_fwd<T>(L, a.gu, F, w("mproj.w"), D, F, N, xs[l + 1], D, w("mproj.b"), a.x1, D);
  }

  void fwd_bwd(PassIO<T>& io, double* loss_sum) override {
    const UnitPlan& u0 = plan->units[0];
    const UnitPlan& uf = plan->units[Ly + 1];
    const AttnGeom<T> g = geom();
    // ---------------- forward ----------------
    {
      const T* P0 = io.params(0);
      io.prefetch(1);
      embed_fwd<T>(L, tok, Tn + 1, nseq, Tn, P0 + u0.t("wte").offset, P0 + u0.t("wpe").offset, xs[0], D);
    }
    for (int l = 0; l < Ly; ++l) {
      const T* Pl = io.params(1 + l);
      io.prefetch(l + 2);
      block_fwd(Pl, plan->units[1 + l], l, true);
    }
    const T* Pf = io.params(Ly + 1);
    io.prefetch(tied ? 0 : Ly);
    const T* Whead = tied ? io.params(0) + u0.t("wte").offset : Pf + uf.t("head.w").offset;
    if (tied) io.prefetch(Ly);
    layernorm_fwd<T>(L, xs[Ly], Pf + uf.t("lnf.g").offset, Pf + uf.t("lnf.b").offset, xf, meanf, rstdf, N, D, eps);
    linear_fwd<T>(L, xf, D, Whead, V, D, N, logits, V, (const T*)nullptr);
    cross_entropy<T>(L, logits, tok + 1, Tn + 1, Tn, loss_rows, N, V, 1.0 / ((double)nseq_glob * Tn));
    // ---------------- backward ----------------
    // weight / bias / gain gradients go to the side stream (Ls); the data-gradient chain stays on L
    // and only waits for the side stream when a scratch set is about to be reused (lag 1)
    const Launch& Ls = ss.lane();
    ss.begin_pass();
    T* G0 = tied ? io.grads(0) : nullptr;
    T* Gf = io.grads(Ly + 1);
    // deferral needs the layers' gradient buffers at a constant stride (no collective: one
    // contiguous gradient shard with identical block units)
    bool defer = defer_ok && !io.collective();
    int64_t gstride = 0;
    if (defer) {
      gstride = io.grads(2) - io.grads(1);
      for (int l = 2; l < Ly && defer; ++l) defer = io.grads(1 + l) - io.grads(1) == (int64_t)l * gstride;
    }
    int cur = 0;  // dxs[cur] = dL/d(residual stream) entering the current block from above
    T* dx_top = defer ? s_dx + (int64_t)(Ly - 1) * N * D : dxs[0];
    T* dx_emb = dx_top;  // the gradient leaving block 0 (input of the embedding backward)
    ss.fork();
    linear_wgrad<T>(Ls, logits, V, xf, D, V, D, N, tied ? G0 + u0.t("wte").offset : Gf + uf.t("head.w").offset);
    linear_dgrad<T>(L, logits, V, Whead, V, D, N, dhf, D);
    ss.fork();
    colreduce<T>(Ls, 1, dhf, D, xs[Ly], meanf, rstdf, Gf + uf.t("lnf.g").offset, Gf + uf.t("lnf.b").offset, N, D,
                 false);
    layernorm_bwd<T>(L, dhf, xs[Ly], meanf, rstdf, Pf + uf.t("lnf.g").offset, nullptr, dx_top, N, D);
    if (io.collective()) ss.join();
    io.grads_done(Ly + 1);
    for (int l = Ly - 1; l >= 0; --l) {
      const UnitPlan& ub = plan->units[1 + l];
      const T* Pl = io.params(1 + l);
      if (l >= 1) io.prefetch(l);
      T* Gl = io.grads(1 + l);
      auto w = [&](const char* n) { return Pl + ub.t(n).offset; };
      auto gw = [&](const char* n) { return Gl + ub.t(n).offset; };
      const int set = (Ly - 1 - l) & 1;
      ss.wait_mark(set);  // the side stream is done with this set (and with dxs[cur + 1]) from two layers up
      // checkpointing: the two top blocks' activations are still in their sets from the forward
      if (ckpt && l < Ly - 2) block_fwd(Pl, ub, l, false);
      Layer& a = act(l);
      T *dx1 = bb[set].dx1, *dh1 = bb[set].dh1, *dh2 = bb[set].dh2, *dqkv = bb[set].dqkv, *du = bb[set].du;
      T* dx = dxs[cur];
      T* dxn = dxs[(cur + 1) % 3];
      if (defer) {
        dx1 = s_dx1 + (int64_t)l * N * D; dqkv = s_dqkv + (int64_t)l * N * 3 * D; du = s_du + (int64_t)l * N * F;
        dx = s_dx + (int64_t)l * N * D;
        dxn = l > 0 ? s_dx + (int64_t)(l - 1) * N * D : dxs[1];
      }
      dx_emb = dxn;
      // MLP: xs[l+1] = x1 + mproj(gelu(fc(ln2(x1))))
      ss.fork();
      if (!defer) linear_wgrad<T>(Ls, dx, D, a.gu, F, D, F, N, gw("mproj.w"));
      colreduce<T>(Ls, 0, dx, D, nullptr, nullptr, nullptr, gw("mproj.b"), nullptr, N, D, false);
      linear_dgrad<T>(L, dx, D, w("mproj.w"), D, F, N, du, F, ACT_DGELU, a.u, F);
      ss.fork();
      if (!defer) linear_wgrad<T>(Ls, du, F, a.h2, D, F, D, N, gw("fc.w"));
      colreduce<T>(Ls, 0, du, F, nullptr, nullptr, nullptr, gw("fc.b"), nullptr, N, F, false);
      linear_dgrad<T>(L, du, F, w("fc.w"), F, D, N, dh2, D);
      ss.fork();
      colreduce<T>(Ls, 1, dh2, D, a.x1, a.mean2, a.rstd2, gw("ln2.g"), gw("ln2.b"), N, D, false);
      layernorm_bwd<T>(L, dh2, a.x1, a.mean2, a.rstd2, w("ln2.g"), dx, dx1, N, D);
      // attention: x1 = xs[l] + proj(attn(ln1(xs[l])))
      ss.fork();
      if (!defer) linear_wgrad<T>(Ls, dx1, D, a.o, D, D, D, N, gw("proj.w"));
      colreduce<T>(Ls, 0, dx1, D, nullptr, nullptr, nullptr, gw("proj.b"), nullptr, N, D, false);
      linear_dgrad<T>(L, dx1, D, w("proj.w"), D, D, N, do_, D);
      attention_bwd<T>(L, g, a.qkv, a.P, do_, dP, dqkv);
      ss.fork();
      if (!defer) linear_wgrad<T>(Ls, dqkv, 3 * D, a.h1, D, 3 * D, D, N, gw("qkv.w"));
      colreduce<T>(Ls, 0, dqkv, 3 * D, nullptr, nullptr, nullptr, gw("qkv.b"), nullptr, N, 3 * D, false);
      linear_dgrad<T>(L, dqkv, 3 * D, w("qkv.w"), 3 * D, D, N, dh1, D);
      ss.fork();
      colreduce<T>(Ls, 1, dh1, D, xs[l], a.mean1, a.rstd1, gw("ln1.g"), gw("ln1.b"), N, D, false);
      layernorm_bwd<T>(L, dh1, xs[l], a.mean1, a.rstd1, w("ln1.g"), dx1, dxn, N, D);
      ss.mark(set);
      if (io.collective()) ss.join();  // the unit's reduce-scatter needs its weight gradients
      io.grads_done(1 + l);
      cur = (cur + 1) % 3;
    }
    if (defer) {  // the four weight gradients of every block, one batched launch each
      const UnitPlan& u1 = plan->units[1];
      T* G1 = io.grads(1);
      const int64_t nd = (int64_t)N * D, nf = (int64_t)N * F;
      ss.fork();
      linear_wgrad_batched<T>(Ls, s_dx, D, nd, s_gu, F, nf, D, F, N, G1 + u1.t("mproj.w").offset, gstride, Ly);
      linear_wgrad_batched<T>(Ls, s_du, F, nf, s_h2, D, nd, F, D, N, G1 + u1.t("fc.w").offset, gstride, Ly);
      linear_wgrad_batched<T>(Ls, s_dx1, D, nd, s_o, D, nd, D, D, N, G1 + u1.t("proj.w").offset, gstride, Ly);
      linear_wgrad_batched<T>(Ls, s_dqkv, 3 * D, 3 * nd, s_h1, D, nd, 3 * D, D, N, G1 + u1.t("qkv.w").offset,
                              gstride, Ly);
    }
    ss.join();  // all side work (incl. the tied head gradient into G0) before the embedding backward
    if (!tied) G0 = io.grads(0);
    embed_bwd_rows<T>(L, csr, dx_emb, G0 + u0.t("wte").offset, V, D, tied);
    pos_bwd<T>(L, dx_emb, G0 + u0.t("wpe").offset, nseq, Tn, D);
    io.grads_done(0);
    sum_rows_f64(L, loss_rows, N, loss_sum);
  }
};

// ------------------------------------------------------------------------------------------
template <class T>
struct LlamaRunner : Runner<T> {
  Arena A;
  Launch L;
  const LayoutPlan* plan;
  int nseq, Tn, N, D, Hq, Hkv, hd, F, V, Ly, nseq_glob;
  int64_t Wq;  // width of the packed q|k|v projection
  bool tied, ckpt;
  double eps;
  int32_t* tok;
  EmbedCSR csr;
  double* loss_rows;
  T *cos_t, *sin_t;
  std::vector<T*> xs;
  struct Layer { T *rstd1, *h1, *qkv, *P, *o, *x1, *rstd2, *h2, *ab, *f; };
  std::vector<Layer> ly;  // one set per layer, or two (activation checkpointing; see GptRunner)
  T *rstdf, *xf, *logits;
  // backward scratch: two sets for what the side stream reads (lag 1), three residual gradients
  struct Bwd { T *dx1, *dh1, *dh2, *dqkv, *dab; } bb[2];
  T *dxs[3], *dhf, *dP, *do_, *df;
  SideStream ss;

  LlamaRunner(const slq_model_desc& d, const LayoutPlan& p, const HostBatch& b, const Launch& L_, bool dry = false)
      : L(L_), plan(&p) {
    A.dry = dry;
    if (!dry) ss.init(L);
    nseq = b.n_seq; nseq_glob = b.n_seq_global; Tn = d.seq_len; N = nseq * Tn; D = d.d_model; Hq = d.n_heads;
    Hkv = d.n_kv_heads; hd = D / Hq; F = d.d_ff; V = d.vocab; Ly = d.n_layers; tied = d.tie_embeddings != 0;
    eps = d.norm_eps;
    ckpt = d.act_ckpt != 0 && Ly > 0;
    Wq = (int64_t)(Hq + 2 * Hkv) * hd;
    tok = upload<int32_t>(A, b.tokens.data(), (int64_t)nseq * (Tn + 1));
    if (dry) {
      A.alloc<int32_t>(V + 1); A.alloc<int32_t>(N); A.alloc<int32_t>(V + 1);
      A.alloc<int32_t>(embed_chunks_bound(N, V) + 1);
    } else {
      std::vector<int32_t> off, pos, coff, cbeg;
      build_embed_csr(b.tokens, nseq, Tn, V, off, pos, coff, cbeg);
      csr.off = upload<int32_t>(A, off.data(), V + 1);
      csr.pos = upload<int32_t>(A, pos.data(), (int64_t)N);
      csr.coff = upload<int32_t>(A, coff.data(), V + 1);
      csr.cbeg = upload<int32_t>(A, cbeg.data(), (int64_t)cbeg.size());
      csr.nchunks = (int)cbeg.size() - 1;
    }
    loss_rows = A.alloc<double>(std::max(N, 1));
    {  // RoPE tables: angle(t, i) = t * theta^(-2i/hd)
      const int half = hd / 2;
      std::vector<T> c((size_t)Tn * half), s((size_t)Tn * half);
      for (int t = 0; t < Tn; ++t)
        for (int i = 0; i < half; ++i) {
          const double inv = pow(d.rope_theta, -(2.0 * i) / hd);
          const double ang = (double)t * inv;
          c[(size_t)t * half + i] = (T)cos(ang);
          s[(size_t)t * half + i] = (T)sin(ang);
        }
      cos_t = upload<T>(A, c.data(), (int64_t)c.size());
      sin_t = upload<T>(A, s.data(), (int64_t)s.size());
    }
    for (int l = 0; l <= Ly; ++l) xs.push_back(A.alloc<T>((int64_t)N * D));
    const int64_t PP = (int64_t)nseq * Hq * Tn * Tn;
    const int nsets = ckpt ? std::min(Ly, 2) : Ly;
    for (int l = 0; l < nsets; ++l) {
      Layer a;
      a.rstd1 = A.alloc<T>(N); a.h1 = A.alloc<T>((int64_t)N * D); a.qkv = A.alloc<T>((int64_t)N * Wq);
      a.P = A.alloc<T>(PP); a.o = A.alloc<T>((int64_t)N * Hq * hd); a.x1 = A.alloc<T>((int64_t)N * D);
      a.rstd2 = A.alloc<T>(N); a.h2 = A.alloc<T>((int64_t)N * D); a.ab = A.alloc<T>((int64_t)N * 2 * F);
      a.f = A.alloc<T>((int64_t)N * F);
      ly.push_back(a);
    }
    rstdf = A.alloc<T>(N); xf = A.alloc<T>((int64_t)N * D);
    A.cat = AC_LOGITS;
    logits = A.alloc<T>((int64_t)N * V);
    A.cat = AC_SCRATCH;
    for (int i = 0; i < 3; ++i) dxs[i] = A.alloc<T>((int64_t)N * D);
    for (Bwd& b2 : bb) {
      b2.dx1 = A.alloc<T>((int64_t)N * D); b2.dh1 = A.alloc<T>((int64_t)N * D); b2.dh2 = A.alloc<T>((int64_t)N * D);
      b2.dqkv = A.alloc<T>((int64_t)N * Wq); b2.dab = A.alloc<T>((int64_t)N * 2 * F);
    }
    dhf = A.alloc<T>((int64_t)N * D); dP = A.alloc<T>(PP); do_ = A.alloc<T>((int64_t)N * Hq * hd);
    df = A.alloc<T>((int64_t)N * F);
    if (!dry) {
      size_t wm = 0, wsd = 0;
      plan_ws(wm, wsd);
      L.ws->reserve(wm);
      ss.ws.reserve(wsd);
    }
  }
  size_t arena_bytes(int c) const override { return A.bytes[c]; }
  void plan_ws(size_t& main, size_t& side) const override {
    linear_ws<T>(L, (int)Wq, D, N, main, side);
    linear_ws<T>(L, D, Hq * hd, N, main, side);
    linear_ws<T>(L, 2 * F, D, N, main, side);
    linear_ws<T>(L, D, F, N, main, side);
    linear_ws<T>(L, V, D, N, main, side);
    main = std::max(main, sizeof(T) * (size_t)embed_chunks_bound(N, V) * D);
    side = std::max(side, colreduce_ws_bytes<T>(N, D));
    main = std::max(main, attn_ws<T>(L, geom()));
  }
  double tokens_global() const override { return (double)nseq_glob * Tn; }
  int first_nonfinite_seq() override { return first_nonfinite_group(loss_rows, N, Tn, L.stream); }
  double flops_per_pass() const override {
    const double lin = (double)Ly * ((double)Wq * D + (double)Hq * hd * D + 3.0 * D * F) + (double)V * D;
    const double attn = (double)Ly * 4.0 * Tn * Tn * Hq * hd * nseq;
    return 3.0 * (2.0 * N * lin + attn);
  }
  AttnGeom<T> geom() const {
    AttnGeom<T> g;
    g.nseq = nseq; g.Tn = Tn; g.Hq = Hq; g.Hkv = Hkv; g.hd = hd; g.W = Wq;
    g.qo = 0; g.ko = (int64_t)Hq * hd; g.vo = (int64_t)(Hq + Hkv) * hd; g.ldo = (int64_t)Hq * hd;
    return g;
  }
  Layer& act(int l) { return ckpt ? ly[(Ly - 1 - l) & 1] : ly[l]; }

  // block l's forward from xs[l] into act(l); `out`: also xs[l + 1] = x1 + wd(swiglu(...))
  void block_fwd(const T* Pl, const UnitPlan& ub, int l, bool out) {
    auto w = [&](const char* n) { return Pl + ub.t(n).offset; };
    const AttnGeom<T> g = geom();
    const int64_t HD = (int64_t)Hq * hd;
    Layer& a = act(l);
    rmsnorm_fwd<T>(L, xs[l], w("attn_norm"), a.h1, a.rstd1, N, D, eps);
    // wq, wk, wv are contiguous rows of one [Wq x D] matrix in the canonical order
    linear_fwd<T>(L, a.h1, D, w("wq"), (int)Wq, D, N, a.qkv, Wq, (const T*)nullptr);
    rope<T>(L, a.qkv + g.qo, Wq, N, Tn, Hq, hd, cos_t, sin_t, false);
    rope<T>(L, a.qkv + g.ko, Wq, N, Tn, Hkv, hd, cos_t, sin_t, false);
    attention_fwd<T>(L, g, a.qkv, a.P, a.o);
    linear_fwd<T>(L, a.o, HD, w("wo"), D, (int)HD, N, a.x1, D, (const T*)nullptr, xs[l], D);
    rmsnorm_fwd<T>(L, a.x1, w("mlp_norm"), a.h2, a.rstd2, N, D, eps);
    // wg, wu contiguous: ab = h2 [wg; wu]^T
    linear_fwd<T>(L, a.h2, D, w("wg"), 2 * F, D, N, a.ab, 2 * F, (const T*)nullptr);
    swiglu_fwd<T>(L, a.ab, a.f, N, F);
    if (out) linear_fwd<T>(L, a.f, F, w("wd"), D, F, N, xs[l + 1], D, (const T*)nullptr, a.x1, D);
  }

  void fwd_bwd(PassIO<T>& io, double* loss_sum) override {
    const UnitPlan& u0 = plan->units[0];
    const UnitPlan& uf = plan->units[Ly + 1];
    const AttnGeom<T> g = geom();
    const int64_t HD = (int64_t)Hq * hd;
    {
      const T* P0 = io.params(0);
      io.prefetch(1);
      embed_fwd<T>(L, tok, Tn + 1, nseq, Tn, P0 + u0.t("tok").offset, (const T*)nullptr, xs[0], D);
    }
    for (int l = 0; l < Ly; ++l) {
      const T* Pl = io.params(1 + l);
      io.prefetch(l + 2);
      block_fwd(Pl, plan->units[1 + l], l, true);
    }
    const T* Pf = io.params(Ly + 1);
    io.prefetch(tied ? 0 : Ly);
    const T* Whead = tied ? io.params(0) + u0.t("tok").offset : Pf + uf.t("head.w").offset;
    if (tied) io.prefetch(Ly);
    rmsnorm_fwd<T>(L, xs[Ly], Pf + uf.t("norm").offset, xf, rstdf, N, D, eps);
    linear_fwd<T>(L, xf, D, Whead, V, D, N, logits, V, (const T*)nullptr);
    cross_entropy<T>(L, logits, tok + 1, Tn + 1, Tn, loss_rows, N, V, 1.0 / ((double)nseq_glob * Tn));

    const Launch& Ls = ss.lane();
    ss.begin_pass();
    T* G0 = tied ? io.grads(0) : nullptr;
    T* Gf = io.grads(Ly + 1);
    int cur = 0;
    ss.fork();
    linear_wgrad<T>(Ls, logits, V, xf, D, V, D, N, tied ? G0 + u0.t("tok").offset : Gf + uf.t("head.w").offset);
    linear_dgrad<T>(L, logits, V, Whead, V, D, N, dhf, D);
    ss.fork();
    colreduce<T>(Ls, 2, dhf, D, xs[Ly], nullptr, rstdf, Gf + uf.t("norm").offset, nullptr, N, D, false);
    rmsnorm_bwd<T>(L, dhf, xs[Ly], rstdf, Pf + uf.t("norm").offset, nullptr, dxs[cur], N, D);
    if (io.collective()) ss.join();
    io.grads_done(Ly + 1);
    for (int l = Ly - 1; l >= 0; --l) {
      const UnitPlan& ub = plan->units[1 + l];
      const T* Pl = io.params(1 + l);
      if (l >= 1) io.prefetch(l);
      T* Gl = io.grads(1 + l);
      auto w = [&](const char* n) { return Pl + ub.t(n).offset; };
      auto gw = [&](const char* n) { return Gl + ub.t(n).offset; };
      const int set = (Ly - 1 - l) & 1;
      ss.wait_mark(set);  // side stream done with this scratch set (two layers up)
      if (ckpt && l < Ly - 2) block_fwd(Pl, ub, l, false);  // recompute (checkpointing)
      Layer& a = act(l);
      T *dx1 = bb[set].dx1, *dh1 = bb[set].dh1, *dh2 = bb[set].dh2, *dqkv = bb[set].dqkv, *dab = bb[set].dab;
      T* dx = dxs[cur];
      T* dxn = dxs[(cur + 1) % 3];
      ss.fork();
      linear_wgrad<T>(Ls, dx, D, a.f, F, D, F, N, gw("wd"));
      linear_dgrad<T>(L, dx, D, w("wd"), D, F, N, df, F);
      swiglu_bwd<T>(L, df, a.ab, dab, N, F);
      ss.fork();
      linear_wgrad<T>(Ls, dab, 2 * F, a.h2, D, 2 * F, D, N, gw("wg"));
      linear_dgrad<T>(L, dab, 2 * F, w("wg"), 2 * F, D, N, dh2, D);
      ss.fork();
      colreduce<T>(Ls, 2, dh2, D, a.x1, nullptr, a.rstd2, gw("mlp_norm"), nullptr, N, D, false);
      rmsnorm_bwd<T>(L, dh2, a.x1, a.rstd2, w("mlp_norm"), dx, dx1, N, D);
      ss.fork();
      linear_wgrad<T>(Ls, dx1, D, a.o, HD, D, (int)HD, N, gw("wo"));
      linear_dgrad<T>(L, dx1, D, w("wo"), D, (int)HD, N, do_, HD);
      attention_bwd<T>(L, g, a.qkv, a.P, do_, dP, dqkv);
      rope<T>(L, dqkv + g.qo, Wq, N, Tn, Hq, hd, cos_t, sin_t, true);
      rope<T>(L, dqkv + g.ko, Wq, N, Tn, Hkv, hd, cos_t, sin_t, true);
      ss.fork();
      linear_wgrad<T>(Ls, dqkv, Wq, a.h1, D, (int)Wq, D, N, gw("wq"));
      linear_dgrad<T>(L, dqkv, Wq, w("wq"), (int)Wq, D, N, dh1, D);
      ss.fork();
      colreduce<T>(Ls, 2, dh1, D, xs[l], nullptr, a.rstd1, gw("attn_norm"), nullptr, N, D, false);
      rmsnorm_bwd<T>(L, dh1, xs[l], a.rstd1, w("attn_norm"), dx1, dxn, N, D);
      ss.mark(set);
      if (io.collective()) ss.join();
      io.grads_done(1 + l);
      cur = (cur + 1) % 3;
    }
    ss.join();
    if (!tied) G0 = io.grads(0);
    embed_bwd_rows<T>(L, csr, dxs[cur], G0 + u0.t("tok").offset, V, D, tied);
    io.grads_done(0);
    sum_rows_f64(L, loss_rows, N, loss_sum);
  }
};

}  // namespace

template <class T>
std::unique_ptr<Runner<T>> make_runner(const slq_model_desc& d, const LayoutPlan& plan, const HostBatch& b,
                                       const Launch& L, bool dry) {
  if (d.arch == SLQ_ARCH_MLP) return std::unique_ptr<Runner<T>>(new MlpRunner<T>(d, plan, b, L, dry));
  if (d.arch == SLQ_ARCH_GPT) return std::unique_ptr<Runner<T>>(new GptRunner<T>(d, plan, b, L, dry));
  return std::unique_ptr<Runner<T>>(new LlamaRunner<T>(d, plan, b, L, dry));
}

template std::unique_ptr<Runner<double>> make_runner<double>(const slq_model_desc&, const LayoutPlan&,
                                                             const HostBatch&, const Launch&, bool);
template std::unique_ptr<Runner<float>> make_runner<float>(const slq_model_desc&, const LayoutPlan&,
                                                           const HostBatch&, const Launch&, bool);

}  // namespace slq

namespace slq {
namespace {
__global__ void k_fill_unit(double* x, int64_t n, uint64_t seed, double amp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    x[i] = amp * ((double)(int64_t)(z >> 11) / 4503599627370496.0 - 1.0);  // uniform [-amp, amp)
  }
}
}  // namespace
}  // namespace slq

extern "C" slq_status slq_diag_attn_oz(int32_t device, int32_t nseq, int32_t Tn, int32_t Hq, int32_t Hkv, int32_t hd,
                                       int32_t S, int32_t iters, double* err, double* ms) {
  using namespace slq;
  std::vector<double*> bufs;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto cleanup = [&] {
    for (double* p : bufs) cudaFree(p);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  };
  try {
    SLQ_CHECK_ARG(nseq > 0 && Tn > 0 && Hq > 0 && Hkv > 0 && Hq % Hkv == 0 && hd > 0 && S >= 4 && S <= 7 &&
                      iters >= 0 && err && ms, "arguments");
    SLQ_CUDA(cudaSetDevice(device));
    AttnGeom<double> g;
    g.nseq = nseq; g.Tn = Tn; g.Hq = Hq; g.Hkv = Hkv; g.hd = hd;
    g.W = (int64_t)(Hq + 2 * Hkv) * hd; g.qo = 0; g.ko = (int64_t)Hq * hd; g.vo = (int64_t)(Hq + Hkv) * hd;
    g.ldo = (int64_t)Hq * hd;
    const int64_t N = (int64_t)nseq * Tn, PP = (int64_t)nseq * Hq * Tn * Tn;
    auto alloc = [&](int64_t n) {
      double* p = nullptr;
      SLQ_CUDA(cudaMalloc(&p, sizeof(double) * (size_t)std::max<int64_t>(n, 1)));
      bufs.push_back(p);
      return p;
    };
    double* qkv = alloc(N * g.W);
    double* dO = alloc(N * g.ldo);
    double *P[2], *dP[2], *o[2], *dq[2];
    for (int i = 0; i < 2; ++i) {
      P[i] = alloc(PP); dP[i] = alloc(PP); o[i] = alloc(N * g.ldo); dq[i] = alloc(N * g.W);
    }
    k_fill_unit<<<1024, 256>>>(qkv, N * g.W, 21, 2.0);
    k_fill_unit<<<1024, 256>>>(dO, N * g.ldo, 22, 1.0);
    Workspace ws;
    int64_t launches = 0;
    Launch Ld{0, nullptr, &ws, &launches};
    Launch Lo = Ld;
    Lo.gemm_mode = 2; Lo.oz_S = S; Lo.oz_min_mnk = 0;
    SLQ_CHECK_ARG(attn_oz_eligible(Lo, shape_of(g)), "shape not eligible for the Ozaki attention path");
    const Launch* Ls[2] = {&Ld, &Lo};
    for (int i = 0; i < 2; ++i) {
      attention_fwd<double>(*Ls[i], g, qkv, P[i], o[i]);
      attention_bwd<double>(*Ls[i], g, qkv, P[i], dO, dP[i], dq[i]);
    }
    SLQ_CUDA(cudaDeviceSynchronize());
    // errors relative to each output's max norm: O, dQ, dK, dV
    std::vector<double> h[2][2];
    for (int i = 0; i < 2; ++i) {
      h[i][0].resize((size_t)(N * g.ldo));
      h[i][1].resize((size_t)(N * g.W));
      SLQ_CUDA(cudaMemcpy(h[i][0].data(), o[i], sizeof(double) * h[i][0].size(), cudaMemcpyDeviceToHost));
      SLQ_CUDA(cudaMemcpy(h[i][1].data(), dq[i], sizeof(double) * h[i][1].size(), cudaMemcpyDeviceToHost));
    }
    for (int k = 0; k < 4; ++k) {
      const std::vector<double>& a = h[0][k == 0 ? 0 : 1];
      const std::vector<double>& b = h[1][k == 0 ? 0 : 1];
      const int64_t ld = k == 0 ? g.ldo : g.W;
      const int64_t c0 = k == 0 ? 0 : (k == 1 ? g.qo : (k == 2 ? g.ko : g.vo));
      const int64_t nc = k <= 1 ? (int64_t)Hq * hd : (int64_t)Hkv * hd;
      double mx = 0.0, md = 0.0;
      bool bad = false;
      for (int64_t r = 0; r < N; ++r)
        for (int64_t c = 0; c < nc; ++c) {
          const double x = a[(size_t)(r * ld + c0 + c)], y = b[(size_t)(r * ld + c0 + c)];
          if (!std::isfinite(y)) bad = true;
          mx = std::max(mx, fabs(x));
          md = std::max(md, fabs(x - y));
        }
      err[k] = bad ? INFINITY : (mx > 0 ? md / mx : md);
    }
    SLQ_CUDA(cudaEventCreate(&e0));
    SLQ_CUDA(cudaEventCreate(&e1));
    for (int i = 0; i < 2; ++i) {
      float t = 0.f;
      if (iters > 0) {
        SLQ_CUDA(cudaEventRecord(e0));
        for (int it = 0; it < iters; ++it) {
          attention_fwd<double>(*Ls[i], g, qkv, P[i], o[i]);
          attention_bwd<double>(*Ls[i], g, qkv, P[i], dO, dP[i], dq[i]);
        }
        SLQ_CUDA(cudaEventRecord(e1));
        SLQ_CUDA(cudaEventSynchronize(e1));
        SLQ_CUDA(cudaEventElapsedTime(&t, e0, e1));
      }
      ms[i] = iters > 0 ? t / iters : 0.0;
    }
    cleanup();
    return SLQ_OK;
  } catch (const Error& e) {
    cleanup();
    return e.status;
  }
}
