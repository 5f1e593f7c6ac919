// GPT gradient passes in paired (mean, half-difference) form: ONE pass evaluates both
// grad L(theta + eta v) and grad L(theta - eta v) as (gbar, gtil) without ever subtracting two
// rounded gradients (see paired.cu for the arithmetic).  The layer sequence
// mirrors GptRunner in model.cu; every activation is a pair of fp32 buffers.
#include <math.h>

#include <algorithm>

#include "model.h"
#include "paired.h"

namespace slq {

namespace {

struct ArenaP {
  std::vector<void*> ptrs;
  template <class U>
  U* alloc(int64_t n) {
    void* p = nullptr;
    if (n > 0) SLQ_CUDA(cudaMalloc(&p, sizeof(U) * (size_t)n));
    ptrs.push_back(p);
    return (U*)p;
  }
  Pair pair(int64_t n) { return Pair{alloc<float>(n), alloc<float>(n)}; }
  ~ArenaP() {
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
};


// y = x W^T (+ bias) (+ resid), all pairs
void plinear_fwd(const Launch& L, CPair x, int64_t ldx, CPair W, int out, int in, int N, Pair y, int64_t ldy,
                 CPair bias, CPair resid = CPair(), int64_t ldr = 0) {
  PairGemm g;
  g.M = N; g.N = out; g.K = in;
  g.A[0] = x.m; g.A[1] = x.d; g.sAm = ldx; g.sAk = 1;
  g.B[0] = W.m; g.B[1] = W.d; g.sBk = 1; g.sBn = in;
  g.C[0] = y.m; g.C[1] = y.d; g.ldc = ldy;
  g.bias[0] = bias.m; g.bias[1] = bias.d;
  g.resid[0] = resid.m; g.resid[1] = resid.d; g.ldr = ldr;
  gemm_pair(L, g);
}
// dx = dy W
void plinear_dgrad(const Launch& L, CPair dy, int64_t lddy, CPair W, int out, int in, int N, Pair dx, int64_t lddx) {
  PairGemm g;
  g.M = N; g.N = in; g.K = out;
  g.A[0] = dy.m; g.A[1] = dy.d; g.sAm = lddy; g.sAk = 1;
  g.B[0] = W.m; g.B[1] = W.d; g.sBk = in; g.sBn = 1;
  g.C[0] = dx.m; g.C[1] = dx.d; g.ldc = lddx;
  gemm_pair(L, g);
}
// dW = dy^T x
void plinear_wgrad(const Launch& L, CPair dy, int64_t lddy, CPair x, int64_t ldx, int out, int in, int N, Pair dW) {
  PairGemm g;
  g.M = out; g.N = in; g.K = N;
  g.A[0] = dy.m; g.A[1] = dy.d; g.sAm = 1; g.sAk = lddy;
  g.B[0] = x.m; g.B[1] = x.d; g.sBk = ldx; g.sBn = 1;
  g.C[0] = dW.m; g.C[1] = dW.d; g.ldc = in;
  gemm_pair(L, g);
}

CPair off(CPair p, int64_t o) { return CPair(p.m + o, p.d + o); }
Pair off(Pair p, int64_t o) { return Pair{p.m + o, p.d + o}; }

struct PairedGptRunner : Runner<float> {
  ArenaP A;
  Launch L;
  const LayoutPlan* plan;
  int nseq, Tn, N, D, H, hd, F, V, Ly, nseq_glob;
  bool tied;
  double eps;
  int32_t* tok;
  EmbedCSR csr;
  double* loss_rows;
  std::vector<Pair> xs;
  struct Layer {
    double4 *st1, *st2;
    Pair h1, qkv, P, o, x1, h2, u, gu;
  };
  std::vector<Layer> ly;
  double4* stf;
  Pair xf, logits, dxs[2], dx1, dh1, dh2, dqkv, dP, do_, du, dgu;

  PairedGptRunner(const slq_model_desc& d, const LayoutPlan& p, const HostBatch& b, const Launch& L_)
      : L(L_), plan(&p) {
    nseq = b.n_seq; nseq_glob = b.n_seq_global; Tn = d.seq_len; N = nseq * Tn; D = d.d_model; H = d.n_heads;
    hd = D / H; F = d.d_ff; V = d.vocab; Ly = d.n_layers; tied = d.tie_embeddings != 0; eps = d.norm_eps;
    tok = A.alloc<int32_t>((int64_t)nseq * (Tn + 1));
    SLQ_CUDA(cudaMemcpy(tok, b.tokens.data(), 4 * b.tokens.size(), cudaMemcpyHostToDevice));
    {
      std::vector<int32_t> o, ps, co, cb;
      build_embed_csr(b.tokens, nseq, Tn, V, o, ps, co, cb);
      auto up = [&](const std::vector<int32_t>& v) {
        int32_t* d_ = A.alloc<int32_t>((int64_t)v.size());
        SLQ_CUDA(cudaMemcpy(d_, v.data(), 4 * v.size(), cudaMemcpyHostToDevice));
        return d_;
      };
      csr.off = up(o);
      csr.pos = up(ps);
      csr.coff = up(co);
      csr.cbeg = up(cb);
      csr.nchunks = (int)cb.size() - 1;
    }
    loss_rows = A.alloc<double>(std::max(N, 1));
    for (int l = 0; l <= Ly; ++l) xs.push_back(A.pair((int64_t)N * D));
    const int64_t PP = (int64_t)nseq * H * Tn * Tn;
    for (int l = 0; l < Ly; ++l) {
      Layer a;
      a.st1 = A.alloc<double4>(N); a.st2 = A.alloc<double4>(N);
      a.h1 = A.pair((int64_t)N * D); a.qkv = A.pair((int64_t)N * 3 * D); a.P = A.pair(PP);
      a.o = A.pair((int64_t)N * D); a.x1 = A.pair((int64_t)N * D); a.h2 = A.pair((int64_t)N * D);
      a.u = A.pair((int64_t)N * F); a.gu = A.pair((int64_t)N * F);
      ly.push_back(a);
    }
    stf = A.alloc<double4>(N);
    xf = A.pair((int64_t)N * D); logits = A.pair((int64_t)N * V);
    dxs[0] = A.pair((int64_t)N * D); dxs[1] = A.pair((int64_t)N * D); dx1 = A.pair((int64_t)N * D);
    dh1 = A.pair((int64_t)N * D); dh2 = A.pair((int64_t)N * D); dqkv = A.pair((int64_t)N * 3 * D); dP = A.pair(PP);
    do_ = A.pair((int64_t)N * D); du = A.pair((int64_t)N * F); dgu = A.pair((int64_t)N * F);
  }
  bool paired() const override { return true; }
  double tokens_global() const override { return (double)nseq_glob * Tn; }
  int first_nonfinite_seq() override { return first_nonfinite_group(loss_rows, N, Tn, L.stream); }
  double flops_per_pass() const override {  // one paired pass = the FLOPs of two plain passes x2 (pair products)
    const double lin = (double)Ly * (3.0 * D * D + D * D + 2.0 * D * F) + (double)V * D;
    const double attn = (double)Ly * 4.0 * Tn * Tn * D * nseq;
    return 2.0 * 3.0 * (2.0 * N * lin + attn);
  }
  void fwd_bwd(PassIO<float>&, double*) override {
    throw Error(SLQ_EUNSUPPORTED, "paired runner needs fwd_bwd_pair");
  }

  // batched pair GEMM over (b, h) for the attention products
  void attn_gemm(int M, int Nn, int K, CPair Am, int64_t sAm, int64_t sAk, BatchOff oA, CPair Bm, int64_t sBk,
                 int64_t sBn, BatchOff oB, Pair C, int64_t ldc, BatchOff oC, float alpha, int tri) {
    PairGemm g;
    g.M = M; g.N = Nn; g.K = K; g.batch = nseq * H;
    g.A[0] = Am.m; g.A[1] = Am.d; g.sAm = sAm; g.sAk = sAk; g.offA = oA;
    g.B[0] = Bm.m; g.B[1] = Bm.d; g.sBk = sBk; g.sBn = sBn; g.offB = oB;
    g.C[0] = C.m; g.C[1] = C.d; g.ldc = ldc; g.offC = oC;
    g.alpha = alpha; g.tri = tri;
    gemm_pair(L, g);
  }

  void fwd_bwd_pair(PassIO<float>& im, PassIO<float>& id, double* loss_sum) override {
    const UnitPlan& u0 = plan->units[0];
    const UnitPlan& uf = plan->units[Ly + 1];
    const float scale = (float)(1.0 / sqrt((double)hd));
    const int64_t W3 = 3 * D;
    const BatchOff qo{Tn * W3, hd, H, 1}, po{(int64_t)Tn * Tn, 0, 1, 1}, oo{(int64_t)Tn * D, hd, H, 1};
    auto prm = [&](int u, const UnitPlan& up, const char* n) {
      return CPair(im.params(u) + up.t(n).offset, id.params(u) + up.t(n).offset);
    };
    // ---------------- forward ----------------
    {
      const CPair wte = prm(0, u0, "wte"), wpe = prm(0, u0, "wpe");
      embed_fwd<float>(L, tok, Tn + 1, nseq, Tn, wte.m, wpe.m, xs[0].m, D);
      embed_fwd<float>(L, tok, Tn + 1, nseq, Tn, wte.d, wpe.d, xs[0].d, D);
    }
    for (int l = 0; l < Ly; ++l) {
      const UnitPlan& ub = plan->units[1 + l];
      auto w = [&](const char* n) { return prm(1 + l, ub, n); };
      Layer& a = ly[l];
      pair_layernorm_fwd(L, xs[l], w("ln1.g"), w("ln1.b"), a.h1, a.st1, N, D, eps);
      plinear_fwd(L, a.h1, D, w("qkv.w"), 3 * D, D, N, a.qkv, W3, w("qkv.b"));
      attn_gemm(Tn, Tn, hd, CPair(a.qkv), W3, 1, qo, off(CPair(a.qkv), D), 1, W3, qo, a.P, Tn, po, scale,
                TRI_SKIP_UPPER);
      pair_softmax_causal_fwd(L, a.P, (int64_t)nseq * H * Tn, Tn);
      attn_gemm(Tn, hd, Tn, CPair(a.P), Tn, 1, po, off(CPair(a.qkv), 2 * D), W3, 1, qo, a.o, D, oo, 1.0f, TRI_K_LE_M);
      plinear_fwd(L, a.o, D, w("proj.w"), D, D, N, a.x1, D, w("proj.b"), xs[l], D);
      pair_layernorm_fwd(L, a.x1, w("ln2.g"), w("ln2.b"), a.h2, a.st2, N, D, eps);
      plinear_fwd(L, a.h2, D, w("fc.w"), F, D, N, a.u, F, w("fc.b"));
      pair_gelu_fwd(L, a.u, a.gu, (int64_t)N * F);
      plinear_fwd(L, a.gu, F, w("mproj.w"), D, F, N, xs[l + 1], D, w("mproj.b"), a.x1, D);
    }
    const CPair Whead = tied ? prm(0, u0, "wte") : prm(Ly + 1, uf, "head.w");
    pair_layernorm_fwd(L, xs[Ly], prm(Ly + 1, uf, "lnf.g"), prm(Ly + 1, uf, "lnf.b"), xf, stf, N, D, eps);
    plinear_fwd(L, xf, D, Whead, V, D, N, logits, V, CPair());
    pair_cross_entropy(L, logits, tok + 1, Tn + 1, Tn, loss_rows, N, V, 1.0 / ((double)nseq_glob * Tn));
    // ---------------- backward ----------------
    auto grd = [&](int u, const UnitPlan& up, const char* n) {
      return Pair{im.grads(u) + up.t(n).offset, id.grads(u) + up.t(n).offset};
    };
    int cur = 0;
    Pair G0w{nullptr, nullptr};
    if (tied) G0w = grd(0, u0, "wte");
    plinear_wgrad(L, logits, V, xf, D, V, D, N, tied ? G0w : grd(Ly + 1, uf, "head.w"));
    plinear_dgrad(L, logits, V, Whead, V, D, N, dh2, D);
    pair_layernorm_params(L, dh2, xs[Ly], stf, grd(Ly + 1, uf, "lnf.g"), grd(Ly + 1, uf, "lnf.b"), N, D);
    pair_layernorm_bwd(L, dh2, xs[Ly], stf, prm(Ly + 1, uf, "lnf.g"), CPair(), dxs[cur], N, D);
    im.grads_done(Ly + 1);
    id.grads_done(Ly + 1);
    for (int l = Ly - 1; l >= 0; --l) {
      const UnitPlan& ub = plan->units[1 + l];
      auto w = [&](const char* n) { return prm(1 + l, ub, n); };
      auto gw = [&](const char* n) { return grd(1 + l, ub, n); };
      Layer& a = ly[l];
      const Pair dx = dxs[cur], dxn = dxs[cur ^ 1];
      // MLP
      plinear_wgrad(L, dx, D, a.gu, F, D, F, N, gw("mproj.w"));
      colreduce<float>(L, 0, dx.m, D, nullptr, nullptr, nullptr, gw("mproj.b").m, nullptr, N, D, false);
      colreduce<float>(L, 0, dx.d, D, nullptr, nullptr, nullptr, gw("mproj.b").d, nullptr, N, D, false);
      plinear_dgrad(L, dx, D, w("mproj.w"), D, F, N, dgu, F);
      pair_gelu_bwd(L, dgu, a.u, du, (int64_t)N * F);
      plinear_wgrad(L, du, F, a.h2, D, F, D, N, gw("fc.w"));
      colreduce<float>(L, 0, du.m, F, nullptr, nullptr, nullptr, gw("fc.b").m, nullptr, N, F, false);
      colreduce<float>(L, 0, du.d, F, nullptr, nullptr, nullptr, gw("fc.b").d, nullptr, N, F, false);
      plinear_dgrad(L, du, F, w("fc.w"), F, D, N, dh2, D);
      pair_layernorm_params(L, dh2, a.x1, a.st2, gw("ln2.g"), gw("ln2.b"), N, D);
      pair_layernorm_bwd(L, dh2, a.x1, a.st2, w("ln2.g"), dx, dx1, N, D);
      // attention
      plinear_wgrad(L, dx1, D, a.o, D, D, D, N, gw("proj.w"));
      colreduce<float>(L, 0, dx1.m, D, nullptr, nullptr, nullptr, gw("proj.b").m, nullptr, N, D, false);
      colreduce<float>(L, 0, dx1.d, D, nullptr, nullptr, nullptr, gw("proj.b").d, nullptr, N, D, false);
      plinear_dgrad(L, dx1, D, w("proj.w"), D, D, N, do_, D);
      // dV = P^T dO
      attn_gemm(Tn, hd, Tn, CPair(a.P), 1, Tn, po, CPair(do_), D, 1, oo, off(dqkv, 2 * D), W3, qo, 1.0f, TRI_K_GE_M);
      // dP = dO V^T
      attn_gemm(Tn, Tn, hd, CPair(do_), D, 1, oo, off(CPair(a.qkv), 2 * D), 1, W3, qo, dP, Tn, po, 1.0f,
                TRI_SKIP_UPPER);
      pair_softmax_bwd(L, a.P, dP, (int64_t)nseq * H * Tn, Tn);
      // dQ = scale dS K ; dK = scale dS^T Q
      attn_gemm(Tn, hd, Tn, CPair(dP), Tn, 1, po, off(CPair(a.qkv), D), W3, 1, qo, dqkv, W3, qo, scale, TRI_K_LE_M);
      attn_gemm(Tn, hd, Tn, CPair(dP), 1, Tn, po, CPair(a.qkv), W3, 1, qo, off(dqkv, D), W3, qo, scale, TRI_K_GE_M);
      plinear_wgrad(L, dqkv, W3, a.h1, D, 3 * D, D, N, gw("qkv.w"));
      colreduce<float>(L, 0, dqkv.m, W3, nullptr, nullptr, nullptr, gw("qkv.b").m, nullptr, N, 3 * D, false);
      colreduce<float>(L, 0, dqkv.d, W3, nullptr, nullptr, nullptr, gw("qkv.b").d, nullptr, N, 3 * D, false);
      plinear_dgrad(L, dqkv, W3, w("qkv.w"), 3 * D, D, N, dh1, D);
      pair_layernorm_params(L, dh1, xs[l], a.st1, gw("ln1.g"), gw("ln1.b"), N, D);
      pair_layernorm_bwd(L, dh1, xs[l], a.st1, w("ln1.g"), dx1, dxn, N, D);
      im.grads_done(1 + l);
      id.grads_done(1 + l);
      cur ^= 1;
    }
    const Pair gwte = grd(0, u0, "wte"), gwpe = grd(0, u0, "wpe");
    embed_bwd_rows<float>(L, csr, dxs[cur].m, gwte.m, V, D, tied);
    embed_bwd_rows<float>(L, csr, dxs[cur].d, gwte.d, V, D, tied);
    pos_bwd<float>(L, dxs[cur].m, gwpe.m, nseq, Tn, D);
    pos_bwd<float>(L, dxs[cur].d, gwpe.d, nseq, Tn, D);
    im.grads_done(0);
    id.grads_done(0);
    sum_rows_f64(L, loss_rows, N, loss_sum);
  }
};


// Llama in paired form (RMSNorm, RoPE, GQA attention, SwiGLU, no biases, untied or tied head):
// the layer sequence mirrors LlamaRunner in model.cu with every activation a pair of fp32 buffers.
// RoPE is linear, so it acts on the mean and the half-difference separately; RMSNorm and SwiGLU
// are evaluated at both points in fp64 (paired.cu).
struct PairedLlamaRunner : Runner<float> {
  ArenaP A;
  Launch L;
  const LayoutPlan* plan;
  int nseq, Tn, N, D, Hq, Hkv, hd, F, V, Ly, nseq_glob;
  int64_t Wq;
  bool tied;
  double eps;
  int32_t* tok;
  EmbedCSR csr;
  double* loss_rows;
  float *cos_t, *sin_t;
  std::vector<Pair> xs;
  struct Layer {
    double2 *st1, *st2;
    Pair h1, qkv, P, o, x1, h2, ab, f;
  };
  std::vector<Layer> ly;
  double2* stf;
  Pair xf, logits, dxs[2], dx1, dh1, dh2, dqkv, dP, do_, df, dab;

  PairedLlamaRunner(const slq_model_desc& d, const LayoutPlan& p, const HostBatch& b, const Launch& L_)
      : L(L_), plan(&p) {
    nseq = b.n_seq; nseq_glob = b.n_seq_global; Tn = d.seq_len; N = nseq * Tn; D = d.d_model; Hq = d.n_heads;
    Hkv = d.n_kv_heads; hd = D / Hq; F = d.d_ff; V = d.vocab; Ly = d.n_layers; tied = d.tie_embeddings != 0;
    eps = d.norm_eps;
    Wq = (int64_t)(Hq + 2 * Hkv) * hd;
    tok = A.alloc<int32_t>((int64_t)nseq * (Tn + 1));
    SLQ_CUDA(cudaMemcpy(tok, b.tokens.data(), 4 * b.tokens.size(), cudaMemcpyHostToDevice));
    auto up = [&](const void* src, size_t bytes) {
      void* d_ = A.alloc<uint8_t>((int64_t)bytes);
      SLQ_CUDA(cudaMemcpy(d_, src, bytes, cudaMemcpyHostToDevice));
      return d_;
    };
    {
      std::vector<int32_t> o, ps, co, cb;
      build_embed_csr(b.tokens, nseq, Tn, V, o, ps, co, cb);
      csr.off = (int32_t*)up(o.data(), 4 * o.size());
      csr.pos = (int32_t*)up(ps.data(), 4 * ps.size());
      csr.coff = (int32_t*)up(co.data(), 4 * co.size());
      csr.cbeg = (int32_t*)up(cb.data(), 4 * cb.size());
      csr.nchunks = (int)cb.size() - 1;
    }
    {  // RoPE tables (as LlamaRunner): angle(t, i) = t * theta^(-2i/hd)
      const int half = hd / 2;
      std::vector<float> c((size_t)Tn * half), s((size_t)Tn * half);
      for (int t = 0; t < Tn; ++t)
        for (int i = 0; i < half; ++i) {
          const double ang = (double)t * pow(d.rope_theta, -(2.0 * i) / hd);
          c[(size_t)t * half + i] = (float)cos(ang);
          s[(size_t)t * half + i] = (float)sin(ang);
        }
      cos_t = (float*)up(c.data(), 4 * c.size());
      sin_t = (float*)up(s.data(), 4 * s.size());
    }
    loss_rows = A.alloc<double>(std::max(N, 1));
    for (int l = 0; l <= Ly; ++l) xs.push_back(A.pair((int64_t)N * D));
    const int64_t PP = (int64_t)nseq * Hq * Tn * Tn;
    for (int l = 0; l < Ly; ++l) {
      Layer a;
      a.st1 = A.alloc<double2>(N); a.st2 = A.alloc<double2>(N);
      a.h1 = A.pair((int64_t)N * D); a.qkv = A.pair((int64_t)N * Wq); a.P = A.pair(PP);
      a.o = A.pair((int64_t)N * Hq * hd); a.x1 = A.pair((int64_t)N * D); a.h2 = A.pair((int64_t)N * D);
      a.ab = A.pair((int64_t)N * 2 * F); a.f = A.pair((int64_t)N * F);
      ly.push_back(a);
    }
    stf = A.alloc<double2>(N);
    xf = A.pair((int64_t)N * D); logits = A.pair((int64_t)N * V);
    dxs[0] = A.pair((int64_t)N * D); dxs[1] = A.pair((int64_t)N * D); dx1 = A.pair((int64_t)N * D);
    dh1 = A.pair((int64_t)N * D); dh2 = A.pair((int64_t)N * D); dqkv = A.pair((int64_t)N * Wq); dP = A.pair(PP);
    do_ = A.pair((int64_t)N * Hq * hd); df = A.pair((int64_t)N * F); dab = A.pair((int64_t)N * 2 * F);
  }
  bool paired() const override { return true; }
  double tokens_global() const override { return (double)nseq_glob * Tn; }
  int first_nonfinite_seq() override { return first_nonfinite_group(loss_rows, N, Tn, L.stream); }
  double flops_per_pass() const override {
    const double lin = (double)Ly * ((double)Wq * D + (double)Hq * hd * D + 3.0 * D * F) + (double)V * D;
    const double attn = (double)Ly * 4.0 * Tn * Tn * Hq * hd * nseq;
    return 2.0 * 3.0 * (2.0 * N * lin + attn);
  }
  void fwd_bwd(PassIO<float>&, double*) override {
    throw Error(SLQ_EUNSUPPORTED, "paired runner needs fwd_bwd_pair");
  }

  void attn_gemm(int batch, int M, int Nn, int K, CPair Am, int64_t sAm, int64_t sAk, BatchOff oA, CPair Bm, int64_t sBk,
                 int64_t sBn, BatchOff oB, Pair C, int64_t ldc, BatchOff oC, float alpha, int tri, bool acc = false) {
    PairGemm g;
    g.M = M; g.N = Nn; g.K = K; g.batch = batch;
    g.A[0] = Am.m; g.A[1] = Am.d; g.sAm = sAm; g.sAk = sAk; g.offA = oA;
    g.B[0] = Bm.m; g.B[1] = Bm.d; g.sBk = sBk; g.sBn = sBn; g.offB = oB;
    g.C[0] = C.m; g.C[1] = C.d; g.ldc = ldc; g.offC = oC;
    g.alpha = alpha; g.tri = tri; g.accumulate = acc;
    gemm_pair(L, g);
  }
  void rope2(Pair x, int64_t col, int heads, bool inverse) {
    rope<float>(L, x.m + col, Wq, N, Tn, heads, hd, cos_t, sin_t, inverse);
    rope<float>(L, x.d + col, Wq, N, Tn, heads, hd, cos_t, sin_t, inverse);
  }

  void fwd_bwd_pair(PassIO<float>& im, PassIO<float>& id, double* loss_sum) override {
    const UnitPlan& u0 = plan->units[0];
    const UnitPlan& uf = plan->units[Ly + 1];
    const float scale = (float)(1.0 / sqrt((double)hd));
    const int rep = Hq / Hkv;
    const int64_t HD = (int64_t)Hq * hd, ko = HD, vo = HD + (int64_t)Hkv * hd;
    // geometry as AttnGeom in model.cu: q head h reads kv head h / rep
    const BatchOff qoff{Tn * Wq, hd, Hq, 1}, kvoff{Tn * Wq, hd, Hq, rep}, po{(int64_t)Tn * Tn, 0, 1, 1},
        ooff{Tn * HD, hd, Hq, 1};
    auto prm = [&](int u, const UnitPlan& upl, const char* n) {
      return CPair(im.params(u) + upl.t(n).offset, id.params(u) + upl.t(n).offset);
    };
    {
      const CPair emb = prm(0, u0, "tok");
      embed_fwd<float>(L, tok, Tn + 1, nseq, Tn, emb.m, (const float*)nullptr, xs[0].m, D);
      embed_fwd<float>(L, tok, Tn + 1, nseq, Tn, emb.d, (const float*)nullptr, xs[0].d, D);
    }
    for (int l = 0; l < Ly; ++l) {
      const UnitPlan& ub = plan->units[1 + l];
      auto w = [&](const char* n) { return prm(1 + l, ub, n); };
      Layer& a = ly[l];
      pair_rmsnorm_fwd(L, xs[l], w("attn_norm"), a.h1, a.st1, N, D, eps);
      plinear_fwd(L, a.h1, D, w("wq"), (int)Wq, D, N, a.qkv, Wq, CPair());
      rope2(a.qkv, 0, Hq, false);
      rope2(a.qkv, ko, Hkv, false);
      attn_gemm(nseq * Hq, Tn, Tn, hd, CPair(a.qkv), Wq, 1, qoff, off(CPair(a.qkv), ko), 1, Wq, kvoff, a.P, Tn, po,
                scale, TRI_SKIP_UPPER);
      pair_softmax_causal_fwd(L, a.P, (int64_t)nseq * Hq * Tn, Tn);
      attn_gemm(nseq * Hq, Tn, hd, Tn, CPair(a.P), Tn, 1, po, off(CPair(a.qkv), vo), Wq, 1, kvoff, a.o, HD, ooff, 1.0f,
                TRI_K_LE_M);
      plinear_fwd(L, a.o, HD, w("wo"), D, (int)HD, N, a.x1, D, CPair(), xs[l], D);
      pair_rmsnorm_fwd(L, a.x1, w("mlp_norm"), a.h2, a.st2, N, D, eps);
      plinear_fwd(L, a.h2, D, w("wg"), 2 * F, D, N, a.ab, 2 * F, CPair());
      pair_swiglu_fwd(L, a.ab, a.f, N, F);
      plinear_fwd(L, a.f, F, w("wd"), D, F, N, xs[l + 1], D, CPair(), a.x1, D);
    }
    const CPair Whead = tied ? prm(0, u0, "tok") : prm(Ly + 1, uf, "head.w");
    pair_rmsnorm_fwd(L, xs[Ly], prm(Ly + 1, uf, "norm"), xf, stf, N, D, eps);
    plinear_fwd(L, xf, D, Whead, V, D, N, logits, V, CPair());
    pair_cross_entropy(L, logits, tok + 1, Tn + 1, Tn, loss_rows, N, V, 1.0 / ((double)nseq_glob * Tn));
    // ---------------- backward ----------------
    auto grd = [&](int u, const UnitPlan& upl, const char* n) {
      return Pair{im.grads(u) + upl.t(n).offset, id.grads(u) + upl.t(n).offset};
    };
    int cur = 0;
    plinear_wgrad(L, logits, V, xf, D, V, D, N, tied ? grd(0, u0, "tok") : grd(Ly + 1, uf, "head.w"));
    plinear_dgrad(L, logits, V, Whead, V, D, N, dh2, D);
    pair_rmsnorm_params(L, dh2, xs[Ly], stf, grd(Ly + 1, uf, "norm"), N, D);
    pair_rmsnorm_bwd(L, dh2, xs[Ly], stf, prm(Ly + 1, uf, "norm"), CPair(), dxs[cur], N, D);
    im.grads_done(Ly + 1);
    id.grads_done(Ly + 1);
    for (int l = Ly - 1; l >= 0; --l) {
      const UnitPlan& ub = plan->units[1 + l];
      auto w = [&](const char* n) { return prm(1 + l, ub, n); };
      auto gw = [&](const char* n) { return grd(1 + l, ub, n); };
      Layer& a = ly[l];
      const Pair dx = dxs[cur], dxn = dxs[cur ^ 1];
      // MLP: xs[l+1] = x1 + wd(swiglu(h2 [wg; wu]^T))
      plinear_wgrad(L, dx, D, a.f, F, D, F, N, gw("wd"));
      plinear_dgrad(L, dx, D, w("wd"), D, F, N, df, F);
      pair_swiglu_bwd(L, df, a.ab, dab, N, F);
      plinear_wgrad(L, dab, 2 * F, a.h2, D, 2 * F, D, N, gw("wg"));
      plinear_dgrad(L, dab, 2 * F, w("wg"), 2 * F, D, N, dh2, D);
      pair_rmsnorm_params(L, dh2, a.x1, a.st2, gw("mlp_norm"), N, D);
      pair_rmsnorm_bwd(L, dh2, a.x1, a.st2, w("mlp_norm"), dx, dx1, N, D);
      // attention
      plinear_wgrad(L, dx1, D, a.o, HD, D, (int)HD, N, gw("wo"));
      plinear_dgrad(L, dx1, D, w("wo"), D, (int)HD, N, do_, HD);
      // dV[b, g] = sum_r P[b, g rep + r]^T dO[b, g rep + r];  dK likewise with dS and Q
      for (int r = 0; r < rep; ++r)
        attn_gemm(nseq * Hkv, Tn, hd, Tn, off(CPair(a.P), (int64_t)r * Tn * Tn), 1, Tn,
                  BatchOff{(int64_t)Hq * Tn * Tn, (int64_t)rep * Tn * Tn, Hkv, 1}, off(CPair(do_), (int64_t)r * hd), HD,
                  1, BatchOff{Tn * HD, (int64_t)rep * hd, Hkv, 1}, off(dqkv, vo), Wq, BatchOff{Tn * Wq, hd, Hkv, 1}, 1.0f,
                  TRI_K_GE_M, r > 0);
      // dP = dO V^T
      attn_gemm(nseq * Hq, Tn, Tn, hd, CPair(do_), HD, 1, ooff, off(CPair(a.qkv), vo), 1, Wq, kvoff, dP, Tn, po, 1.0f,
                TRI_SKIP_UPPER);
      pair_softmax_bwd(L, a.P, dP, (int64_t)nseq * Hq * Tn, Tn);
      // dQ = scale dS K
      attn_gemm(nseq * Hq, Tn, hd, Tn, CPair(dP), Tn, 1, po, off(CPair(a.qkv), ko), Wq, 1, kvoff, dqkv, Wq, qoff, scale,
                TRI_K_LE_M);
      for (int r = 0; r < rep; ++r)
        attn_gemm(nseq * Hkv, Tn, hd, Tn, off(CPair(dP), (int64_t)r * Tn * Tn), 1, Tn,
                  BatchOff{(int64_t)Hq * Tn * Tn, (int64_t)rep * Tn * Tn, Hkv, 1}, off(CPair(a.qkv), (int64_t)r * hd),
                  Wq, 1, BatchOff{Tn * Wq, (int64_t)rep * hd, Hkv, 1}, off(dqkv, ko), Wq, BatchOff{Tn * Wq, hd, Hkv, 1},
                  scale, TRI_K_GE_M, r > 0);
      rope2(dqkv, 0, Hq, true);
      rope2(dqkv, ko, Hkv, true);
      plinear_wgrad(L, dqkv, Wq, a.h1, D, (int)Wq, D, N, gw("wq"));
      plinear_dgrad(L, dqkv, Wq, w("wq"), (int)Wq, D, N, dh1, D);
      pair_rmsnorm_params(L, dh1, xs[l], a.st1, gw("attn_norm"), N, D);
      pair_rmsnorm_bwd(L, dh1, xs[l], a.st1, w("attn_norm"), dx1, dxn, N, D);
      im.grads_done(1 + l);
      id.grads_done(1 + l);
      cur ^= 1;
    }
    const Pair gemb = grd(0, u0, "tok");
    embed_bwd_rows<float>(L, csr, dxs[cur].m, gemb.m, V, D, tied);
    embed_bwd_rows<float>(L, csr, dxs[cur].d, gemb.d, V, D, tied);
    im.grads_done(0);
    id.grads_done(0);
    sum_rows_f64(L, loss_rows, N, loss_sum);
  }
};

}  // namespace

std::unique_ptr<Runner<float>> make_paired_runner(const slq_model_desc& d, const LayoutPlan& plan,
                                                  const HostBatch& b, const Launch& L) {
  if (d.arch == SLQ_ARCH_GPT) return std::unique_ptr<Runner<float>>(new PairedGptRunner(d, plan, b, L));
  if (d.arch == SLQ_ARCH_LLAMA) return std::unique_ptr<Runner<float>>(new PairedLlamaRunner(d, plan, b, L));
  return nullptr;
}

}  // namespace slq
