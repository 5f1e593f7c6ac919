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

}  // namespace

std::unique_ptr<Runner<float>> make_paired_runner(const slq_model_desc& d, const LayoutPlan& plan,
                                                  const HostBatch& b, const Launch& L) {
  if (d.arch == SLQ_ARCH_GPT) return std::unique_ptr<Runner<float>>(new PairedGptRunner(d, plan, b, L));
  return nullptr;
}

}  // namespace slq
