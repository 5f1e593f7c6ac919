#include "layout.h"

#include "common.h"

namespace slq {

const TensorSlot& UnitPlan::t(const std::string& n) const {
  for (auto& s : tensors)
    if (s.name == n) return s;
  throw Error(SLQ_EINVAL, "internal: no tensor " + n);
}

void validate_desc(const slq_model_desc& d) {
  SLQ_CHECK_ARG(d.arch == SLQ_ARCH_MLP || d.arch == SLQ_ARCH_GPT || d.arch == SLQ_ARCH_LLAMA, "arch");
  SLQ_CHECK_ARG(d.pass_numerics >= SLQ_PASS_FP64 && d.pass_numerics <= SLQ_PASS_BF16, "pass_numerics");
  SLQ_CHECK_ARG(d.param_dtype == SLQ_PARAM_FP32 || d.param_dtype == SLQ_PARAM_BF16, "param_dtype");
  SLQ_CHECK_ARG(d.reorth == SLQ_REORTH_NONE || d.reorth == SLQ_REORTH_FULL || d.reorth == SLQ_REORTH_WINDOW,
                "reorth");
  SLQ_CHECK_ARG(d.reorth != SLQ_REORTH_WINDOW || d.reorth_window >= 2, "reorth_window >= 2 for SLQ_REORTH_WINDOW");
  SLQ_CHECK_ARG(d.basis_dtype == SLQ_BASIS_FP32 || d.basis_dtype == SLQ_BASIS_BF16, "basis_dtype");
  SLQ_CHECK_ARG(d.basis_dtype == SLQ_BASIS_FP32 || d.reorth != SLQ_REORTH_NONE,
                "a bf16 basis needs reorth FULL or WINDOW (NONE keeps no basis)");
  SLQ_CHECK_ARG(d.perturb == SLQ_PERTURB_EXACT || d.perturb == SLQ_PERTURB_STORAGE, "perturb");
  SLQ_CHECK_ARG(d.max_steps >= 1 && d.max_steps <= 4096, "max_steps in [1, 4096]");
  SLQ_CHECK_ARG(d.eps_default > 0, "eps_default > 0");
  if (d.arch == SLQ_ARCH_MLP) {
    SLQ_CHECK_ARG(d.d_in > 0 && d.d_hidden > 0 && d.n_classes > 1, "MLP dims");
    return;
  }
  SLQ_CHECK_ARG(d.n_layers >= 1 && d.d_model > 0 && d.n_heads > 0 && d.d_ff > 0 && d.vocab > 1 &&
                    d.seq_len > 0, "transformer dims");
  SLQ_CHECK_ARG(d.d_model % d.n_heads == 0, "d_model % n_heads");
  SLQ_CHECK_ARG(d.norm_eps > 0, "norm_eps");
  if (d.arch == SLQ_ARCH_LLAMA) {
    SLQ_CHECK_ARG(d.n_kv_heads > 0 && d.n_heads % d.n_kv_heads == 0, "n_heads % n_kv_heads");
    SLQ_CHECK_ARG((d.d_model / d.n_heads) % 2 == 0, "RoPE needs an even head dim");
    SLQ_CHECK_ARG(d.rope_theta > 0, "rope_theta");
  }
}

namespace {
struct Builder {
  LayoutPlan plan;
  UnitPlan cur;
  void add(const std::string& n, int64_t r, int64_t c = 1) {
    cur.tensors.push_back({n, cur.numel, r, c});
    cur.numel += r * c;
  }
  void close() {
    plan.units.push_back(cur);
    cur = UnitPlan();
  }
};
}  // namespace

LayoutPlan plan_layout(const slq_model_desc& d, int world) {
  validate_desc(d);
  SLQ_CHECK_ARG(world >= 1, "world_size >= 1");
  Builder b;
  if (d.arch == SLQ_ARCH_MLP) {
    b.add("fc1.w", d.d_hidden, d.d_in);
    b.add("fc1.b", d.d_hidden);
    b.add("fc2.w", d.n_classes, d.d_hidden);
    b.add("fc2.b", d.n_classes);
    b.close();
  } else {
    const int64_t D = d.d_model, F = d.d_ff, V = d.vocab;
    if (d.arch == SLQ_ARCH_GPT) {
      b.add("wte", V, D);
      b.add("wpe", d.seq_len, D);
      b.close();
      for (int l = 0; l < d.n_layers; ++l) {
        b.add("ln1.g", D); b.add("ln1.b", D);
        b.add("qkv.w", 3 * D, D); b.add("qkv.b", 3 * D);
        b.add("proj.w", D, D); b.add("proj.b", D);
        b.add("ln2.g", D); b.add("ln2.b", D);
        b.add("fc.w", F, D); b.add("fc.b", F);
        b.add("mproj.w", D, F); b.add("mproj.b", D);
        b.close();
      }
      b.add("lnf.g", D); b.add("lnf.b", D);
      if (!d.tie_embeddings) b.add("head.w", V, D);
      b.close();
    } else {
      const int64_t hd = D / d.n_heads;
      b.add("tok", V, D);
      b.close();
      for (int l = 0; l < d.n_layers; ++l) {
        b.add("attn_norm", D);
        b.add("wq", d.n_heads * hd, D);
        b.add("wk", d.n_kv_heads * hd, D);
        b.add("wv", d.n_kv_heads * hd, D);
        b.add("wo", D, d.n_heads * hd);
        b.add("mlp_norm", D);
        b.add("wg", F, D); b.add("wu", F, D); b.add("wd", D, F);
        b.close();
      }
      b.add("norm", D);
      if (!d.tie_embeddings) b.add("head.w", V, D);
      b.close();
    }
  }
  LayoutPlan& p = b.plan;
  p.world = world;
  int64_t g = 0, l = 0;
  const int64_t align = 16 * (int64_t)world;
  for (auto& u : p.units) {
    u.global_offset = g;
    u.padded = ceil_div(u.numel, align) * align;
    u.chunk = u.padded / world;
    u.local_offset = l;
    g += u.numel;
    l += u.chunk;
  }
  p.P = g;
  p.P_loc = l;
  return p;
}

}  // namespace slq
