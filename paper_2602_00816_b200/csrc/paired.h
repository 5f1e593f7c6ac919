// Paired (mean, half-difference) evaluation of the two gradient passes (paired.cu).
#pragma once

#include "kernels.h"

namespace slq {

struct Pair {
  float* m;  // mean of the +/- evaluations
  float* d;  // half-difference
};
struct CPair {
  const float* m;
  const float* d;
  CPair() : m(nullptr), d(nullptr) {}
  CPair(const float* m_, const float* d_) : m(m_), d(d_) {}
  CPair(const Pair& p) : m(p.m), d(p.d) {}
};

// C+- = A+- B+- with pair products: C_mean = A_m B_m + A_d B_d, C_diff = A_m B_d + A_d B_m,
// then alpha, bias (pair), residual (pair), accumulate.  Non-batched on tcgen05 when
// L.gemm_mode == 1 (fp32-faithful three-term splits), else fp32 SIMT.
struct PairGemm {
  int M = 0, N = 0, K = 0, batch = 1;
  const float* A[2] = {nullptr, nullptr};
  int64_t sAm = 0, sAk = 0;
  BatchOff offA;
  const float* B[2] = {nullptr, nullptr};
  int64_t sBk = 0, sBn = 0;
  BatchOff offB;
  float* C[2] = {nullptr, nullptr};
  int64_t ldc = 0;
  BatchOff offC;
  float alpha = 1.0f;
  const float* bias[2] = {nullptr, nullptr};
  const float* resid[2] = {nullptr, nullptr};
  int64_t ldr = 0;
  bool accumulate = false;
  int tri = TRI_NONE;
};
void gemm_pair(const Launch& L, const PairGemm& g);

void pair_layernorm_fwd(const Launch& L, CPair x, CPair g, CPair b, Pair y, double4* stats, int rows, int D,
                        double eps);
void pair_layernorm_bwd(const Launch& L, CPair dy, CPair x, const double4* stats, CPair g, CPair dres, Pair dx,
                        int rows, int D);
void pair_layernorm_params(const Launch& L, CPair dy, CPair x, const double4* stats, Pair dg, Pair db, int rows,
                           int cols);
void pair_rmsnorm_fwd(const Launch& L, CPair x, CPair g, Pair y, double2* stats, int rows, int D, double eps);
void pair_rmsnorm_bwd(const Launch& L, CPair dy, CPair x, const double2* stats, CPair g, CPair dres, Pair dx, int rows,
                      int D);
void pair_rmsnorm_params(const Launch& L, CPair dy, CPair x, const double2* stats, Pair dg, int rows, int cols);
void pair_swiglu_fwd(const Launch& L, CPair ab, Pair f, int rows, int F);
void pair_swiglu_bwd(const Launch& L, CPair df, CPair ab, Pair dab, int rows, int F);
void pair_gelu_fwd(const Launch& L, CPair u, Pair y, int64_t n);
void pair_gelu_bwd(const Launch& L, CPair dy, CPair u, Pair du, int64_t n);
void pair_softmax_causal_fwd(const Launch& L, Pair S, int64_t rows, int Tn);
void pair_softmax_bwd(const Launch& L, CPair P, Pair dP, int64_t rows, int Tn);
void pair_cross_entropy(const Launch& L, Pair logits, const int32_t* tgt, int tgt_stride, int Tn, double* loss_rows,
                        int rows, int V, double inv_ntok);
// out = fl32(eta * v): the half-difference of the perturbed parameters, thetatil = eta v
void pair_scale(const Launch& L, const float* v, double eta, float* out, int64_t n);

}  // namespace slq
