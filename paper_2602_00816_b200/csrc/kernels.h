// Kernel launchers (device code in *.cu).  All launches go to L.stream and are recorded by the
// per-class profiler.  T is the pass arithmetic type (double for SLQ_PASS_FP64, float for FP32).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "common.h"

namespace slq {

struct Workspace {
  void* ptr = nullptr;
  size_t bytes = 0;
  std::vector<void*> retired;              // outgrown buffers (graphs may reference them)
  void* get(size_t need, cudaStream_t s);  // grows when too small; never frees a live buffer
  void reserve(size_t need);               // exactly `need` bytes up front (the planned maximum)
  // zero-initialised arrival counters (fixed size, allocated on first use outside graph capture);
  // every kernel that uses them leaves them zero again.  nullptr when n exceeds the array.
  unsigned* cnt = nullptr;
  static constexpr size_t kCounters = 1 << 16;
  unsigned* counters(size_t n);
  ~Workspace();
};

struct Launch {
  cudaStream_t stream;
  Profiler* prof;
  Workspace* ws;      // split-K / reduction scratch
  int64_t* launches;  // launch counter
  int gemm_mode = 0;  // float GEMMs: 0 = SIMT fp32, 1 = tcgen05 bf16x3 split (fp32-faithful),
                      // 3 = tcgen05 single bf16 term (native bf16);
                      // double GEMMs: 0 = DMMA (mma.sync f64), 2 = tcgen05 int8 Ozaki (gemm_oz)
  double oz_min_mnk = 1e9;  // gemm_mode 2: dense GEMMs with M N K below this stay on DMMA (desc.oz_min_mnk)
  int oz_S = 7;             // gemm_mode 2: Ozaki digit planes (desc.oz_slices)
};

// batch addressing of one operand: offset(z) = (z / div) * outer + ((z % div) / rep) * inner
struct BatchOff {
  int64_t outer = 0, inner = 0;
  int div = 1, rep = 1;
};

enum Act { ACT_NONE = 0, ACT_GELU = 1, ACT_TANH = 2, ACT_DGELU = 3, ACT_DTANH = 4 };

// causal-attention structure exploited by the batched attention GEMMs (row index = query t,
// column / k index = key j, nonzero only for j <= t):
//   TRI_SKIP_UPPER: C tiles entirely above the diagonal are neither computed nor written
//   TRI_K_LE_M:     A(m, k) == 0 for k > m  -> k loop stops at the tile's last row
//   TRI_K_GE_M:     A(m, k) == 0 for k < m  -> k loop starts at the tile's first row
enum Tri { TRI_NONE = 0, TRI_SKIP_UPPER = 1, TRI_K_LE_M = 2, TRI_K_GE_M = 3 };

template <class T>
struct GemmArgs {
  // C[z](m, n) (+)= epilogue( alpha * sum_k A[z](m, k) * B[z](k, n) )
  int M = 0, N = 0, K = 0, batch = 1;
  const T* A = nullptr;
  int64_t sAm = 0, sAk = 0;  // one of them must be 1
  BatchOff offA;
  const T* B = nullptr;
  int64_t sBk = 0, sBn = 0;  // one of them must be 1
  BatchOff offB;
  T* C = nullptr;
  int64_t ldc = 0;
  BatchOff offC;
  T alpha = T(1);
  const T* bias = nullptr;   // [N], added after scaling
  const T* resid = nullptr;  // added: resid[m * ldr + n]
  int64_t ldr = 0;
  const T* aux = nullptr;  // DGELU: pre-activation u;  DTANH: tanh output h
  int64_t ldaux = 0;
  T* C2 = nullptr;  // GELU: also store the pre-activation here
  int64_t ldc2 = 0;
  int act = ACT_NONE;
  bool accumulate = false;  // C += result instead of C = result
  int tri = TRI_NONE;
};

template <class T>
void gemm(const Launch& L, const GemmArgs<T>& a);
// workspace bytes L.ws->get() is asked for by gemm(L, a) (split-K partials, Ozaki digit planes):
// the memory plan and the up-front reservation of every pass workspace use it
template <class T>
size_t gemm_ws_bytes(const Launch& L, const GemmArgs<T>& a);
size_t oz_ws_bytes(int M, int N, int K, int S);
size_t tc_ws_bytes(int M, int N, int K, int terms);

// fp64 GEMM as exact INT8 digit products on the tcgen05 tensor cores (Ozaki scheme, S digit
// planes of 7 bits per operand; oz_gemm.cu).  batch == 1, dense (tri == TRI_NONE) only.
void gemm_oz(const Launch& L, const GemmArgs<double>& a, int S);

// S digit planes of one operand, already sliced: plane q of plane-batch zb, row r at
// d + ((q * nb + zb) * rows + r) * Kp (rows = M for A, N for B); ex[zb * rows + r] the row
// exponents (nullptr: 0).  GEMM batch z reads plane batch z0 + boff(z).
struct OzPlanes {
  const int8_t* d = nullptr;
  const int* ex = nullptr;
  int nb = 1, Kp = 0, z0 = 0;
  BatchOff z;
};
// batched (optionally causal, a.tri) fp64 GEMM C[z] = alpha A[z] B[z] (+ C[z] with accumulate)
// from pre-sliced planes (the attention path): a.M, a.N, a.K, a.batch, a.tri, a.C, a.ldc, a.offC,
// a.alpha, a.accumulate are used; a.A / a.B are ignored
void gemm_oz_planes(const Launch& L, int S, const OzPlanes& A, const OzPlanes& B, const GemmArgs<double>& a);

// Causal multi-head attention with its six contractions as batched Ozaki GEMMs and the digit
// planes of P and dS emitted by the softmax kernels (oz_attn.cu).  Geometry as model.cu's
// AttnGeom: qkv rows r = b Tn + t (ld W), q head h at column qo + h hd, kv head g at ko / vo + g hd;
// o / dO rows with ld ldo; P, dP [nseq Hq][Tn][Tn].
struct AttnShape {
  int nseq, Tn, Hq, Hkv, hd;
  int64_t W, qo, ko, vo, ldo;
};
bool attn_oz_eligible(const Launch& L, const AttnShape& g);
size_t attn_oz_ws_bytes(const Launch& L, const AttnShape& g);
void attention_fwd_oz(const Launch& L, const AttnShape& g, const double* qkv, double* P, double* o);
void attention_bwd_oz(const Launch& L, const AttnShape& g, const double* qkv, const double* P, const double* dO,
                      double* dP, double* dqkv);

// fp32-faithful GEMM on the tcgen05 tensor cores: every fp32 operand is split into three bf16
// terms (x = x0 + x1 + x2, 24 significant bits) and the six products with i + j <= 2 are
// accumulated in one fp32 TMEM accumulator (tc_gemm.cu).  batch == 1 only.  terms = 1: the
// operands are rounded once to bf16 and one product is formed (the native-bf16 pass mode).
void gemm_tc_bf16x3(const Launch& L, const GemmArgs<float>& a, int terms = 3);

// building blocks of multi-operand tcgen05 GEMMs (tc_gemm.cu)
struct TcTerms {  // three bf16 terms of one fp32 operand, K-contiguous [rows x ldk]
  void* t[3];
  int rows;
  int64_t ldk;
};
struct TcProd {  // one product A[ia].t[ta] . B[ib].t[tb]^T
  int ia, ta, ib, tb;
};
struct TcPlan {
  int bn, splits, tps;
  size_t partial_bytes;
};
size_t tc_terms_bytes(int rows, int K);
// X viewed as [rows x K], element (r, k) at r * s_row + k * s_k (one stride 1); writes 3 terms at dst
TcTerms tc_split_terms(const Launch& L, const float* X, int rows, int K, int64_t s_row, int64_t s_k, void* dst);
TcPlan tc_plan(int M, int N, int K, int nprods);
// epi.C (+)= epilogue(sum_p A[ia].t[ta] . B[ib].t[tb]^T) with epi's bias / resid / accumulate
void tc_gemm_products(const Launch& L, const TcPlan& plan, int M, int N, int K, const TcTerms* A, int nA,
                      const TcTerms* B, int nB, const TcProd* prods, int nprods, const GemmArgs<float>& epi,
                      void* partial_ws);

// ---- layers (layers.cu) ----
template <class T> void convert_f32(const Launch& L, const float* x, T* y, int64_t n);
template <class T> void embed_fwd(const Launch& L, const int32_t* tok, int tok_stride, int nseq, int T_,
                                  const T* wte, const T* wpe, T* x, int D);
// token positions grouped by vocabulary row (CSR), and each row's list cut into chunks of at most
// kEmbedChunk positions: chunk c covers pos[cbeg[c] .. cbeg[c + 1]), row v owns chunks
// [coff[v], coff[v + 1])
constexpr int kEmbedChunk = 16;
struct EmbedCSR {
  const int32_t* off = nullptr;
  const int32_t* pos = nullptr;
  const int32_t* coff = nullptr;
  const int32_t* cbeg = nullptr;
  int nchunks = 0;
};
void build_embed_csr(const std::vector<int32_t>& tok, int nseq, int Tn, int V, std::vector<int32_t>& off,
                     std::vector<int32_t>& pos, std::vector<int32_t>& coff, std::vector<int32_t>& cbeg);
template <class T> void embed_bwd_rows(const Launch& L, const EmbedCSR& csr, const T* dx, T* dW, int V, int D,
                                       bool accumulate);
template <class T> void pos_bwd(const Launch& L, const T* dx, T* dwpe, int nseq, int T_, int D);
template <class T> void layernorm_fwd(const Launch& L, const T* x, const T* g, const T* b, T* y, T* mean,
                                      T* rstd, int rows, int D, double eps);
template <class T> void layernorm_bwd(const Launch& L, const T* dy, const T* x, const T* mean, const T* rstd,
                                      const T* g, const T* dres, T* dx, int rows, int D);
template <class T> void rmsnorm_fwd(const Launch& L, const T* x, const T* g, T* y, T* rstd, int rows, int D,
                                    double eps);
template <class T> void rmsnorm_bwd(const Launch& L, const T* dy, const T* x, const T* rstd, const T* g,
                                    const T* dres, T* dx, int rows, int D);
// column reductions over rows (deterministic two-stage):
//   mode 0: out0[c] = sum_r dy[r,c]                                  (bias grad)
//   mode 1: out0[c] = sum_r dy*(x-mean)*rstd, out1[c] = sum_r dy     (LayerNorm g, b)
//   mode 2: out0[c] = sum_r dy*x*rstd                                 (RMSNorm g)
template <class T> void colreduce(const Launch& L, int mode, const T* dy, int64_t lddy, const T* x,
                                  const T* mean, const T* rstd, T* out0, T* out1, int rows, int cols,
                                  bool accumulate);
template <class T> void softmax_causal_fwd(const Launch& L, T* S, int64_t rows, int T_);
template <class T> void softmax_bwd(const Launch& L, const T* P, T* dP, int64_t rows, int T_);
template <class T> void cross_entropy(const Launch& L, T* logits, const int32_t* tgt, int tgt_stride, int T_,
                                      double* loss_rows, int rows, int V, double inv_ntok);
void sum_rows_f64(const Launch& L, const double* x, int n, double* out);
template <class T> void rope(const Launch& L, T* x, int64_t ld, int rows, int T_, int heads, int hd,
                             const T* cos_t, const T* sin_t, bool inverse);
// ab = [rows][2F] holding (a | b) per row (gate | up); f = silu(a) * b  [rows][F]
template <class T> void swiglu_fwd(const Launch& L, const T* ab, T* f, int rows, int F);
template <class T> void swiglu_bwd(const Launch& L, const T* df, const T* ab, T* dab, int rows, int F);
template <class T> void add_inplace(const Launch& L, T* y, const T* x, int64_t n);

// ---- vector ops of the Lanczos / FD path (vec.cu) ----
struct UnitDev {  // per-unit layout for device kernels
  int64_t local_offset, chunk, global_offset, numel, start_in_unit;
};
void probe_fill(const Launch& L, float* q, int64_t n_loc, const UnitDev* units, int n_units, uint64_t seed,
                double inv_sqrt_P);
template <class T> void perturb(const Launch& L, const float* theta, const float* v, float eta, T* plus,
                                T* minus, int64_t n);
// SLQ_PERTURB_EXACT with fp64 passes: plus/minus = theta +- eta*v in fp64 (rounded product, rounded sum)
void perturb_exact(const Launch& L, const float* theta, const float* v, double eta, double* plus, double* minus,
                   int64_t n);
// no-basis Lanczos: q_k = (w_raw - alpha_prev q_prev) / beta_k formed, stored and used for theta+- in one pass
template <class T> void perturb_lanczos(const Launch& L, bool exact, const float* theta, const float* w_raw,
                                        const float* q_prev, double alpha_prev, double beta_k, double eps,
                                        float* q_out, T* plus, T* minus, int64_t n);
// w = (g+ - g-) inv2eta - beta_k q_prev; partials[3 * block + {0,1,2}] = <w,q_k>, <w,w>, <q_k,q_k>
template <class T> void fd_partials3(const Launch& L, const T* gp, const T* gm, double inv2eta, double beta_k,
                                     const float* q_prev, const float* q_k, float* w, int64_t n, double* partials);
// partial sums of squares / dots -> partials[nblocks * k]; finalize by reduce_partials
int vec_nblocks(int64_t n);
void sumsq_partials(const Launch& L, const float* x, int64_t n, double* partials);
template <class T> void fd_w(const Launch& L, const T* gp, const T* gm, double inv2eta, const double* beta_k,
                             const float* q_prev, float* w, const float* q_k, int64_t n, double* partials);
template <class T> void fd_out(const Launch& L, const T* gp, const T* gm, double inv2eta, float* out,
                               int64_t n, int* nonfinite);
template <class T> void to_f32(const Launch& L, const T* g, float* out, int64_t n);
void reduce_partials(const Launch& L, const double* partials, int nblocks, int k, double* out);
void axpy_dev(const Launch& L, float* w, const float* q, const double* coef, double sign, int64_t n,
              double* sumsq_partials_out);
void scale_by_inv_sqrt(const Launch& L, const float* w, const double* sumsq, float* q_next, int64_t n);
int reorth_nblocks(int64_t n);
// Q: the stored Lanczos basis, fp32 or bf16 rows (B = float | __nv_bfloat16)
template <class B>
void reorth_dots(const Launch& L, const B* Q, int64_t ldq, int k, const float* w, int64_t n, double* partials);
// w -= Q[0:k]^T c; optionally the next pass's partial dots (part_dots [nb x k]) and/or ||w||^2 (part_norm [nb])
template <class B>
void reorth_update(const Launch& L, const B* Q, int64_t ldq, int k, const double* c, float* w,
                   int64_t n, double* part_dots, double* part_norm);
// one pass over Q: partials [nb x 2k] of Q^T w (first k) and Q^T q (last k)
template <class B>
void reorth_dots2(const Launch& L, const B* Q, int64_t ldq, int k, const float* w, const float* q, int64_t n,
                  double* partials);
// Gram step of the two-pass CGS2: cg = [Q^T w | Q^T q_ks] (reduced); updates row/col ks of the Gram
// matrix G (ldg), writes alpha = (Q^T w)[ks] and coef = c1 + (c1 - G c1)
void gram_coef(const Launch& L, const double* cg, int k, int ks, double* G, int ldg, double* coef, double* alpha);
// *beta = *hist = sqrt(max(*sumsq, 0)) (device-side recurrence scalar)
void step_beta(const Launch& L, const double* sumsq, double* beta, double* hist);
// bf16 basis row + exact fp32 working copy: q = bf16(x / sqrt(*sumsq)), or bf16(x * mul) if sumsq == null
void store_bf16(const Launch& L, const float* x, const double* sumsq, double mul, __nv_bfloat16* row, float* qf,
                int64_t n);
void nonfinite_check(const Launch& L, const float* x, int64_t n, int* flag);
void dot_partials(const Launch& L, const float* a, const float* b, int64_t n, double* partials);  // [vec_nblocks(n)]
void axpby(const Launch& L, float* y, const float* x, double a, double b, int64_t n);             // y = a x + b y
void mask_range(const Launch& L, const float* v, float* out, int64_t lo, int64_t hi, int64_t n);
// over [lo, hi): partials[4 * block + {0..3}] = sum (a-b)^2, a.a, a.b, b.b; returns the block count
int cmp4_partials(const Launch& L, const float* a, const float* b, int64_t lo, int64_t hi, double* partials);

}  // namespace slq
