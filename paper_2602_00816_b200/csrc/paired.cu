// Cancellation-free paired evaluation of Eq. (1).
//
// Every tensor of the two gradient evaluations is carried as a pair (mean, half-difference):
//   x+- = xbar +- xtil,    xbar = (x+ + x-)/2,   xtil = (x+ - x-)/2,
// starting from theta+- = theta +- eta v  (thetabar = theta, thetatil = eta v) and ending with
// gtil = (g+ - g-)/2, so Hv ~= gtil / eta is Eq. (1) with no subtraction of two nearly equal
// gradients.  Bilinear steps use the exact pair-product identities
//   (a b)bar = abar bbar + atil btil,      (a b)til = abar btil + atil bbar,
// (GEMMs: fp32-faithful on tcgen05 via three-term bf16 splits, or fp32 SIMT for the batched
// attention products).  Every other step (LayerNorm, GELU, softmax, cross-entropy and their
// backward) rebuilds x+- = xbar +- xtil in fp64 (exact: both are fp32), evaluates the step at
// both points in fp64 and stores (mean, half-difference) in fp32.  The fp32 rounding of a mean is
// common to both points and cancels in every later difference; a half-difference keeps fp32
// relative accuracy, so the FD difference is never formed from rounded gradients.
#include <cuda_runtime.h>
#include <math.h>

#include "paired.h"

namespace slq {

namespace {

constexpr int kWarp = 32;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

inline int grid_for(int64_t n, int threads, int cap = 148 * 16) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), cap));
}

#define PLAUNCH(cls, grid, block, kernel, ...)          \
  do {                                                  \
    LaunchScope scope_(L.prof, cls, L.stream);          \
    kernel<<<grid, block, 0, L.stream>>>(__VA_ARGS__);  \
    SLQ_CUDA(cudaGetLastError());                       \
    ++*L.launches;                                      \
  } while (0)

__device__ __forceinline__ void store_pair(float* m, float* d, int64_t i, double yp, double ym) {
  m[i] = (float)(0.5 * (yp + ym));
  d[i] = (float)(0.5 * (yp - ym));
}

// ---- LayerNorm: one warp per row; stats[row] = (mu+, r+, mu-, r-) in fp64 ----
__global__ void k_pln_fwd(const float* __restrict__ xm, const float* __restrict__ xd, const float* __restrict__ gm,
                          const float* __restrict__ gd, const float* __restrict__ bm, const float* __restrict__ bd,
                          float* __restrict__ ym, float* __restrict__ yd, double4* __restrict__ stats, int rows, int D,
                          double eps) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int64_t o = (int64_t)row * D;
  double sp = 0, sm = 0;
  for (int c = lane; c < D; c += kWarp) {
    const double a = xm[o + c], b = xd[o + c];
    sp += a + b;
    sm += a - b;
  }
  const double mup = wsum(sp) / D, mum = wsum(sm) / D;
  double vp = 0, vm = 0;
  for (int c = lane; c < D; c += kWarp) {
    const double a = xm[o + c], b = xd[o + c];
    const double cp = a + b - mup, cm = a - b - mum;
    vp += cp * cp;
    vm += cm * cm;
  }
  const double rp = 1.0 / sqrt(wsum(vp) / D + eps), rm = 1.0 / sqrt(wsum(vm) / D + eps);
  for (int c = lane; c < D; c += kWarp) {
    const double a = xm[o + c], b = xd[o + c];
    const double g0 = gm[c], g1 = gd[c], b0 = bm[c], b1 = bd[c];
    const double yp = (a + b - mup) * rp * (g0 + g1) + (b0 + b1);
    const double yq = (a - b - mum) * rm * (g0 - g1) + (b0 - b1);
    store_pair(ym, yd, o + c, yp, yq);
  }
  if (lane == 0) stats[row] = make_double4(mup, rp, mum, rm);
}

__global__ void k_pln_bwd(const float* __restrict__ dym, const float* __restrict__ dyd, const float* __restrict__ xm,
                          const float* __restrict__ xd, const double4* __restrict__ stats, const float* __restrict__ gm,
                          const float* __restrict__ gd, const float* __restrict__ rm_, const float* __restrict__ rd_,
                          float* __restrict__ dxm, float* __restrict__ dxd, int rows, int D) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int64_t o = (int64_t)row * D;
  const double4 s = stats[row];
  double a1 = 0, a2 = 0, b1 = 0, b2 = 0;
  for (int c = lane; c < D; c += kWarp) {
    const double x0 = xm[o + c], x1 = xd[o + c], d0 = dym[o + c], d1 = dyd[o + c];
    const double g0 = gm[c], g1 = gd[c];
    const double hp = (d0 + d1) * (g0 + g1), hm = (d0 - d1) * (g0 - g1);
    const double xp = (x0 + x1 - s.x) * s.y, xq = (x0 - x1 - s.z) * s.w;
    a1 += hp;
    a2 += hp * xp;
    b1 += hm;
    b2 += hm * xq;
  }
  a1 = wsum(a1) / D;
  a2 = wsum(a2) / D;
  b1 = wsum(b1) / D;
  b2 = wsum(b2) / D;
  for (int c = lane; c < D; c += kWarp) {
    const double x0 = xm[o + c], x1 = xd[o + c], d0 = dym[o + c], d1 = dyd[o + c];
    const double g0 = gm[c], g1 = gd[c];
    const double hp = (d0 + d1) * (g0 + g1), hm = (d0 - d1) * (g0 - g1);
    const double xp = (x0 + x1 - s.x) * s.y, xq = (x0 - x1 - s.z) * s.w;
    double vp = s.y * (hp - a1 - xp * a2), vq = s.w * (hm - b1 - xq * b2);
    if (rm_) {
      const double r0 = rm_[o + c], r1 = rd_[o + c];
      vp += r0 + r1;
      vq += r0 - r1;
    }
    store_pair(dxm, dxd, o + c, vp, vq);
  }
}

// LN gains / biases: column sums over rows of dy+- * xhat+- and dy+- (fp64), two stages
__global__ void k_pln_param1(const float* __restrict__ dym, const float* __restrict__ dyd, const float* __restrict__ xm,
                             const float* __restrict__ xd, const double4* __restrict__ stats, double* __restrict__ part,
                             int rows, int cols, int rpb) {
  __shared__ double s[4][8][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int c = blockIdx.x * 32 + tx;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  double gp = 0, gq = 0, bp = 0, bq = 0;
  if (c < cols) {
    for (int r = r0 + ty; r < r1; r += 8) {
      const int64_t i = (int64_t)r * cols + c;
      const double4 st = stats[r];
      const double d0 = dym[i], d1 = dyd[i], x0 = xm[i], x1 = xd[i];
      const double dp = d0 + d1, dq = d0 - d1;
      gp += dp * (x0 + x1 - st.x) * st.y;
      gq += dq * (x0 - x1 - st.z) * st.w;
      bp += dp;
      bq += dq;
    }
  }
  s[0][ty][tx] = gp;
  s[1][ty][tx] = gq;
  s[2][ty][tx] = bp;
  s[3][ty][tx] = bq;
  __syncthreads();
  if (ty < 4 && c < cols) {
    double acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += s[ty][i][tx];
    part[((int64_t)blockIdx.y * 4 + ty) * cols + c] = acc;
  }
}

// stage 2: fixed-order sum of the partials; outputs (mean, half-difference) pairs (optionally accumulated)
__global__ void k_pair_cols2(const double* __restrict__ part, int nparts, int nq, int cols, float* __restrict__ om0,
                             float* __restrict__ od0, float* __restrict__ om1, float* __restrict__ od1, bool acc) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double v[4] = {0, 0, 0, 0};
  for (int p = 0; p < nparts; ++p)
    for (int q = 0; q < nq; ++q) v[q] += part[((int64_t)p * nq + q) * cols + c];
  float* outs_m[2] = {om0, om1};
  float* outs_d[2] = {od0, od1};
  for (int k = 0; k < nq / 2; ++k) {
    if (!outs_m[k]) continue;
    const float m = (float)(0.5 * (v[2 * k] + v[2 * k + 1])), d = (float)(0.5 * (v[2 * k] - v[2 * k + 1]));
    outs_m[k][c] = acc ? outs_m[k][c] + m : m;
    outs_d[k][c] = acc ? outs_d[k][c] + d : d;
  }
}

// ---- RMSNorm (Llama): one warp per row; stats[row] = (r+, r-), y+- = x+- r+- g+- ----
__global__ void k_prms_fwd(const float* __restrict__ xm, const float* __restrict__ xd, const float* __restrict__ gm,
                           const float* __restrict__ gd, float* __restrict__ ym, float* __restrict__ yd,
                           double2* __restrict__ stats, int rows, int D, double eps) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int64_t o = (int64_t)row * D;
  double sp = 0, sq = 0;
  for (int c = lane; c < D; c += kWarp) {
    const double xp = (double)xm[o + c] + xd[o + c], xq = (double)xm[o + c] - xd[o + c];
    sp += xp * xp;
    sq += xq * xq;
  }
  const double rp = 1.0 / sqrt(wsum(sp) / D + eps), rq = 1.0 / sqrt(wsum(sq) / D + eps);
  for (int c = lane; c < D; c += kWarp) {
    const double a = xm[o + c], b = xd[o + c], g0 = gm[c], g1 = gd[c];
    store_pair(ym, yd, o + c, (a + b) * rp * (g0 + g1), (a - b) * rq * (g0 - g1));
  }
  if (lane == 0) stats[row] = make_double2(rp, rq);
}

// dx+- = r+- (h+- - x+- r+-^2 mean(h+- x+-)) (+ dres+-), h = dy g
__global__ void k_prms_bwd(const float* __restrict__ dym, const float* __restrict__ dyd, const float* __restrict__ xm,
                           const float* __restrict__ xd, const double2* __restrict__ stats, const float* __restrict__ gm,
                           const float* __restrict__ gd, const float* __restrict__ rm_, const float* __restrict__ rd_,
                           float* __restrict__ dxm, float* __restrict__ dxd, int rows, int D) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int64_t o = (int64_t)row * D;
  const double2 s = stats[row];
  double ap = 0, aq = 0;
  for (int c = lane; c < D; c += kWarp) {
    const double x0 = xm[o + c], x1 = xd[o + c], d0 = dym[o + c], d1 = dyd[o + c], g0 = gm[c], g1 = gd[c];
    ap += (d0 + d1) * (g0 + g1) * (x0 + x1);
    aq += (d0 - d1) * (g0 - g1) * (x0 - x1);
  }
  ap = wsum(ap) / D;
  aq = wsum(aq) / D;
  for (int c = lane; c < D; c += kWarp) {
    const double x0 = xm[o + c], x1 = xd[o + c], d0 = dym[o + c], d1 = dyd[o + c], g0 = gm[c], g1 = gd[c];
    double vp = s.x * ((d0 + d1) * (g0 + g1) - (x0 + x1) * s.x * s.x * ap);
    double vq = s.y * ((d0 - d1) * (g0 - g1) - (x0 - x1) * s.y * s.y * aq);
    if (rm_) {
      const double r0 = rm_[o + c], r1 = rd_[o + c];
      vp += r0 + r1;
      vq += r0 - r1;
    }
    store_pair(dxm, dxd, o + c, vp, vq);
  }
}

// RMSNorm gains: column sums over rows of dy+- x+- r+- (fp64), two stages
__global__ void k_prms_param1(const float* __restrict__ dym, const float* __restrict__ dyd, const float* __restrict__ xm,
                              const float* __restrict__ xd, const double2* __restrict__ stats, double* __restrict__ part,
                              int rows, int cols, int rpb) {
  __shared__ double s[2][8][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int c = blockIdx.x * 32 + tx;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  double gp = 0, gq = 0;
  if (c < cols) {
    for (int r = r0 + ty; r < r1; r += 8) {
      const int64_t i = (int64_t)r * cols + c;
      const double2 st = stats[r];
      const double d0 = dym[i], d1 = dyd[i], x0 = xm[i], x1 = xd[i];
      gp += (d0 + d1) * (x0 + x1) * st.x;
      gq += (d0 - d1) * (x0 - x1) * st.y;
    }
  }
  s[0][ty][tx] = gp;
  s[1][ty][tx] = gq;
  __syncthreads();
  if (ty < 2 && c < cols) {
    double acc = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += s[ty][i][tx];
    part[((int64_t)blockIdx.y * 2 + ty) * cols + c] = acc;
  }
}

// ---- SwiGLU (Llama): ab = [a | b] per row (gate | up, 2F wide), f = silu(a) b ----
__device__ __forceinline__ double sigm_d(double x) { return 1.0 / (1.0 + exp(-x)); }

__global__ void k_pswiglu_fwd(const float* __restrict__ abm, const float* __restrict__ abd, float* __restrict__ fm,
                              float* __restrict__ fd, int rows, int F) {
  const int64_t n = (int64_t)rows * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F, j = i % F, ia = r * 2 * F + j, ib = ia + F;
    const double ap = (double)abm[ia] + abd[ia], aq = (double)abm[ia] - abd[ia];
    const double bp = (double)abm[ib] + abd[ib], bq = (double)abm[ib] - abd[ib];
    store_pair(fm, fd, i, ap * sigm_d(ap) * bp, aq * sigm_d(aq) * bq);
  }
}

__global__ void k_pswiglu_bwd(const float* __restrict__ dfm, const float* __restrict__ dfd, const float* __restrict__ abm,
                              const float* __restrict__ abd, float* __restrict__ dabm, float* __restrict__ dabd, int rows,
                              int F) {
  const int64_t n = (int64_t)rows * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F, j = i % F, ia = r * 2 * F + j, ib = ia + F;
    const double ap = (double)abm[ia] + abd[ia], aq = (double)abm[ia] - abd[ia];
    const double bp = (double)abm[ib] + abd[ib], bq = (double)abm[ib] - abd[ib];
    const double dp = (double)dfm[i] + dfd[i], dq = (double)dfm[i] - dfd[i];
    const double sp = sigm_d(ap), sq = sigm_d(aq);
    store_pair(dabm, dabd, ia, dp * bp * sp * (1.0 + ap * (1.0 - sp)), dq * bq * sq * (1.0 + aq * (1.0 - sq)));
    store_pair(dabm, dabd, ib, dp * ap * sp, dq * aq * sq);
  }
}

// ---- GELU (tanh form) ----
__device__ __forceinline__ double gelu_d(double u) {
  const double c = 0.7978845608028654;
  return 0.5 * u * (1.0 + tanh(c * (u + 0.044715 * u * u * u)));
}
__device__ __forceinline__ double gelu_grad_d(double u) {
  const double c = 0.7978845608028654;
  const double t = tanh(c * (u + 0.044715 * u * u * u));
  return 0.5 * (1.0 + t) + 0.5 * u * (1.0 - t * t) * c * (1.0 + 3 * 0.044715 * u * u);
}

__global__ void k_pgelu_fwd(const float* __restrict__ um, const float* __restrict__ ud, float* __restrict__ ym,
                            float* __restrict__ yd, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = um[i], b = ud[i];
    store_pair(ym, yd, i, gelu_d(a + b), gelu_d(a - b));
  }
}

__global__ void k_pgelu_bwd(const float* __restrict__ dym, const float* __restrict__ dyd, const float* __restrict__ um,
                            const float* __restrict__ ud, float* __restrict__ dum, float* __restrict__ dud, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = um[i], b = ud[i], d0 = dym[i], d1 = dyd[i];
    store_pair(dum, dud, i, (d0 + d1) * gelu_grad_d(a + b), (d0 - d1) * gelu_grad_d(a - b));
  }
}

// ---- causal softmax over rows of length Tn (row r: query t = r % Tn, keys j <= t), in place ----
__global__ void k_psoftmax_fwd(float* __restrict__ sm, float* __restrict__ sd, int64_t rows, int Tn) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int t = (int)(row % Tn);
  float* a = sm + row * Tn;
  float* b = sd + row * Tn;
  double mp = -INFINITY, mq = -INFINITY;
  for (int j = lane; j <= t; j += kWarp) {
    const double x = a[j], y = b[j];
    mp = fmax(mp, x + y);
    mq = fmax(mq, x - y);
  }
  mp = wmax(mp);
  mq = wmax(mq);
  double zp = 0, zq = 0;
  for (int j = lane; j <= t; j += kWarp) {
    const double x = a[j], y = b[j];
    zp += exp(x + y - mp);
    zq += exp(x - y - mq);
  }
  zp = 1.0 / wsum(zp);
  zq = 1.0 / wsum(zq);
  for (int j = lane; j < Tn; j += kWarp) {
    if (j <= t) {
      const double x = a[j], y = b[j];
      store_pair(a, b, j, exp(x + y - mp) * zp, exp(x - y - mq) * zq);
    } else {
      a[j] = 0.0f;
      b[j] = 0.0f;
    }
  }
}

// dS+- = P+- (dP+- - sum_j dP+- P+-), in place into dP
__global__ void k_psoftmax_bwd(const float* __restrict__ pm, const float* __restrict__ pd, float* __restrict__ gm,
                               float* __restrict__ gd, int64_t rows, int Tn) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int t = (int)(row % Tn);
  const float* p0 = pm + row * Tn;
  const float* p1 = pd + row * Tn;
  float* d0 = gm + row * Tn;
  float* d1 = gd + row * Tn;
  double sp = 0, sq = 0;
  for (int j = lane; j <= t; j += kWarp) {
    const double pp = (double)p0[j] + p1[j], pq = (double)p0[j] - p1[j];
    const double dp = (double)d0[j] + d1[j], dq = (double)d0[j] - d1[j];
    sp += pp * dp;
    sq += pq * dq;
  }
  sp = wsum(sp);
  sq = wsum(sq);
  for (int j = lane; j < Tn; j += kWarp) {
    if (j <= t) {
      const double pp = (double)p0[j] + p1[j], pq = (double)p0[j] - p1[j];
      const double dp = (double)d0[j] + d1[j], dq = (double)d0[j] - d1[j];
      store_pair(d0, d1, j, pp * (dp - sp), pq * (dq - sq));
    } else {
      d0[j] = 0.0f;
      d1[j] = 0.0f;
    }
  }
}

// ---- token cross-entropy, one block per row; logits pair -> (softmax - onehot)/N pair in place ----
__global__ void k_pce(float* __restrict__ zm, float* __restrict__ zd, const int32_t* __restrict__ tgt, int tgt_stride,
                      int Tn, double* __restrict__ loss_rows, int V, double inv_ntok) {
  const int row = blockIdx.x;
  float* a = zm + (int64_t)row * V;
  float* b = zd + (int64_t)row * V;
  const int y = tgt[(int64_t)(row / Tn) * tgt_stride + row % Tn];
  __shared__ double red[2][32];
  double mp = -INFINITY, mq = -INFINITY;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const double x = a[j], e = b[j];
    mp = fmax(mp, x + e);
    mq = fmax(mq, x - e);
  }
  mp = wmax(mp);
  mq = wmax(mq);
  const int w = threadIdx.x / kWarp, l = threadIdx.x % kWarp, nw = blockDim.x / kWarp;
  if (l == 0) {
    red[0][w] = mp;
    red[1][w] = mq;
  }
  __syncthreads();
  mp = -INFINITY;
  mq = -INFINITY;
  for (int i = 0; i < nw; ++i) {
    mp = fmax(mp, red[0][i]);
    mq = fmax(mq, red[1][i]);
  }
  __syncthreads();
  double sp = 0, sq = 0;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const double x = a[j], e = b[j];
    sp += exp(x + e - mp);
    sq += exp(x - e - mq);
  }
  sp = wsum(sp);
  sq = wsum(sq);
  if (l == 0) {
    red[0][w] = sp;
    red[1][w] = sq;
  }
  __syncthreads();
  sp = 0;
  sq = 0;
  for (int i = 0; i < nw; ++i) {
    sp += red[0][i];
    sq += red[1][i];
  }
  if (threadIdx.x == 0) {
    const double lp = mp + log(sp) - ((double)a[y] + b[y]);
    const double lq = mq + log(sq) - ((double)a[y] - b[y]);
    loss_rows[row] = 0.5 * (lp + lq);
  }
  __syncthreads();
  const double ip = 1.0 / sp, iq = 1.0 / sq;
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const double x = a[j], e = b[j];
    double pp = exp(x + e - mp) * ip, pq = exp(x - e - mq) * iq;
    if (j == y) {
      pp -= 1.0;
      pq -= 1.0;
    }
    store_pair(a, b, j, pp * inv_ntok, pq * inv_ntok);
  }
}

__global__ void k_pscale(const float* __restrict__ v, double eta, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)(eta * (double)v[i]);
}

}  // namespace

// ------------------------------------------------------------------------------------------
void pair_layernorm_fwd(const Launch& L, CPair x, CPair g, CPair b, Pair y, double4* stats, int rows, int D,
                        double eps) {
  if (rows == 0) return;
  PLAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, k_pln_fwd, x.m, x.d, g.m, g.d, b.m, b.d, y.m, y.d, stats, rows, D,
          eps);
}

void pair_layernorm_bwd(const Launch& L, CPair dy, CPair x, const double4* stats, CPair g, CPair dres, Pair dx,
                        int rows, int D) {
  if (rows == 0) return;
  PLAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, k_pln_bwd, dy.m, dy.d, x.m, x.d, stats, g.m, g.d, dres.m, dres.d,
          dx.m, dx.d, rows, D);
}

void pair_layernorm_params(const Launch& L, CPair dy, CPair x, const double4* stats, Pair dg, Pair db, int rows,
                           int cols) {
  if (cols == 0) return;
  const int cblocks = (int)ceil_div(cols, 32);
  int rblocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 64), ceil_div(2 * 148, cblocks)));
  const int rpb = (int)ceil_div(std::max(rows, 1), rblocks);
  rblocks = (int)ceil_div(std::max(rows, 1), rpb);
  double* part = (double*)L.ws->get(sizeof(double) * 4 * (size_t)rblocks * cols, L.stream);
  PLAUNCH(KC_NORM, dim3(cblocks, rblocks), 256, k_pln_param1, dy.m, dy.d, x.m, x.d, stats, part, rows, cols, rpb);
  PLAUNCH(KC_NORM, (int)ceil_div(cols, 128), 128, k_pair_cols2, part, rblocks, 4, cols, dg.m, dg.d, db.m, db.d, false);
}

void pair_rmsnorm_fwd(const Launch& L, CPair x, CPair g, Pair y, double2* stats, int rows, int D, double eps) {
  if (rows == 0) return;
  PLAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, k_prms_fwd, x.m, x.d, g.m, g.d, y.m, y.d, stats, rows, D, eps);
}
void pair_rmsnorm_bwd(const Launch& L, CPair dy, CPair x, const double2* stats, CPair g, CPair dres, Pair dx, int rows,
                      int D) {
  if (rows == 0) return;
  PLAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, k_prms_bwd, dy.m, dy.d, x.m, x.d, stats, g.m, g.d, dres.m, dres.d,
          dx.m, dx.d, rows, D);
}
void pair_rmsnorm_params(const Launch& L, CPair dy, CPair x, const double2* stats, Pair dg, int rows, int cols) {
  if (cols == 0) return;
  const int cblocks = (int)ceil_div(cols, 32);
  int rblocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 64), ceil_div(2 * 148, cblocks)));
  const int rpb = (int)ceil_div(std::max(rows, 1), rblocks);
  rblocks = (int)ceil_div(std::max(rows, 1), rpb);
  double* part = (double*)L.ws->get(sizeof(double) * 2 * (size_t)rblocks * cols, L.stream);
  PLAUNCH(KC_NORM, dim3(cblocks, rblocks), 256, k_prms_param1, dy.m, dy.d, x.m, x.d, stats, part, rows, cols, rpb);
  PLAUNCH(KC_NORM, (int)ceil_div(cols, 128), 128, k_pair_cols2, part, rblocks, 2, cols, dg.m, dg.d, (float*)nullptr,
          (float*)nullptr, false);
}
void pair_swiglu_fwd(const Launch& L, CPair ab, Pair f, int rows, int F) {
  const int64_t n = (int64_t)rows * F;
  if (n == 0) return;
  PLAUNCH(KC_ELEM, grid_for(n, 256), 256, k_pswiglu_fwd, ab.m, ab.d, f.m, f.d, rows, F);
}
void pair_swiglu_bwd(const Launch& L, CPair df, CPair ab, Pair dab, int rows, int F) {
  const int64_t n = (int64_t)rows * F;
  if (n == 0) return;
  PLAUNCH(KC_ELEM, grid_for(n, 256), 256, k_pswiglu_bwd, df.m, df.d, ab.m, ab.d, dab.m, dab.d, rows, F);
}

void pair_gelu_fwd(const Launch& L, CPair u, Pair y, int64_t n) {
  if (n == 0) return;
  PLAUNCH(KC_ELEM, grid_for(n, 256), 256, k_pgelu_fwd, u.m, u.d, y.m, y.d, n);
}

void pair_gelu_bwd(const Launch& L, CPair dy, CPair u, Pair du, int64_t n) {
  if (n == 0) return;
  PLAUNCH(KC_ELEM, grid_for(n, 256), 256, k_pgelu_bwd, dy.m, dy.d, u.m, u.d, du.m, du.d, n);
}

void pair_softmax_causal_fwd(const Launch& L, Pair S, int64_t rows, int Tn) {
  if (rows == 0) return;
  PLAUNCH(KC_ATTN, (int)ceil_div(rows, 8), 256, k_psoftmax_fwd, S.m, S.d, rows, Tn);
}

void pair_softmax_bwd(const Launch& L, CPair P, Pair dP, int64_t rows, int Tn) {
  if (rows == 0) return;
  PLAUNCH(KC_ATTN, (int)ceil_div(rows, 8), 256, k_psoftmax_bwd, P.m, P.d, dP.m, dP.d, rows, Tn);
}

void pair_cross_entropy(const Launch& L, Pair logits, const int32_t* tgt, int tgt_stride, int Tn, double* loss_rows,
                        int rows, int V, double inv_ntok) {
  if (rows == 0) return;
  PLAUNCH(KC_CE, rows, 256, k_pce, logits.m, logits.d, tgt, tgt_stride, Tn, loss_rows, V, inv_ntok);
}

void pair_scale(const Launch& L, const float* v, double eta, float* out, int64_t n) {
  PLAUNCH(KC_PERTURB, grid_for(n, 256, 148 * 4), 256, k_pscale, v, eta, out, n);
}

// ------------------------------------------------------------------------------------------
void gemm_pair(const Launch& L, const PairGemm& g) {
  if (g.M == 0 || g.N == 0) return;
  if (L.gemm_mode == 1 && g.batch == 1 && g.K > 0) {
    // tensor cores: split the four operands once, then the mean and the half-difference GEMMs
    const size_t ta = tc_terms_bytes(g.M, g.K), tb = tc_terms_bytes(g.N, g.K);
    static const TcProd kMean[7] = {{0, 0, 0, 0}, {0, 0, 0, 1}, {0, 1, 0, 0}, {0, 1, 0, 1},
                                    {0, 0, 0, 2}, {0, 2, 0, 0}, {1, 0, 1, 0}};
    static const TcProd kDiff[12] = {{0, 0, 1, 0}, {0, 0, 1, 1}, {0, 1, 1, 0}, {0, 1, 1, 1}, {0, 0, 1, 2}, {0, 2, 1, 0},
                                     {1, 0, 0, 0}, {1, 0, 0, 1}, {1, 1, 0, 0}, {1, 1, 0, 1}, {1, 0, 0, 2}, {1, 2, 0, 0}};
    const TcPlan pm = tc_plan(g.M, g.N, g.K, 7), pd = tc_plan(g.M, g.N, g.K, 12);
    const size_t pbytes = std::max(pm.partial_bytes, pd.partial_bytes);
    uint8_t* base = (uint8_t*)L.ws->get(2 * ta + 2 * tb + pbytes, L.stream);
    TcTerms A[2], B[2];
    for (int i = 0; i < 2; ++i) {
      A[i] = tc_split_terms(L, g.A[i], g.M, g.K, g.sAm, g.sAk, base + i * ta);
      B[i] = tc_split_terms(L, g.B[i], g.N, g.K, g.sBn, g.sBk, base + 2 * ta + i * tb);
    }
    void* part = base + 2 * ta + 2 * tb;
    for (int h = 0; h < 2; ++h) {
      GemmArgs<float> e;
      e.C = g.C[h];
      e.ldc = g.ldc;
      e.alpha = g.alpha;
      e.bias = g.bias[h];
      e.resid = g.resid[h];
      e.ldr = g.ldr;
      e.accumulate = g.accumulate;
      if (h == 0)
        tc_gemm_products(L, pm, g.M, g.N, g.K, A, 2, B, 2, kMean, 7, e, part);
      else
        tc_gemm_products(L, pd, g.M, g.N, g.K, A, 2, B, 2, kDiff, 12, e, part);
    }
    return;
  }
  // SIMT fp32: C_mean = a_m b_m + a_d b_d,  C_diff = a_m b_d + a_d b_m
  for (int h = 0; h < 2; ++h) {
    for (int t = 0; t < 2; ++t) {
      GemmArgs<float> a;
      a.M = g.M; a.N = g.N; a.K = g.K; a.batch = g.batch;
      a.A = g.A[t]; a.sAm = g.sAm; a.sAk = g.sAk; a.offA = g.offA;
      a.B = g.B[h ^ t]; a.sBk = g.sBk; a.sBn = g.sBn; a.offB = g.offB;
      a.C = g.C[h]; a.ldc = g.ldc; a.offC = g.offC;
      a.alpha = g.alpha;
      a.tri = g.tri;
      if (t == 0) {
        a.bias = g.bias[h];
        a.resid = g.resid[h];
        a.ldr = g.ldr;
        a.accumulate = g.accumulate;
      } else {
        a.accumulate = true;
      }
      Launch Ls = L;
      Ls.gemm_mode = 0;  // batched / SIMT path
      gemm<float>(Ls, a);
    }
  }
}

}  // namespace slq
