// Shard-local vector kernels of the FD-HVP / Lanczos path:
// Rademacher probe from the integer splitmix64 hash, out-of-place fp32 FMA perturbation,
// the FD difference fused with the three-term update, deterministic fixed-grid reductions
// (partials in fp64, finalised in a fixed order), and the CGS reorthogonalisation GEMVs.
// All are HBM-bound streaming kernels: one pass, vectorised where aligned, grids sized in
// multiples of the 148 SMs.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>

#include "kernels.h"

namespace slq {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// fixed-order block sum; result valid in thread 0
__device__ __forceinline__ double block_sum_d(double v) {
  __shared__ double red[32];
  v = warp_sum_d(v);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double r = 0.0;
  if (w == 0) {
    r = (l < (int)(blockDim.x / 32)) ? red[l] : 0.0;
    r = warp_sum_d(r);
  }
  return r;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// q[i] = s(seed, gid(i)) / sqrt(P); padding -> 0
__global__ void k_probe(float* __restrict__ q, int64_t n, const UnitDev* __restrict__ units, int nu, uint64_t key,
                        double inv_sqrt_P) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int lo = 0, hi = nu - 1;
    while (lo < hi) {  // last unit with local_offset <= i
      const int mid = (lo + hi + 1) / 2;
      if (units[mid].local_offset <= i) lo = mid; else hi = mid - 1;
    }
    const UnitDev u = units[lo];
    const int64_t p = u.start_in_unit + (i - u.local_offset);
    float v = 0.0f;
    if (p < u.numel) {
      const uint64_t gid = (uint64_t)(u.global_offset + p);
      const bool neg = (splitmix64(key ^ gid) >> 63) != 0;
      v = (float)(neg ? -inv_sqrt_P : inv_sqrt_P);
    }
    q[i] = v;
  }
}

template <class T>
__global__ void k_perturb(const float* __restrict__ th, const float* __restrict__ v, float eta, T* __restrict__ plus,
                          T* __restrict__ minus, int64_t n) {
  const int64_t n4 = n / 4;
  const float4* th4 = reinterpret_cast<const float4*>(th);
  const float4* v4 = reinterpret_cast<const float4*>(v);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 t = th4[i], d = v4[i];
    const int64_t b = 4 * i;
    plus[b + 0] = (T)__fmaf_rn(eta, d.x, t.x);
    plus[b + 1] = (T)__fmaf_rn(eta, d.y, t.y);
    plus[b + 2] = (T)__fmaf_rn(eta, d.z, t.z);
    plus[b + 3] = (T)__fmaf_rn(eta, d.w, t.w);
    minus[b + 0] = (T)__fmaf_rn(-eta, d.x, t.x);
    minus[b + 1] = (T)__fmaf_rn(-eta, d.y, t.y);
    minus[b + 2] = (T)__fmaf_rn(-eta, d.z, t.z);
    minus[b + 3] = (T)__fmaf_rn(-eta, d.w, t.w);
  }
  for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    plus[i] = (T)__fmaf_rn(eta, v[i], th[i]);
    minus[i] = (T)__fmaf_rn(-eta, v[i], th[i]);
  }
}

// theta +- eta*v in fp64 with explicit roundings (product, then sum; no contraction) -- the
// same two operations, in the same order, as evaluating theta + eta*v in fp64 elementwise
__global__ void k_perturb_exact(const float* __restrict__ th, const float* __restrict__ v, double eta,
                                double* __restrict__ plus, double* __restrict__ minus, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double t = (double)th[i];
    const double d = __dmul_rn(eta, (double)v[i]);
    plus[i] = __dadd_rn(t, d);
    minus[i] = __dsub_rn(t, d);
  }
}

// Lanczos step without a stored basis (deferred normalisation): forms
// q_k = (w_raw - alpha_prev q_prev) / beta_k from the previous step's residual, stores it, and
// writes theta +- eps q_k in the same pass.  EXACT: fp64 points (rounded product, rounded sum)
// from the stored fp32 q_k; STORAGE: fmaf into fp32.
template <class T, bool EXACT>
__global__ void k_perturb_lanczos(const float* __restrict__ th, const float* __restrict__ w_raw,
                                  const float* __restrict__ q_prev, double alpha_prev, double inv_beta, double eps,
                                  float eps_f, float* __restrict__ q_out, T* __restrict__ plus, T* __restrict__ minus,
                                  int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float q = (float)(((double)w_raw[i] - alpha_prev * (double)q_prev[i]) * inv_beta);
    q_out[i] = q;
    if (EXACT) {
      const double t = (double)th[i];
      const double d = __dmul_rn(eps, (double)q);
      plus[i] = (T)__dadd_rn(t, d);
      minus[i] = (T)__dsub_rn(t, d);
    } else {
      plus[i] = (T)__fmaf_rn(eps_f, q, th[i]);
      minus[i] = (T)__fmaf_rn(-eps_f, q, th[i]);
    }
  }
}

// FD difference fused with the three-term update and the three Lanczos partials (one HBM pass,
// north-star row (d)): w = (g+ - g-) inv2eta - beta_k q_prev;  partials <w,q_k>, <w,w>, <q_k,q_k>
template <class T>
__global__ void k_fd_partials3(const T* __restrict__ gp, const T* __restrict__ gm, double inv2eta, double beta_k,
                               const float* __restrict__ q_prev, const float* __restrict__ q_k, float* __restrict__ w,
                               int64_t n, double* __restrict__ part) {
  double s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double d = (gm ? (double)gp[i] - (double)gm[i] : (double)gp[i]) * inv2eta;
    if (q_prev) d -= beta_k * (double)q_prev[i];
    const float wf = (float)d;
    w[i] = wf;
    const double wd = wf, qd = q_k[i];
    s1 += wd * qd;
    s2 += wd * wd;
    s3 += qd * qd;
  }
  s1 = block_sum_d(s1);
  s2 = block_sum_d(s2);
  s3 = block_sum_d(s3);
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x + 0] = s1;
    part[3 * blockIdx.x + 1] = s2;
    part[3 * blockIdx.x + 2] = s3;
  }
}

__global__ void k_sumsq(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    s += v * v;
  }
  s = block_sum_d(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// w = (g+ - g-) * inv2eta - beta_k * q_prev ; partial <w, q_k> (w after fp32 rounding)
template <class T>
__global__ void k_fd_w(const T* __restrict__ gp, const T* __restrict__ gm, double inv2eta,
                       const double* __restrict__ beta_k, const float* __restrict__ q_prev, float* __restrict__ w,
                       const float* __restrict__ q_k, int64_t n, double* __restrict__ part) {
  const double b = beta_k ? *beta_k : 0.0;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double d = (gm ? (double)gp[i] - (double)gm[i] : (double)gp[i]) * inv2eta;
    if (beta_k) d -= b * (double)q_prev[i];
    const float wf = (float)d;
    w[i] = wf;
    if (part) s += (double)wf * (double)q_k[i];
  }
  if (part) {
    s = block_sum_d(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

template <class T>
__global__ void k_fd_out(const T* __restrict__ gp, const T* __restrict__ gm, double inv2eta, float* __restrict__ out,
                         int64_t n, int* __restrict__ nonfinite) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double d = (gm ? (double)gp[i] - (double)gm[i] : (double)gp[i]) * inv2eta;
    if (!isfinite(d)) bad = 1;
    out[i] = (float)d;
  }
  if (bad && nonfinite) atomicOr(nonfinite, 1);
}

template <class T>
__global__ void k_to_f32(const T* __restrict__ g, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (float)g[i];
}

// out[j] = sum_b part[b * k + j], fixed order (one block per j)
__global__ void k_reduce_partials(const double* __restrict__ part, int nb, int k, double* __restrict__ out) {
  const int j = blockIdx.x;
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += part[(int64_t)b * k + j];
  s = block_sum_d(s);
  if (threadIdx.x == 0) out[j] = s;
}

// w += sign * coef * q ; optional partial ||w||^2
__global__ void k_axpy(float* __restrict__ w, const float* __restrict__ q, const double* __restrict__ coef, double sign,
                       int64_t n, double* __restrict__ part) {
  const double c = sign * *coef;
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = (float)((double)w[i] + c * (double)q[i]);
    w[i] = v;
    s += (double)v * (double)v;
  }
  if (part) {
    s = block_sum_d(s);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
}

__global__ void k_scale_inv_sqrt(const float* __restrict__ w, const double* __restrict__ sumsq, float* __restrict__ q,
                                 int64_t n) {
  const double inv = 1.0 / sqrt(*sumsq);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    q[i] = (float)((double)w[i] * inv);
}

constexpr int kReorthChunk = 4096;

// The CGS kernels work on 4096-element chunks (one block each; the chunk of w lives in shared
// memory).  Q rows are P_loc apart and P_loc is a multiple of 16, so every chunk is float4-aligned.
constexpr int kRThreads = 256;
constexpr int kRGroups = kReorthChunk / 4 / kRThreads;  // float4 groups per thread in the update

// 4 consecutive basis elements as float4 (the basis is stored fp32 or bf16)
__device__ __forceinline__ float4 ld_q4(const float* p, int i4) { return reinterpret_cast<const float4*>(p)[i4]; }
__device__ __forceinline__ float4 ld_q4(const __nv_bfloat16* p, int i4) {
  const uint2 u = reinterpret_cast<const uint2*>(p)[i4];
  const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
  const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  const float2 a = __bfloat1622float2(lo), b = __bfloat1622float2(hi);
  return make_float4(a.x, a.y, b.x, b.y);
}

// partial dots of the shared-memory chunk ws[0, len) with rows 0..k-1 of Q (one warp per row)
template <class B>
__device__ __forceinline__ void chunk_dots(const B* __restrict__ Q, int64_t ldq, int k, int64_t base, int len,
                                           const float* ws, double* __restrict__ part_row) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int n4 = len / 4;
  const float4* w4 = reinterpret_cast<const float4*>(ws);
  for (int j = warp; j < k; j += nw) {
    const B* q = Q + (int64_t)j * ldq + base;
    double s0 = 0.0, s1 = 0.0;
    int i = lane;
    for (; i + 32 < n4; i += 64) {
      const float4 a = ld_q4(q, i), b = ld_q4(q, i + 32), x = w4[i], y = w4[i + 32];
      s0 += (double)a.x * x.x + (double)a.y * x.y + (double)a.z * x.z + (double)a.w * x.w;
      s1 += (double)b.x * y.x + (double)b.y * y.y + (double)b.z * y.z + (double)b.w * y.w;
    }
    for (; i < n4; i += 32) {
      const float4 a = ld_q4(q, i), x = w4[i];
      s0 += (double)a.x * x.x + (double)a.y * x.y + (double)a.z * x.z + (double)a.w * x.w;
    }
    const double s = warp_sum_d(s0 + s1);
    if (lane == 0) part_row[j] = s;
  }
}

// partial c_j = Q[j, chunk] . w[chunk] for all j < k
template <class B>
__global__ void __launch_bounds__(kRThreads) k_reorth_dots(const B* __restrict__ Q, int64_t ldq, int k,
                                                           const float* __restrict__ w, int64_t n,
                                                           double* __restrict__ part) {
  __shared__ __align__(16) float ws[kReorthChunk];
  const int64_t base = (int64_t)blockIdx.x * kReorthChunk;
  const int len = (int)(n - base < (int64_t)kReorthChunk ? n - base : (int64_t)kReorthChunk);
  const float4* w4 = reinterpret_cast<const float4*>(w + base);
  for (int i = threadIdx.x; i < len / 4; i += blockDim.x) reinterpret_cast<float4*>(ws)[i] = w4[i];
  __syncthreads();
  chunk_dots(Q, ldq, k, base, len, ws, part + (int64_t)blockIdx.x * k);
}

// w[chunk] -= sum_j c_j Q[j, chunk]; then optionally the next CGS pass's partial dots of the
// updated chunk (the Q chunk was just streamed, so the re-read mostly hits L2) and/or the
// partial ||w||^2
template <class B>
__global__ void __launch_bounds__(kRThreads) k_reorth_update(const B* __restrict__ Q, int64_t ldq, int k,
                                                             const double* __restrict__ c, float* __restrict__ w,
                                                             int64_t n, double* __restrict__ part_dots,
                                                             double* __restrict__ part_norm) {
  extern __shared__ double cs[];
  __shared__ __align__(16) float ws[kReorthChunk];
  for (int j = threadIdx.x; j < k; j += blockDim.x) cs[j] = c[j];
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kReorthChunk;
  const int len = (int)(n - base < (int64_t)kReorthChunk ? n - base : (int64_t)kReorthChunk);
  const int n4 = len / 4;
  double acc[kRGroups][4];
#pragma unroll
  for (int gi = 0; gi < kRGroups; ++gi) acc[gi][0] = acc[gi][1] = acc[gi][2] = acc[gi][3] = 0.0;
  for (int j = 0; j < k; ++j) {
    const double cj = cs[j];
    const B* qrow = Q + (int64_t)j * ldq + base;
#pragma unroll
    for (int gi = 0; gi < kRGroups; ++gi) {
      const int i4 = threadIdx.x + gi * kRThreads;
      if (i4 < n4) {
        const float4 q = ld_q4(qrow, i4);
        acc[gi][0] += cj * q.x; acc[gi][1] += cj * q.y; acc[gi][2] += cj * q.z; acc[gi][3] += cj * q.w;
      }
    }
  }
  double s = 0.0;
  float4* wg = reinterpret_cast<float4*>(w + base);
#pragma unroll
  for (int gi = 0; gi < kRGroups; ++gi) {
    const int i4 = threadIdx.x + gi * kRThreads;
    if (i4 < n4) {
      const float4 o = wg[i4];
      float4 v;
      v.x = (float)((double)o.x - acc[gi][0]);
      v.y = (float)((double)o.y - acc[gi][1]);
      v.z = (float)((double)o.z - acc[gi][2]);
      v.w = (float)((double)o.w - acc[gi][3]);
      wg[i4] = v;
      reinterpret_cast<float4*>(ws)[i4] = v;
      s += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
    }
  }
  if (part_norm) {
    s = block_sum_d(s);
    if (threadIdx.x == 0) part_norm[blockIdx.x] = s;
  }
  if (part_dots) {
    __syncthreads();
    chunk_dots(Q, ldq, k, base, len, ws, part_dots + (int64_t)blockIdx.x * k);
  }
}

// partial c_j = Q[j, chunk] . w[chunk] and g_j = Q[j, chunk] . q[chunk] for all j < k (one pass
// over Q for both; part rows hold [c_0 .. c_{k-1}, g_0 .. g_{k-1}])
template <class B>
__global__ void __launch_bounds__(kRThreads) k_reorth_dots2(const B* __restrict__ Q, int64_t ldq, int k,
                                                            const float* __restrict__ w,
                                                            const float* __restrict__ q, int64_t n,
                                                            double* __restrict__ part) {
  __shared__ __align__(16) float ws[kReorthChunk];
  __shared__ __align__(16) float qs[kReorthChunk];
  const int64_t base = (int64_t)blockIdx.x * kReorthChunk;
  const int len = (int)(n - base < (int64_t)kReorthChunk ? n - base : (int64_t)kReorthChunk);
  for (int i = threadIdx.x; i < len / 4; i += blockDim.x) {
    reinterpret_cast<float4*>(ws)[i] = reinterpret_cast<const float4*>(w + base)[i];
    reinterpret_cast<float4*>(qs)[i] = reinterpret_cast<const float4*>(q + base)[i];
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int n4 = len / 4;
  double* prow = part + (int64_t)blockIdx.x * 2 * k;
  for (int j = warp; j < k; j += nw) {
    const B* qr = Q + (int64_t)j * ldq + base;
    double s0 = 0.0, s1 = 0.0;
    for (int i = lane; i < n4; i += 32) {
      const float4 a = ld_q4(qr, i);
      const float4 x = reinterpret_cast<const float4*>(ws)[i], y = reinterpret_cast<const float4*>(qs)[i];
      s0 += (double)a.x * x.x + (double)a.y * x.y + (double)a.z * x.z + (double)a.w * x.w;
      s1 += (double)a.x * y.x + (double)a.y * y.y + (double)a.z * y.z + (double)a.w * y.w;
    }
    s0 = warp_sum_d(s0);
    s1 = warp_sum_d(s1);
    if (lane == 0) {
      prow[j] = s0;
      prow[k + j] = s1;
    }
  }
}

// Gram step of the two-pass CGS2 (one block): with c1 = Q^T w and g = Q^T q_k (slot ks) from
// k_reorth_dots2, set G[ks][.] = G[.][ks] = g, alpha = c1[ks], and coef = c1 + (c1 - G c1), the sum
// of the two classical Gram-Schmidt passes' coefficients (the second pass's Q^T (w - Q c1) equals
// c1 - G c1 in exact arithmetic), in a fixed summation order.
__global__ void k_gram_coef(const double* __restrict__ cg, int k, int ks, double* __restrict__ G, int ldg,
                            double* __restrict__ coef, double* __restrict__ alpha) {
  extern __shared__ double c1s[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    c1s[j] = cg[j];
    G[(int64_t)ks * ldg + j] = cg[k + j];
    G[(int64_t)j * ldg + ks] = cg[k + j];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double gc = 0.0;
    for (int i = 0; i < k; ++i) gc += G[(int64_t)j * ldg + i] * c1s[i];
    coef[j] = c1s[j] + (c1s[j] - gc);
  }
  if (threadIdx.x == 0) *alpha = c1s[ks];
}

// beta_{k+1} = sqrt(||w||^2) into the recurrence's device scalar and the step history
__global__ void k_step_beta(const double* __restrict__ sumsq, double* __restrict__ beta, double* __restrict__ hist) {
  const double b = sqrt(fmax(*sumsq, 0.0));
  *beta = b;
  *hist = b;
}

// bf16 basis store (R19): q = bf16_RNE(x / sqrt(*sumsq)) (or x * mul when sumsq is
// null: the probe), rounded once from fp64; the fp32 working copy holds the stored value exactly
__global__ void k_store_bf16(const float* __restrict__ x, const double* __restrict__ sumsq, double mul,
                             __nv_bfloat16* __restrict__ row, float* __restrict__ qf, int64_t n) {
  const double beta = sumsq ? sqrt(*sumsq) : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = sumsq ? (double)x[i] / beta : (double)x[i] * mul;
    const __nv_bfloat16 r = __double2bfloat16(v);
    row[i] = r;
    qf[i] = __bfloat162float(r);
  }
}

__global__ void k_dot(const float* __restrict__ a, const float* __restrict__ b, int64_t n, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += (double)a[i] * (double)b[i];
  s = block_sum_d(s);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// y = a x + b y
__global__ void k_axpby(float* __restrict__ y, const float* __restrict__ x, double a, double b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (float)(a * (double)x[i] + b * (double)y[i]);
}

// out = v on [lo, hi), 0 elsewhere
__global__ void k_mask_range(const float* __restrict__ v, float* __restrict__ out, int64_t lo, int64_t hi, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (i >= lo && i < hi) ? v[i] : 0.0f;
}

// over [lo, hi): sum (a-b)^2, a.a, a.b, b.b  -> part[4 * block + j]
__global__ void k_cmp4(const float* __restrict__ a, const float* __restrict__ b, int64_t lo, int64_t hi,
                       double* __restrict__ part) {
  double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a[i], y = b[i];
    s0 += (x - y) * (x - y);
    s1 += x * x;
    s2 += x * y;
    s3 += y * y;
  }
  s0 = block_sum_d(s0);
  s1 = block_sum_d(s1);
  s2 = block_sum_d(s2);
  s3 = block_sum_d(s3);
  if (threadIdx.x == 0) {
    part[4 * blockIdx.x + 0] = s0;
    part[4 * blockIdx.x + 1] = s1;
    part[4 * blockIdx.x + 2] = s2;
    part[4 * blockIdx.x + 3] = s3;
  }
}

__global__ void k_nonfinite(const float* __restrict__ x, int64_t n, int* flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) bad = 1;
  if (bad) atomicOr(flag, 1);
}

}  // namespace

#define VLAUNCH(cls, flops, bytes, grid, block, smem, kernel, ...) \
  do {                                                           \
    LaunchScope scope_(L.prof, cls, L.stream, flops, bytes);     \
    kernel<<<grid, block, smem, L.stream>>>(__VA_ARGS__);        \
    SLQ_CUDA(cudaGetLastError());                                \
    ++*L.launches;                                               \
  } while (0)

int vec_nblocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kThreads * 4), 148 * 4));
}

void probe_fill(const Launch& L, float* q, int64_t n, const UnitDev* units, int nu, uint64_t seed, double inv_sqrt_P) {
  const uint64_t key = [](uint64_t x) {  // host splitmix64(seed)
    x += 0x9E3779B97F4A7C15ull;
    uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }(seed);
  VLAUNCH(KC_VEC, 0, 4.0 * n, vec_nblocks(n), kThreads, 0, k_probe, q, n, units, nu, key, inv_sqrt_P);
}

template <class T>
void perturb(const Launch& L, const float* theta, const float* v, float eta, T* plus, T* minus, int64_t n) {
  VLAUNCH(KC_PERTURB, 4.0 * n, (8.0 + 2.0 * sizeof(T)) * n, vec_nblocks(n), kThreads, 0, k_perturb<T>, theta, v, eta,
          plus, minus, n);
}

void perturb_exact(const Launch& L, const float* theta, const float* v, double eta, double* plus, double* minus,
                   int64_t n) {
  VLAUNCH(KC_PERTURB, 3.0 * n, 24.0 * n, vec_nblocks(n), kThreads, 0, k_perturb_exact, theta, v, eta, plus, minus,
          n);
}

template <class T>
void perturb_lanczos(const Launch& L, bool exact, const float* theta, const float* w_raw, const float* q_prev,
                     double alpha_prev, double beta_k, double eps, float* q_out, T* plus, T* minus, int64_t n) {
  const double inv_beta = 1.0 / beta_k;
  const double bytes = (16.0 + 2.0 * sizeof(T)) * n;  // theta, w_raw, q_prev in; q_k, theta+- out
  if (exact && sizeof(T) == 8) {
    VLAUNCH(KC_PERTURB, 6.0 * n, bytes, vec_nblocks(n), kThreads, 0, (k_perturb_lanczos<T, true>), theta, w_raw,
            q_prev, alpha_prev, inv_beta, eps, (float)eps, q_out, plus, minus, n);
  } else {
    VLAUNCH(KC_PERTURB, 6.0 * n, bytes, vec_nblocks(n), kThreads, 0, (k_perturb_lanczos<T, false>), theta, w_raw,
            q_prev, alpha_prev, inv_beta, eps, (float)eps, q_out, plus, minus, n);
  }
}

template <class T>
void fd_partials3(const Launch& L, const T* gp, const T* gm, double inv2eta, double beta_k, const float* q_prev,
                  const float* q_k, float* w, int64_t n, double* part) {
  const double bytes = (2.0 * sizeof(T) + 8.0 + (q_prev ? 4.0 : 0.0)) * n;
  VLAUNCH(KC_FD, 8.0 * n, bytes, vec_nblocks(n), kThreads, 0, k_fd_partials3<T>, gp, gm, inv2eta, beta_k, q_prev,
          q_k, w, n, part);
}

void sumsq_partials(const Launch& L, const float* x, int64_t n, double* part) {
  VLAUNCH(KC_VEC, 2.0 * n, 4.0 * n, vec_nblocks(n), kThreads, 0, k_sumsq, x, n, part);
}

template <class T>
void fd_w(const Launch& L, const T* gp, const T* gm, double inv2eta, const double* beta_k, const float* q_prev,
          float* w, const float* q_k, int64_t n, double* part) {
  const double bytes = (2.0 * sizeof(T) + 4.0 + (beta_k ? 4.0 : 0.0) + (part ? 4.0 : 0.0)) * n;
  VLAUNCH(KC_FD, 4.0 * n, bytes, vec_nblocks(n), kThreads, 0, k_fd_w<T>, gp, gm, inv2eta, beta_k, q_prev, w, q_k, n,
          part);
}

template <class T>
void fd_out(const Launch& L, const T* gp, const T* gm, double inv2eta, float* out, int64_t n, int* nonfinite) {
  VLAUNCH(KC_FD, 2.0 * n, (2.0 * sizeof(T) + 4.0) * n, vec_nblocks(n), kThreads, 0, k_fd_out<T>, gp, gm, inv2eta,
          out, n, nonfinite);
}

template <class T>
void to_f32(const Launch& L, const T* g, float* out, int64_t n) {
  VLAUNCH(KC_VEC, 0, (sizeof(T) + 4.0) * n, vec_nblocks(n), kThreads, 0, k_to_f32<T>, g, out, n);
}

void reduce_partials(const Launch& L, const double* part, int nb, int k, double* out) {
  if (k == 0) return;
  VLAUNCH(KC_VEC, 0, 8.0 * nb * k, k, 256, 0, k_reduce_partials, part, nb, k, out);
}

void axpy_dev(const Launch& L, float* w, const float* q, const double* coef, double sign, int64_t n, double* part) {
  VLAUNCH(KC_VEC, 2.0 * n, 12.0 * n, vec_nblocks(n), kThreads, 0, k_axpy, w, q, coef, sign, n, part);
}

void scale_by_inv_sqrt(const Launch& L, const float* w, const double* sumsq, float* q, int64_t n) {
  VLAUNCH(KC_VEC, 1.0 * n, 8.0 * n, vec_nblocks(n), kThreads, 0, k_scale_inv_sqrt, w, sumsq, q, n);
}

int reorth_nblocks(int64_t n) { return (int)std::max<int64_t>(1, ceil_div(n, kReorthChunk)); }

template <class B>
void reorth_dots(const Launch& L, const B* Q, int64_t ldq, int k, const float* w, int64_t n, double* part) {
  SLQ_CHECK_ARG(n % 4 == 0 && ldq % 4 == 0, "reorth needs float4-aligned shards");
  VLAUNCH(KC_REORTH, 2.0 * k * n, (sizeof(B) * (double)k + 4.0) * n, reorth_nblocks(n), kRThreads, 0,
          k_reorth_dots<B>, Q, ldq, k, w, n, part);
}

template <class B>
void reorth_update(const Launch& L, const B* Q, int64_t ldq, int k, const double* c, float* w, int64_t n,
                   double* part_dots, double* part_norm) {
  SLQ_CHECK_ARG(n % 4 == 0 && ldq % 4 == 0, "reorth needs float4-aligned shards");
  // algorithmic bytes: Q once from HBM (the fused dots re-read is the L2-resident chunk) + w r/w
  VLAUNCH(KC_REORTH, (part_dots ? 4.0 : 2.0) * k * n, (sizeof(B) * (double)k + 8.0) * n, reorth_nblocks(n),
          kRThreads, sizeof(double) * k, k_reorth_update<B>, Q, ldq, k, c, w, n, part_dots, part_norm);
}

template <class B>
void reorth_dots2(const Launch& L, const B* Q, int64_t ldq, int k, const float* w, const float* q, int64_t n,
                  double* part) {
  SLQ_CHECK_ARG(n % 4 == 0 && ldq % 4 == 0, "reorth needs float4-aligned shards");
  VLAUNCH(KC_REORTH, 4.0 * k * n, (sizeof(B) * (double)k + 8.0) * n, reorth_nblocks(n), kRThreads, 0,
          k_reorth_dots2<B>, Q, ldq, k, w, q, n, part);
}
template void reorth_dots2<float>(const Launch&, const float*, int64_t, int, const float*, const float*, int64_t,
                                  double*);
template void reorth_dots2<__nv_bfloat16>(const Launch&, const __nv_bfloat16*, int64_t, int, const float*,
                                          const float*, int64_t, double*);

void step_beta(const Launch& L, const double* sumsq, double* beta, double* hist) {
  VLAUNCH(KC_VEC, 1.0, 24.0, 1, 1, 0, k_step_beta, sumsq, beta, hist);
}

void gram_coef(const Launch& L, const double* cg, int k, int ks, double* G, int ldg, double* coef, double* alpha) {
  VLAUNCH(KC_REORTH, 2.0 * k * k, 8.0 * k * k, 1, 128, sizeof(double) * k, k_gram_coef, cg, k, ks, G, ldg, coef,
          alpha);
}

template void reorth_dots<float>(const Launch&, const float*, int64_t, int, const float*, int64_t, double*);
template void reorth_dots<__nv_bfloat16>(const Launch&, const __nv_bfloat16*, int64_t, int, const float*, int64_t,
                                         double*);
template void reorth_update<float>(const Launch&, const float*, int64_t, int, const double*, float*, int64_t,
                                   double*, double*);
template void reorth_update<__nv_bfloat16>(const Launch&, const __nv_bfloat16*, int64_t, int, const double*, float*,
                                           int64_t, double*, double*);

void store_bf16(const Launch& L, const float* x, const double* sumsq, double mul, __nv_bfloat16* row, float* qf,
                int64_t n) {
  VLAUNCH(KC_VEC, 1.0 * n, 10.0 * n, vec_nblocks(n), kThreads, 0, k_store_bf16, x, sumsq, mul, row, qf, n);
}

void dot_partials(const Launch& L, const float* a, const float* b, int64_t n, double* part) {
  VLAUNCH(KC_VEC, 2.0 * n, 8.0 * n, vec_nblocks(n), kThreads, 0, k_dot, a, b, n, part);
}

void axpby(const Launch& L, float* y, const float* x, double a, double b, int64_t n) {
  VLAUNCH(KC_VEC, 3.0 * n, 12.0 * n, vec_nblocks(n), kThreads, 0, k_axpby, y, x, a, b, n);
}

void mask_range(const Launch& L, const float* v, float* out, int64_t lo, int64_t hi, int64_t n) {
  VLAUNCH(KC_VEC, 0, 8.0 * n, vec_nblocks(n), kThreads, 0, k_mask_range, v, out, lo, hi, n);
}

int cmp4_partials(const Launch& L, const float* a, const float* b, int64_t lo, int64_t hi, double* part) {
  const int nb = vec_nblocks(std::max<int64_t>(hi - lo, 1));
  VLAUNCH(KC_VEC, 8.0 * (hi - lo), 8.0 * (hi - lo), nb, kThreads, 0, k_cmp4, a, b, lo, hi, part);
  return nb;
}

void nonfinite_check(const Launch& L, const float* x, int64_t n, int* flag) {
  VLAUNCH(KC_VEC, 0, 4.0 * n, vec_nblocks(n), kThreads, 0, k_nonfinite, x, n, flag);
}

#define VINST(T)                                                                                              \
  template void perturb<T>(const Launch&, const float*, const float*, float, T*, T*, int64_t);                \
  template void fd_w<T>(const Launch&, const T*, const T*, double, const double*, const float*, float*,       \
                        const float*, int64_t, double*);                                                      \
  template void fd_out<T>(const Launch&, const T*, const T*, double, float*, int64_t, int*);                  \
  template void to_f32<T>(const Launch&, const T*, float*, int64_t);                                          \
  template void perturb_lanczos<T>(const Launch&, bool, const float*, const float*, const float*, double,     \
                                   double, double, float*, T*, T*, int64_t);                                  \
  template void fd_partials3<T>(const Launch&, const T*, const T*, double, double, const float*, const float*, \
                                float*, int64_t, double*);
VINST(double)
VINST(float)

}  // namespace slq
