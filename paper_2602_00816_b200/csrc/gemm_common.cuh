// Shared device helpers of the GEMM kernels: epilogues, batch addressing, split-K reduce.
#pragma once
#include <cuda_runtime.h>

#include "kernels.h"

namespace slq {
namespace gemm_detail {


__device__ __forceinline__ double dtanh_(double x) { return tanh(x); }
__device__ __forceinline__ float dtanh_(float x) { return tanhf(x); }

template <class T>
__device__ __forceinline__ T gelu_tanh(T u) {
  const T c = T(0.7978845608028654);  // sqrt(2/pi)
  T t = dtanh_(c * (u + T(0.044715) * u * u * u));
  return T(0.5) * u * (T(1) + t);
}

template <class T>
__device__ __forceinline__ T gelu_tanh_grad(T u) {
  const T c = T(0.7978845608028654);
  T t = dtanh_(c * (u + T(0.044715) * u * u * u));
  return T(0.5) * (T(1) + t) + T(0.5) * u * (T(1) - t * t) * c * (T(1) + T(3) * T(0.044715) * u * u);
}

__device__ __forceinline__ int64_t boff(const BatchOff& o, int z) {
  return (int64_t)(z / o.div) * o.outer + (int64_t)((z % o.div) / o.rep) * o.inner;
}

template <class T>
__device__ __forceinline__ void epilogue_store(const GemmArgs<T>& p, T* C, int m, int n, T acc) {
  T v = p.alpha * acc;
  if (p.bias) v += p.bias[n];
  if (p.resid) v += p.resid[(int64_t)m * p.ldr + n];
  T out;
  switch (p.act) {
    case ACT_GELU:
      p.C2[(int64_t)m * p.ldc2 + n] = v;
      out = gelu_tanh(v);
      break;
    case ACT_TANH:
      out = dtanh_(v);
      break;
    case ACT_DGELU:
      out = v * gelu_tanh_grad(p.aux[(int64_t)m * p.ldaux + n]);
      break;
    case ACT_DTANH: {
      T h = p.aux[(int64_t)m * p.ldaux + n];
      out = v * (T(1) - h * h);
      break;
    }
    default:
      out = v;
  }
  T* dst = C + (int64_t)m * p.ldc + n;
  if (p.accumulate)
    *dst += out;
  else
    *dst = out;
}

// two consecutive columns (n, n + 1) of row m; `vec`: every row pitch involved is even and every
// base 16-byte aligned, so the pair is one 16-byte access per array
__device__ __forceinline__ double epi_act(const GemmArgs<double>& p, double v, double aux) {
  switch (p.act) {
    case ACT_GELU: return gelu_tanh(v);
    case ACT_TANH: return dtanh_(v);
    case ACT_DGELU: return v * gelu_tanh_grad(aux);
    case ACT_DTANH: return v * (1.0 - aux * aux);
    default: return v;
  }
}
__device__ __forceinline__ void epilogue_store2(const GemmArgs<double>& p, double* C, int m, int n, double a0,
                                                double a1, bool vec) {
  const int64_t m64 = m;
  double2 b = make_double2(0.0, 0.0), r = b, x = b, c = b;
  if (vec) {
    if (p.bias) b = *reinterpret_cast<const double2*>(p.bias + n);
    if (p.resid) r = *reinterpret_cast<const double2*>(p.resid + m64 * p.ldr + n);
    if (p.aux) x = *reinterpret_cast<const double2*>(p.aux + m64 * p.ldaux + n);
    if (p.accumulate) c = *reinterpret_cast<const double2*>(C + m64 * p.ldc + n);
  } else {
    if (p.bias) b = make_double2(p.bias[n], p.bias[n + 1]);
    if (p.resid) r = make_double2(p.resid[m64 * p.ldr + n], p.resid[m64 * p.ldr + n + 1]);
    if (p.aux) x = make_double2(p.aux[m64 * p.ldaux + n], p.aux[m64 * p.ldaux + n + 1]);
    if (p.accumulate) c = make_double2(C[m64 * p.ldc + n], C[m64 * p.ldc + n + 1]);
  }
  const double v0 = p.alpha * a0 + b.x + r.x, v1 = p.alpha * a1 + b.y + r.y;
  if (p.act == ACT_GELU) {
    if (vec) *reinterpret_cast<double2*>(p.C2 + m64 * p.ldc2 + n) = make_double2(v0, v1);
    else { p.C2[m64 * p.ldc2 + n] = v0; p.C2[m64 * p.ldc2 + n + 1] = v1; }
  }
  double o0 = epi_act(p, v0, x.x), o1 = epi_act(p, v1, x.y);
  if (p.accumulate) { o0 += c.x; o1 += c.y; }
  if (vec) *reinterpret_cast<double2*>(C + m64 * p.ldc + n) = make_double2(o0, o1);
  else { C[m64 * p.ldc + n] = o0; C[m64 * p.ldc + n + 1] = o1; }
}

// ws holds the fp32/fp64 partials of batch entry z, split k at ws[(z * splits + k) * M * N]
// (row-major M x N); the sum over k in fixed order goes through the regular epilogue into C(z)
template <class T>
__global__ void splitk_reduce(GemmArgs<T> p, int splits, const T* __restrict__ ws) {
  const int64_t mn = (int64_t)p.M * p.N, tot = mn * p.batch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const int z = (int)(i / mn);
    const int64_t e = i - z * mn;
    const T* w = ws + (int64_t)z * splits * mn + e;
    T s = T(0);
    for (int k = 0; k < splits; ++k) s += w[k * mn];
    epilogue_store(p, p.C + boff(p.offC, z), (int)(e / p.N), (int)(e % p.N), s);
  }
}

}  // namespace gemm_detail
}  // namespace slq
