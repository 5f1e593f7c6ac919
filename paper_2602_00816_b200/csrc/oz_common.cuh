// Device helpers of the Ozaki INT8 digit scheme shared by the GEMM (oz_gemm.cu) and the attention
// path (oz_attn.cu): row / column exponents, the truncated base-128 digits, and the exact
// int32 -> fp64 conversions of the epilogue.  (DESIGN.md §5 "Ozaki INT8 GEMM".)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace slq {
namespace oz {

// exponent marker of a row / column holding a NaN or an infinity: the slicing cannot represent it,
// so the epilogue scales that output row / column by NaN (non-finite inputs give non-finite
// outputs, as in the DMMA path; the loss then fails the SLQ_ENUMERIC check).  It is the
// largest int, so it survives the max over partial exponents.
constexpr int kExNaN = 0x7fffffff;
constexpr int kExNone = (int)0x80808080;  // "no nonzero element" marker of a partial exponent

// 2^e as a double (e within the normal range), built from the exponent bits
__device__ __forceinline__ double exp2i(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ double scale_of(int e) { return e == kExNaN ? __longlong_as_double(0x7ff8000000000000ll) : exp2i(e); }

// int32 (two's complement bits) -> double, exactly, with one integer op and one fp64 add (the
// I2F.F64 conversion is a slow-path instruction): 2^52 + 2^31 + x has x + 2^31 in its low word
__device__ __forceinline__ double i2d(uint32_t x) {
  return __hiloint2double(0x43300000, (int)(x ^ 0x80000000u)) - 4503601774854144.0;
}

// !(|x| <= DBL_MAX): NaN or +-inf
__device__ __forceinline__ bool nonfinite(double x) { return !(fabs(x) <= 1.7976931348623157e308); }

__device__ __forceinline__ int exp_of(double mx, bool nf = false) {
  if (nf) return kExNaN;
  if (!(mx > 0.0)) return 0;
  int e;
  frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)  ->  mx < 2^e
  return e;
}

// The S digits of x for row exponent e (|x| < 2^e): the truncated base-128 expansion of x 2^-e,
// d_p = trunc(128 r_p), r_{p+1} = 128 r_p - d_p.  Computed exactly in integers:
// Q = trunc(x 2^(7S - e)) (an exact power-of-two scaling, |Q| < 2^(7S)), d_p = sign(x) *
// ((|Q| >> 7 (S - 1 - p)) & 127) -- the same digits as the fp64 recurrence.
template <int S>
__device__ __forceinline__ void digits(double x, int e, int8_t* d) {
  const long long q = __double2ll_rz(x * __longlong_as_double((long long)(7 * S - e + 1023) << 52));
  const long long mag = q < 0 ? -q : q;
#pragma unroll
  for (int p = 0; p < S; ++p) {
    const int v = (int)((mag >> (7 * (S - 1 - p))) & 127);
    d[p] = (int8_t)(q < 0 ? -v : v);
  }
}

// The S digit planes of 4 consecutive values packed into S words (byte k of w[p] = digit p of x[k],
// two's complement): the magnitudes' digits by shifts, the signs applied to all four bytes at once
// (per-byte negation (b ^ 0xff) + 1 with __vadd4, no carries between bytes).  Same digits as digits<S>.
template <int S>
__device__ __forceinline__ void digits4(const double* x, int e, uint32_t* w) {
  const double sc = __longlong_as_double((long long)(7 * S - e + 1023) << 52);
  unsigned long long mag[4];
  uint32_t neg = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long q = __double2ll_rz(x[k] * sc);
    neg |= (q < 0 ? 0xffu : 0u) << (8 * k);
    mag[k] = (unsigned long long)(q < 0 ? -q : q);
  }
#pragma unroll
  for (int p = 0; p < S; ++p) {
    uint32_t v = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) v |= (uint32_t)((mag[k] >> (7 * (S - 1 - p))) & 127u) << (8 * k);
    w[p] = __vadd4(v ^ neg, neg & 0x01010101u);
  }
}

}  // namespace oz
}  // namespace slq
