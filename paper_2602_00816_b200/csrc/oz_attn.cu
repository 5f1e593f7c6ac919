// Causal multi-head attention of the FP64_OZ passes on the tcgen05 INT8 tensor cores.
//
// The six contractions of one attention layer (P:391-405 counts them in T_grad) -- S = Q K^T,
// O = P V in the forward; dP = dO V^T, dV = P^T dO, dQ = dS K, dK = dS^T Q in the backward -- run
// as batched Ozaki GEMMs (gemm_oz_planes: exact INT8 digit products, one launch per contraction,
// causal tiles skipped or k-clipped) instead of FP64 DMMA.  Their operands are sliced here:
//   * Q, K, V, dO rows (hd contiguous values per (head, position)): one warp per row;
//   * K, V, dO', Q' columns (the B operands whose k index is the position): one CTA per head and
//     32 columns, transposed through shared memory;
//   * P and dS: emitted by the softmax kernels themselves -- the forward writes P (fp64, for the
//     backward) and its row digits; the backward writes the digits of dS (row-major, for dQ) and,
//     transposed, of P and dS (for dV and dK).  No fp64 dS is ever stored.
// The transposed P / dS operands keep their row exponents: P^T's digits are those of P_qk 2^-r_q,
// and the factor 2^r_q moves into the other operand, dV = sum_q (P_qk 2^-r_q) (2^r_q dO_q) (same for
// dK with dS's exponents e_q and Q) -- an exact power-of-two rescaling, so the only error is the
// dropped digits of the Ozaki scheme (oz_gemm.cu header), bounded relative to the rescaled operand.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>

#include "common.h"
#include "kernels.h"
#include "oz_common.cuh"

namespace slq {
namespace oz {

__device__ __forceinline__ double nanmax(double a, double b) { return (b > a || b != b) ? b : a; }
__device__ __forceinline__ double warp_nanmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_fmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_add(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- head rows: row (zb, t) = X[(b T + t) ld + col0 + h hd + 0 .. hd-1], zb = b heads + h ----
struct RowJob {
  const double* X;
  int64_t ld, col0;
  int heads, T, hd, nb;
  int8_t* out;  // [S][nb][T][hd]
  int* ex;      // [nb][T]
  int blocks0;
};
struct RowJobs {
  RowJob j[2];
  int n;
};

constexpr int kRowsPerWarp = 4;

// hd in {32, 64, 128}: each lane owns 4 consecutive values (two 16-byte loads, one packed word per
// digit plane), LPR = hd / 4 lanes per row, 32 / LPR rows per warp pass, kRowsPerWarp rows per warp
// (all loads issued before the first reduction); other hd (multiples of 32): vpl = hd / 32 values
// per lane, one row per warp pass
template <int S>
__global__ void __launch_bounds__(256) k_att_rows(const __grid_constant__ RowJobs js) {
  const RowJob& jb = (js.n > 1 && (int)blockIdx.x >= js.j[1].blocks0) ? js.j[1] : js.j[0];
  // 32-bit row arithmetic (nb T < 2^31; 64-bit divisions made this kernel integer-bound)
  const int r0 = ((blockIdx.x - jb.blocks0) * 8 + threadIdx.x / 32) * kRowsPerWarp;
  const int lane = threadIdx.x % 32;
  const int nrows = jb.nb * jb.T;
  if (r0 >= nrows) return;
  // the warp's rows are consecutive positions of one head (T % kRowsPerWarp == 0)
  const int zb = r0 / jb.T, t0 = r0 - zb * jb.T;
  const int b = zb / jb.heads, h = zb - b * jb.heads;
  const double* xb = jb.X + ((int64_t)b * jb.T + t0) * jb.ld + jb.col0 + (int64_t)h * jb.hd;
  const int64_t plane = (int64_t)nrows * jb.hd;
  if (jb.hd == 32 || jb.hd == 64 || jb.hd == 128) {
    const int lpr = jb.hd / 4, rpp = 32 / lpr;  // lanes per row, rows per pass
    const int sub = lane / lpr, col = 4 * (lane % lpr);
    double v[kRowsPerWarp][4];
#pragma unroll
    for (int it = 0; it < kRowsPerWarp; ++it) {
      const int rr = it * rpp + sub;  // (rows beyond kRowsPerWarp: idle lanes)
      if (rr < kRowsPerWarp) {
        const double* x = xb + (int64_t)rr * jb.ld + col;
        const double2 a = *reinterpret_cast<const double2*>(x);
        const double2 c = *reinterpret_cast<const double2*>(x + 2);
        v[it][0] = a.x; v[it][1] = a.y; v[it][2] = c.x; v[it][3] = c.y;
      } else {
        v[it][0] = v[it][1] = v[it][2] = v[it][3] = 0.0;
      }
      if ((it + 1) * rpp >= kRowsPerWarp) break;
    }
#pragma unroll
    for (int it = 0; it < kRowsPerWarp; ++it) {
      const int rr = it * rpp + sub;
      double mx = 0.0;
      bool nf = false;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        mx = fmax(mx, fabs(v[it][k]));
        nf |= nonfinite(v[it][k]);
      }
      for (int o = lpr / 2; o > 0; o >>= 1) {  // reduce within the row's lpr lanes
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        nf |= __shfl_xor_sync(0xffffffffu, (int)nf, o) != 0;
      }
      if (rr < kRowsPerWarp) {
        const int r = r0 + rr;
        const int e = exp_of(mx, nf);
        if (lane % lpr == 0) jb.ex[r] = e;
        uint32_t w[S];
        digits4<S>(v[it], nf ? 0 : e, w);
        int8_t* o = jb.out + (int64_t)r * jb.hd + col;
#pragma unroll
        for (int q = 0; q < S; ++q) *reinterpret_cast<uint32_t*>(o + q * plane) = w[q];
      }
      if ((it + 1) * rpp >= kRowsPerWarp) break;
    }
    return;
  }
  const int vpl = jb.hd / 32;  // consecutive values per lane
  xb += lane * vpl;
  double v[kRowsPerWarp][4];
#pragma unroll
  for (int rr = 0; rr < kRowsPerWarp; ++rr) {
    const int r = r0 + rr;
    const double* x = xb + (int64_t)rr * jb.ld - lane * vpl;
#pragma unroll
    for (int i = 0; i < 4; ++i) v[rr][i] = (r < nrows && i < vpl) ? x[lane * vpl + i] : 0.0;
  }
#pragma unroll
  for (int rr = 0; rr < kRowsPerWarp; ++rr) {
    const int64_t r = r0 + rr;
    if (r >= nrows) break;
    double mx = 0.0;
    bool nf = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mx = fmax(mx, fabs(v[rr][i]));
      nf |= nonfinite(v[rr][i]);
    }
    mx = warp_fmax(mx);
    nf = __any_sync(0xffffffffu, nf);
    const int e = exp_of(mx, nf);
    if (lane == 0) jb.ex[r] = e;
    const int ed = nf ? 0 : e;
    int8_t d[4][S];
#pragma unroll
    for (int i = 0; i < 4; ++i) digits<S>(v[rr][i], ed, d[i]);
    int8_t* o = jb.out + r * jb.hd + lane * vpl;
#pragma unroll
    for (int q = 0; q < S; ++q)
      for (int i = 0; i < vpl; ++i) o[q * plane + i] = d[i][q];
  }
}

// ---- head columns, transposed: row (zb, dcol) of the output holds X[t][dcol] 2^pre[zb][t] over
// t = 0 .. T-1 (the B operand of O = P V, dQ, dV, dK); exponent per (zb, dcol) over all t ----
struct ColJob {
  const double* X;
  int64_t ld, col0;
  int heads, T, hd, nb;
  const int* pre;  // [nb][T] power-of-two row pre-scale (nullptr: none)
  int8_t* out;     // [S][nb][hd][T]
  int* ex;         // [nb][hd]
};

// One 512-thread CTA per (head, 8 columns): 8 columns x 64 t-lanes (each warp reads 4 rows x 64 B);
// pass 1 the column maxima (8 loads in flight per thread), pass 2 128-deep t chunks through a
// shared tile, each thread 2 consecutive t of one column (64 threads write a column's 128 bytes)
constexpr int kColW = 8;

template <int S>
__global__ void __launch_bounds__(512) k_att_cols(const __grid_constant__ ColJob jb) {
  __shared__ double tile[128][kColW + 1];
  __shared__ double red[64][kColW + 1];
  __shared__ int es[kColW];
  const int dblk = jb.hd / kColW;
  const int zb = blockIdx.x / dblk, d0 = (blockIdx.x % dblk) * kColW;
  const int b = zb / jb.heads, h = zb % jb.heads;
  const double* x = jb.X + (int64_t)b * jb.T * jb.ld + jb.col0 + (int64_t)h * jb.hd + d0;
  const int* pre = jb.pre ? jb.pre + (int64_t)zb * jb.T : nullptr;
  const int tx = threadIdx.x % kColW, ty = threadIdx.x / kColW;  // column, t-lane (64)
  auto val = [&](int t) {
    const double v = x[(int64_t)t * jb.ld + tx];
    return pre ? v * scale_of(pre[t]) : v;
  };
  double mx = 0.0;
  bool nf = false;
  for (int t0 = 0; t0 < jb.T; t0 += 512) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int t = t0 + ty + 64 * i;
      v[i] = t < jb.T ? val(t) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      mx = fmax(mx, fabs(v[i]));
      nf |= nonfinite(v[i]);
    }
  }
  red[ty][tx] = nf ? __longlong_as_double(0x7ff8000000000000ll) : mx;
  __syncthreads();
  if (threadIdx.x < kColW) {
    double m = 0.0;
    bool bad = false;
    for (int i = 0; i < 64; ++i) {
      bad |= red[i][threadIdx.x] != red[i][threadIdx.x];
      m = fmax(m, red[i][threadIdx.x]);
    }
    const int e = exp_of(m, bad);
    es[threadIdx.x] = e;
    jb.ex[(int64_t)zb * jb.hd + d0 + threadIdx.x] = e;
  }
  __syncthreads();
  const int64_t plane = (int64_t)jb.nb * jb.hd * jb.T;
  const int dd = threadIdx.x / 64, tq = (threadIdx.x % 64) * 2;
  const int ed = es[dd] == kExNaN ? 0 : es[dd];
  int8_t* orow = jb.out + ((int64_t)zb * jb.hd + d0 + dd) * jb.T + tq;
  for (int t0 = 0; t0 < jb.T; t0 += 128) {  // T % 128 == 0
    const double v0 = val(t0 + ty), v1 = val(t0 + ty + 64);
    tile[ty][tx] = v0;
    tile[ty + 64][tx] = v1;
    __syncthreads();
    int8_t d[2][S];
    digits<S>(tile[tq][dd], ed, d[0]);
    digits<S>(tile[tq + 1][dd], ed, d[1]);
#pragma unroll
    for (int q = 0; q < S; ++q)
      *reinterpret_cast<uint16_t*>(orow + q * plane + t0) = (uint16_t)((uint8_t)d[0][q] | ((uint8_t)d[1][q] << 8));
    __syncthreads();
  }
}

// The same output with ONE read of X: the CTA's whole 8-column x T strip is staged in shared memory
// by 8-byte cp.async (16 loads in flight per thread at T = 1024), then the column maxima and the
// digits come from shared memory.  Strip [T][kColW + 1] (padded rows).  T <= 2048.
template <int S>
__global__ void __launch_bounds__(512) k_att_cols1(const __grid_constant__ ColJob jb) {
  extern __shared__ double strip[];  // [T][kColW + 1]
  __shared__ double red[64][kColW + 1];
  __shared__ int es[kColW];
  constexpr int LDS = kColW + 1;
  const int dblk = jb.hd / kColW;
  const int zb = blockIdx.x / dblk, d0 = (blockIdx.x % dblk) * kColW;
  const int b = zb / jb.heads, h = zb % jb.heads;
  const double* x = jb.X + (int64_t)b * jb.T * jb.ld + jb.col0 + (int64_t)h * jb.hd + d0;
  const int* pre = jb.pre ? jb.pre + (int64_t)zb * jb.T : nullptr;
  const int tx = threadIdx.x % kColW, ty = threadIdx.x / kColW;  // column, t-lane (64)
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(strip);
  for (int t = ty; t < jb.T; t += 64)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sb + 8u * (uint32_t)(t * LDS + tx)),
                 "l"(x + (int64_t)t * jb.ld + tx)
                 : "memory");
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  auto val = [&](int t, int c) {
    const double v = strip[t * LDS + c];
    return pre ? v * scale_of(pre[t]) : v;
  };
  double mx = 0.0;
  bool nf = false;
  for (int t = ty; t < jb.T; t += 64) {
    const double v = val(t, tx);
    mx = fmax(mx, fabs(v));
    nf |= nonfinite(v);
  }
  red[ty][tx] = nf ? __longlong_as_double(0x7ff8000000000000ll) : mx;
  __syncthreads();
  if (threadIdx.x < kColW) {
    double m = 0.0;
    bool bad = false;
    for (int i = 0; i < 64; ++i) {
      bad |= red[i][threadIdx.x] != red[i][threadIdx.x];
      m = fmax(m, red[i][threadIdx.x]);
    }
    const int e = exp_of(m, bad);
    es[threadIdx.x] = e;
    jb.ex[(int64_t)zb * jb.hd + d0 + threadIdx.x] = e;
  }
  __syncthreads();
  const int64_t plane = (int64_t)jb.nb * jb.hd * jb.T;
  const int dd = threadIdx.x / 64, tq = (threadIdx.x % 64) * 2;
  const int ed = es[dd] == kExNaN ? 0 : es[dd];
  int8_t* orow = jb.out + ((int64_t)zb * jb.hd + d0 + dd) * jb.T + tq;
  for (int t0 = 0; t0 < jb.T; t0 += 128) {  // T % 128 == 0
    int8_t d[2][S];
    digits<S>(val(t0 + tq, dd), ed, d[0]);
    digits<S>(val(t0 + tq + 1, dd), ed, d[1]);
#pragma unroll
    for (int q = 0; q < S; ++q)
      *reinterpret_cast<uint16_t*>(orow + q * plane + t0) = (uint16_t)((uint8_t)d[0][q] | ((uint8_t)d[1][q] << 8));
  }
}

// ---- forward softmax: S -> P in place (causal, zeros up to the end of the diagonal 128-column
// block, as k_softmax_causal) and P's row digits (row exponent r_q of max_k P_qk = 1 / sum) ----
// one 128-thread block per row (as k_softmax_causal_blk): the row is read once into registers
// (V values per thread, j = tid + 128 i), block reductions for the max and the sum, one write of P
// and of its S digit planes (each warp store covers 32 consecutive bytes of a plane)
template <int S, int V>
__global__ void __launch_bounds__(128) k_att_sm_fwd(double* __restrict__ P, int T, int8_t* __restrict__ out,
                                                    int* __restrict__ ex, int64_t plane) {
  // V values per thread as V / 4 groups of 4 consecutive keys j = 4 (tid + 128 g) + k: 32-byte loads,
  // one packed word per digit plane and group (the byte-per-element stores made this kernel
  // issue-bound)
  constexpr int G = V / 4;
  static_assert(V % 4 == 0, "groups of 4");
  __shared__ double red[4];
  const int row = blockIdx.x;  // (32-bit: rows < 2^31)
  const int q = row - (row / T) * T;
  double* s = P + (int64_t)row * T;
  int8_t* orow = out + (int64_t)row * T;
  const int tid = threadIdx.x, lane = tid % 32, wid = tid / 32;
  double v[V];
  double mx = -INFINITY;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j0 = 4 * (tid + 128 * g);
    if (j0 <= q) {
      const double2 a = *reinterpret_cast<const double2*>(s + j0);
      const double2 b = *reinterpret_cast<const double2*>(s + j0 + 2);
      v[4 * g] = a.x; v[4 * g + 1] = a.y; v[4 * g + 2] = b.x; v[4 * g + 3] = b.y;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (j0 + k > q) v[4 * g + k] = -INFINITY;
      mx = nanmax(mx, v[4 * g + k]);
    }
  }
  mx = warp_nanmax(mx);
  if (lane == 0) red[wid] = mx;
  __syncthreads();
  mx = nanmax(nanmax(red[0], red[1]), nanmax(red[2], red[3]));
  __syncthreads();
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (4 * (tid + 128 * (i / 4)) + (i % 4) <= q) {
      v[i] = exp(v[i] - mx);
      sum += v[i];
    }
  }
  sum = warp_add(sum);
  if (lane == 0) red[wid] = sum;
  __syncthreads();
  const double inv = 1.0 / ((red[0] + red[1]) + (red[2] + red[3]));
  const bool nf = !(inv > 0.0 && inv <= 1.7976931348623157e308);
  const int e = exp_of(inv, nf), ed = nf ? 0 : e;  // max_k P_qk = exp(0) inv = inv < 2^e
  if (tid == 0) ex[row] = e;
  const int jend = min(T, (q / 128 + 1) * 128);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int j0 = 4 * (tid + 128 * g);
    if (j0 < jend) {
      double p[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) p[k] = j0 + k <= q ? v[4 * g + k] * inv : 0.0;
      *reinterpret_cast<double2*>(s + j0) = make_double2(p[0], p[1]);
      *reinterpret_cast<double2*>(s + j0 + 2) = make_double2(p[2], p[3]);
      uint32_t w[S];
      digits4<S>(p, ed, w);
#pragma unroll
      for (int qd = 0; qd < S; ++qd) *reinterpret_cast<uint32_t*>(orow + qd * plane + j0) = w[qd];
    }
  }
}

// ---- backward softmax: dS = P (dP - D), D_q = sum_k P_qk dP_qk, emitted only as digits: dS
// row-major (exponent e_q of max_k |dS_qk|; A of dQ), and transposed [key][query] the digits of
// dS_qk 2^-e_q (A of dK) and of P_qk 2^-r_q (A of dV), r_q the exponent of max_k P_qk ----
// One 512-thread CTA per 32 query rows, two CTAs per SM (the CTAs in flight re-read their rows
// from L2: 2 x 148 x 32 causal rows x 16 B stays below its capacity).  Phase 1: warp w owns rows
// q0 + 2w, q0 + 2w + 1 (D and max P in one sweep, max |dS| in a second; eight loads in flight per
// lane).  Phase 2: 64-key chunks, lane l keys 2l, 2l + 1 of the warp's two rows: P / dP loads and
// dS row digits coalesced; the transposed digits go through [plane][query][key] shared tiles and
// leave as 32-byte rows [key][q0 .. q0 + 31].
template <int S>
__global__ void __launch_bounds__(512, 2) k_att_sm_bwd(const double* __restrict__ P, const double* __restrict__ dP,
                                                       int T, int8_t* __restrict__ pt, int8_t* __restrict__ dsa,
                                                       int8_t* __restrict__ dst, int* __restrict__ exr,
                                                       int* __restrict__ exe, int64_t plane) {
  // chunk width: 128 keys (4 per lane, packed digit words) while the two [S][32][CW] tiles fit the
  // 48 KB of static shared memory, else 64
  constexpr int CW = S <= 5 ? 128 : 64, KPL = CW / 32;
  __shared__ __align__(16) uint8_t tp[S][32][CW];
  __shared__ __align__(16) uint8_t td[S][32][CW];
  const int cpr = T / 32;
  const int64_t zq = blockIdx.x / cpr;
  const int q0 = (blockIdx.x % cpr) * 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // phase 1, the warp's two rows interleaved (16 loads in flight per lane per sweep)
  const int qa = q0 + 2 * warp, qb = qa + 1;  // qb = the longer row
  const double* pr[2] = {P + (zq * T + qa) * (int64_t)T, P + (zq * T + qb) * (int64_t)T};
  const double* gr[2] = {dP + (zq * T + qa) * (int64_t)T, dP + (zq * T + qb) * (int64_t)T};
  // (a NaN / inf in P or dP reaches D or max P: both propagate NaN, so no per-element test)
  double pm[2] = {0.0, 0.0}, Dr[2] = {0.0, 0.0};
  for (int j0 = 0; j0 <= qb; j0 += 128) {
    double a[2][4], c[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int j = j0 + lane + 32 * i;
        const bool in = j <= qa + u;
        a[u][i] = in ? pr[u][j] : 0.0;
        c[u][i] = in ? gr[u][j] : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        pm[u] = nanmax(pm[u], a[u][i]);
        Dr[u] += a[u][i] * c[u][i];
      }
  }
  double dm[2] = {0.0, 0.0};
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    pm[u] = warp_nanmax(pm[u]);
    Dr[u] = warp_add(Dr[u]);
  }
  for (int j0 = 0; j0 <= qb; j0 += 128) {
    double a[2][4], c[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int j = j0 + lane + 32 * i;
        const bool in = j <= qa + u;
        a[u][i] = in ? pr[u][j] : 0.0;
        c[u][i] = in ? gr[u][j] : 0.0;
      }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int i = 0; i < 4; ++i) dm[u] = fmax(dm[u], fabs(a[u][i] * (c[u][i] - Dr[u])));
  }
  int rd[2], ed[2];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    dm[u] = warp_fmax(dm[u]);
    const bool nf = nonfinite(pm[u]) || nonfinite(Dr[u]);
    const int r = exp_of(pm[u], nf), e = exp_of(dm[u], nf);
    if (lane == 0) {
      exr[zq * T + qa + u] = r;
      exe[zq * T + qa + u] = e;
    }
    rd[u] = r == kExNaN ? 0 : r;
    ed[u] = e == kExNaN ? 0 : e;
  }
  const int kend = min(T, (q0 / 128 + 1) * 128);
  for (int c0 = 0; c0 < kend; c0 += CW) {
    const int j = c0 + KPL * lane;
    double pv[2][KPL], gv[2][KPL];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t ro = (zq * T + q0 + 2 * warp + u) * (int64_t)T;
#pragma unroll
      for (int k = 0; k < KPL; k += 2) {
        const double2 a = *reinterpret_cast<const double2*>(P + ro + j + k);
        const double2 c = *reinterpret_cast<const double2*>(dP + ro + j + k);
        pv[u][k] = a.x; pv[u][k + 1] = a.y;
        gv[u][k] = c.x; gv[u][k + 1] = c.y;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int q = q0 + 2 * warp + u;
      double xp[KPL], xs[KPL];
#pragma unroll
      for (int k = 0; k < KPL; ++k) {
        const bool in = j + k <= q;
        xp[k] = in ? pv[u][k] : 0.0;
        xs[k] = in ? pv[u][k] * (gv[u][k] - Dr[u]) : 0.0;
      }
      int8_t* arow = dsa + (zq * T + q) * (int64_t)T;
      if constexpr (KPL == 4) {
        uint32_t ws[S], wp[S];
        digits4<S>(xs, ed[u], ws);
        digits4<S>(xp, rd[u], wp);
#pragma unroll
        for (int qd = 0; qd < S; ++qd) {
          *reinterpret_cast<uint32_t*>(arow + qd * plane + j) = ws[qd];
          *reinterpret_cast<uint32_t*>(&td[qd][2 * warp + u][KPL * lane]) = ws[qd];
          *reinterpret_cast<uint32_t*>(&tp[qd][2 * warp + u][KPL * lane]) = wp[qd];
        }
      } else {
        uint16_t ws[S], wp[S];
#pragma unroll
        for (int qd = 0; qd < S; ++qd) ws[qd] = wp[qd] = 0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          int8_t dgp[S], dgs[S];
          digits<S>(xp[k], rd[u], dgp);
          digits<S>(xs[k], ed[u], dgs);
#pragma unroll
          for (int qd = 0; qd < S; ++qd) {
            ws[qd] |= (uint16_t)((uint8_t)dgs[qd] << (8 * k));
            wp[qd] |= (uint16_t)((uint8_t)dgp[qd] << (8 * k));
          }
        }
#pragma unroll
        for (int qd = 0; qd < S; ++qd) {
          *reinterpret_cast<uint16_t*>(arow + qd * plane + j) = ws[qd];
          *reinterpret_cast<uint16_t*>(&td[qd][2 * warp + u][KPL * lane]) = ws[qd];
          *reinterpret_cast<uint16_t*>(&tp[qd][2 * warp + u][KPL * lane]) = wp[qd];
        }
      }
    }
    __syncthreads();
    // transposed rows: thread (array, plane, key kk) gathers queries q0 .. q0 + 31 of key c0 + kk
    for (int idx = threadIdx.x; idx < 2 * S * CW; idx += 512) {
      const int kk = idx % CW, qd = (idx / CW) % S, arr = idx / (CW * S);
      const uint8_t(*src)[CW] = arr ? td[qd] : tp[qd];
      uint32_t w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        w[u] = (uint32_t)src[4 * u][kk] | ((uint32_t)src[4 * u + 1][kk] << 8) | ((uint32_t)src[4 * u + 2][kk] << 16) |
               ((uint32_t)src[4 * u + 3][kk] << 24);
      int8_t* d = (arr ? dst : pt) + qd * plane + (zq * T + c0 + kk) * (int64_t)T + q0;
      *reinterpret_cast<uint4*>(d) = make_uint4(w[0], w[1], w[2], w[3]);
      *reinterpret_cast<uint4*>(d + 16) = make_uint4(w[4], w[5], w[6], w[7]);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// host side

struct Carve {
  uint8_t* p;
  size_t off = 0;
  template <class X>
  X* take(size_t n) {
    X* r = reinterpret_cast<X*>(p ? p + off : nullptr);
    off += (sizeof(X) * n + 255) & ~(size_t)255;
    return r;
  }
};

struct Bufs {
  // forward
  int8_t *QA, *KB, *PA, *VB;
  int *exQ, *exK, *exP, *exV;
  // backward
  int8_t *DOA, *VR, *PT, *DSA, *DST, *KT, *DOT, *QT;
  int *exDO, *exVR, *exR, *exE, *exKT, *exDOT, *exQT;
  size_t fwd_bytes, bwd_bytes;
};

static Bufs carve(const AttnShape& g, int S, uint8_t* base) {
  const size_t zq = (size_t)g.nseq * g.Hq, zk = (size_t)g.nseq * g.Hkv, T = g.Tn, hd = g.hd;
  Bufs b;
  Carve f{base};
  b.QA = f.take<int8_t>(S * zq * T * hd);
  b.KB = f.take<int8_t>(S * zk * T * hd);
  b.PA = f.take<int8_t>(S * zq * T * T);
  b.VB = f.take<int8_t>(S * zk * hd * T);
  b.exQ = f.take<int>(zq * T);
  b.exK = f.take<int>(zk * T);
  b.exP = f.take<int>(zq * T);
  b.exV = f.take<int>(zk * hd);
  b.fwd_bytes = f.off;
  Carve w{base};
  b.PT = w.take<int8_t>(S * zq * T * T);
  b.DSA = w.take<int8_t>(S * zq * T * T);
  b.DST = w.take<int8_t>(S * zq * T * T);
  b.DOA = w.take<int8_t>(S * zq * T * hd);
  b.VR = w.take<int8_t>(S * zk * T * hd);
  b.KT = w.take<int8_t>(S * zk * hd * T);
  b.DOT = w.take<int8_t>(S * zq * hd * T);
  b.QT = w.take<int8_t>(S * zq * hd * T);
  b.exDO = w.take<int>(zq * T);
  b.exVR = w.take<int>(zk * T);
  b.exR = w.take<int>(zq * T);
  b.exE = w.take<int>(zq * T);
  b.exKT = w.take<int>(zk * hd);
  b.exDOT = w.take<int>(zq * hd);
  b.exQT = w.take<int>(zq * hd);
  b.bwd_bytes = w.off;
  return b;
}

template <int S>
static void launch_rows(const Launch& L, RowJobs js) {
  int nb = 0;
  for (int i = 0; i < js.n; ++i) {
    js.j[i].blocks0 = nb;
    nb += (int)ceil_div((int64_t)js.j[i].nb * js.j[i].T, 8 * kRowsPerWarp);
  }
  if (js.n == 1) js.j[1] = js.j[0];
  double elems = 0;
  for (int i = 0; i < js.n; ++i) elems += (double)js.j[i].nb * js.j[i].T * js.j[i].hd;
  LaunchScope scope(L.prof, KC_OZ_SLICE, L.stream, 0, (8.0 + S) * elems);
  k_att_rows<S><<<nb, 256, 0, L.stream>>>(js);
  SLQ_CUDA(cudaGetLastError());
  ++*L.launches;
}

template <int S>
static void launch_cols(const Launch& L, const ColJob& j) {
  static const bool twopass = getenv("SLQ_OZ_SLICE_TWOPASS") != nullptr;  // A/B switch
  if (!twopass && j.T <= 2048) {
    LaunchScope scope(L.prof, KC_OZ_SLICE, L.stream, 0, (8.0 + S) * (double)j.nb * j.T * j.hd);
    const size_t smem = (size_t)j.T * (kColW + 1) * 8;
    static bool attr = false;
    if (!attr) {
      SLQ_CUDA(cudaFuncSetAttribute(k_att_cols1<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    2048 * (kColW + 1) * 8));
      attr = true;
    }
    k_att_cols1<S><<<j.nb * (j.hd / kColW), 512, smem, L.stream>>>(j);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
    return;
  }
  LaunchScope scope(L.prof, KC_OZ_SLICE, L.stream, 0, (16.0 + S) * (double)j.nb * j.T * j.hd);
  k_att_cols<S><<<j.nb * (j.hd / kColW), 512, 0, L.stream>>>(j);
  SLQ_CUDA(cudaGetLastError());
  ++*L.launches;
}

static BatchOff ident() { return BatchOff{1, 0, 1, 1}; }

template <int S>
static void fwd(const Launch& L, const AttnShape& g, const double* qkv, double* P, double* o) {
  const int zq = g.nseq * g.Hq, zk = g.nseq * g.Hkv, T = g.Tn, hd = g.hd, rep = g.Hq / g.Hkv;
  Bufs b = carve(g, S, (uint8_t*)L.ws->get(attn_oz_ws_bytes(L, g), L.stream));
  const BatchOff kv{g.Hkv, 1, g.Hq, rep};  // q head (b, h) -> kv head (b, h / rep)
  {
    RowJobs js;
    js.n = 2;
    js.j[0] = RowJob{qkv, g.W, g.qo, g.Hq, T, hd, zq, b.QA, b.exQ, 0};
    js.j[1] = RowJob{qkv, g.W, g.ko, g.Hkv, T, hd, zk, b.KB, b.exK, 0};
    launch_rows<S>(L, js);
  }
  {  // S = scale Q K^T (lower tiles only)
    GemmArgs<double> a;
    a.M = T; a.N = T; a.K = hd; a.batch = zq;
    a.C = P; a.ldc = T; a.offC = BatchOff{(int64_t)T * T, 0, 1, 1};
    a.alpha = 1.0 / std::sqrt((double)hd);
    a.tri = TRI_SKIP_UPPER;
    OzPlanes pa, pb;
    pa.d = b.QA; pa.ex = b.exQ; pa.nb = zq; pa.Kp = hd; pa.z = ident();
    pb.d = b.KB; pb.ex = b.exK; pb.nb = zk; pb.Kp = hd; pb.z = kv;
    gemm_oz_planes(L, S, pa, pb, a);
  }
  {
    LaunchScope scope(L.prof, KC_ATTN, L.stream, 0, (16.0 + 8.0 + S) * zq * (T * (T + 128.0) / 2));
    const int64_t rows = (int64_t)zq * T, plane = rows * T;
    if (T <= 512) k_att_sm_fwd<S, 4><<<rows, 128, 0, L.stream>>>(P, T, b.PA, b.exP, plane);
    else if (T <= 1024) k_att_sm_fwd<S, 8><<<rows, 128, 0, L.stream>>>(P, T, b.PA, b.exP, plane);
    else k_att_sm_fwd<S, 16><<<rows, 128, 0, L.stream>>>(P, T, b.PA, b.exP, plane);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
  launch_cols<S>(L, ColJob{qkv, g.W, g.vo, g.Hkv, T, hd, zk, nullptr, b.VB, b.exV});
  {  // O = P V (k clipped to the causal part)
    GemmArgs<double> a;
    a.M = T; a.N = hd; a.K = T; a.batch = zq;
    a.C = o; a.ldc = g.ldo; a.offC = BatchOff{T * g.ldo, hd, g.Hq, 1};
    a.tri = TRI_K_LE_M;
    OzPlanes pa, pb;
    pa.d = b.PA; pa.ex = b.exP; pa.nb = zq; pa.Kp = T; pa.z = ident();
    pb.d = b.VB; pb.ex = b.exV; pb.nb = zk; pb.Kp = T; pb.z = kv;
    gemm_oz_planes(L, S, pa, pb, a);
  }
}

template <int S>
static void bwd(const Launch& L, const AttnShape& g, const double* qkv, const double* P, const double* dO, double* dP,
                double* dqkv) {
  const int zq = g.nseq * g.Hq, zk = g.nseq * g.Hkv, T = g.Tn, hd = g.hd, rep = g.Hq / g.Hkv;
  Bufs b = carve(g, S, (uint8_t*)L.ws->get(attn_oz_ws_bytes(L, g), L.stream));
  const BatchOff kv{g.Hkv, 1, g.Hq, rep};
  const BatchOff q_of_kv{g.Hq, rep, g.Hkv, 1};  // kv head (b, gk) -> q head (b, gk rep) (+ r via z0)
  const double scale = 1.0 / std::sqrt((double)hd);
  {
    RowJobs js;
    js.n = 2;
    js.j[0] = RowJob{dO, g.ldo, 0, g.Hq, T, hd, zq, b.DOA, b.exDO, 0};
    js.j[1] = RowJob{qkv, g.W, g.vo, g.Hkv, T, hd, zk, b.VR, b.exVR, 0};
    launch_rows<S>(L, js);
  }
  {  // dP = dO V^T (lower tiles only)
    GemmArgs<double> a;
    a.M = T; a.N = T; a.K = hd; a.batch = zq;
    a.C = dP; a.ldc = T; a.offC = BatchOff{(int64_t)T * T, 0, 1, 1};
    a.tri = TRI_SKIP_UPPER;
    OzPlanes pa, pb;
    pa.d = b.DOA; pa.ex = b.exDO; pa.nb = zq; pa.Kp = hd; pa.z = ident();
    pb.d = b.VR; pb.ex = b.exVR; pb.nb = zk; pb.Kp = hd; pb.z = kv;
    gemm_oz_planes(L, S, pa, pb, a);
  }
  {
    LaunchScope scope(L.prof, KC_ATTN, L.stream, 0, (32.0 + 3.0 * S) * zq * (T * (T + 128.0) / 2));
    k_att_sm_bwd<S><<<zq * (T / 32), 512, 0, L.stream>>>(P, dP, T, b.PT, b.DSA, b.DST, b.exR, b.exE,
                                                           (int64_t)zq * T * T);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
  launch_cols<S>(L, ColJob{qkv, g.W, g.ko, g.Hkv, T, hd, zk, nullptr, b.KT, b.exKT});
  launch_cols<S>(L, ColJob{dO, g.ldo, 0, g.Hq, T, hd, zq, b.exR, b.DOT, b.exDOT});
  launch_cols<S>(L, ColJob{qkv, g.W, g.qo, g.Hq, T, hd, zq, b.exE, b.QT, b.exQT});
  // dV[b, gk] = sum_r (P~_h)^T dO'_h,  h = gk rep + r  (k = query >= the tile's first key)
  for (int r = 0; r < rep; ++r) {
    GemmArgs<double> a;
    a.M = T; a.N = hd; a.K = T; a.batch = zk;
    a.C = dqkv + g.vo; a.ldc = g.W; a.offC = BatchOff{T * g.W, hd, g.Hkv, 1};
    a.accumulate = r > 0;
    a.tri = TRI_K_GE_M;
    OzPlanes pa, pb;
    pa.d = b.PT; pa.ex = nullptr; pa.nb = zq; pa.Kp = T; pa.z0 = r; pa.z = q_of_kv;
    pb.d = b.DOT; pb.ex = b.exDOT; pb.nb = zq; pb.Kp = T; pb.z0 = r; pb.z = q_of_kv;
    gemm_oz_planes(L, S, pa, pb, a);
  }
  {  // dQ = scale dS K (k = key <= the tile's last query)
    GemmArgs<double> a;
    a.M = T; a.N = hd; a.K = T; a.batch = zq;
    a.C = dqkv + g.qo; a.ldc = g.W; a.offC = BatchOff{T * g.W, hd, g.Hq, 1};
    a.alpha = scale;
    a.tri = TRI_K_LE_M;
    OzPlanes pa, pb;
    pa.d = b.DSA; pa.ex = b.exE; pa.nb = zq; pa.Kp = T; pa.z = ident();
    pb.d = b.KT; pb.ex = b.exKT; pb.nb = zk; pb.Kp = T; pb.z = kv;
    gemm_oz_planes(L, S, pa, pb, a);
  }
  // dK[b, gk] = scale sum_r (dS~_h)^T Q'_h
  for (int r = 0; r < rep; ++r) {
    GemmArgs<double> a;
    a.M = T; a.N = hd; a.K = T; a.batch = zk;
    a.C = dqkv + g.ko; a.ldc = g.W; a.offC = BatchOff{T * g.W, hd, g.Hkv, 1};
    a.alpha = scale;
    a.accumulate = r > 0;
    a.tri = TRI_K_GE_M;
    OzPlanes pa, pb;
    pa.d = b.DST; pa.ex = nullptr; pa.nb = zq; pa.Kp = T; pa.z0 = r; pa.z = q_of_kv;
    pb.d = b.QT; pb.ex = b.exQT; pb.nb = zq; pb.Kp = T; pb.z0 = r; pb.z = q_of_kv;
    gemm_oz_planes(L, S, pa, pb, a);
  }
}

}  // namespace oz

bool attn_oz_eligible(const Launch& L, const AttnShape& g) {
  static const bool off = getenv("SLQ_ATTN_DMMA") && atoi(getenv("SLQ_ATTN_DMMA")) != 0;  // A/B switch
  return !off && L.gemm_mode == 2 && g.Tn % 128 == 0 && g.Tn <= 2048 && g.hd % 32 == 0 && g.hd <= 128 && g.Hkv > 0 &&
         g.Hq % g.Hkv == 0 && (double)g.nseq * g.Hq * g.Tn * (double)g.Tn * g.hd >= L.oz_min_mnk;
}

size_t attn_oz_ws_bytes(const Launch& L, const AttnShape& g) {
  if (!attn_oz_eligible(L, g)) return 0;
  const oz::Bufs b = oz::carve(g, L.oz_S, nullptr);
  return std::max(b.fwd_bytes, b.bwd_bytes);
}

void attention_fwd_oz(const Launch& L, const AttnShape& g, const double* qkv, double* P, double* o) {
  switch (L.oz_S) {
    case 4: oz::fwd<4>(L, g, qkv, P, o); break;
    case 5: oz::fwd<5>(L, g, qkv, P, o); break;
    case 6: oz::fwd<6>(L, g, qkv, P, o); break;
    case 7: oz::fwd<7>(L, g, qkv, P, o); break;
    default: throw Error(SLQ_EINVAL, "oz attention: S in 4..7");
  }
}

void attention_bwd_oz(const Launch& L, const AttnShape& g, const double* qkv, const double* P, const double* dO,
                      double* dP, double* dqkv) {
  switch (L.oz_S) {
    case 4: oz::bwd<4>(L, g, qkv, P, dO, dP, dqkv); break;
    case 5: oz::bwd<5>(L, g, qkv, P, dO, dP, dqkv); break;
    case 6: oz::bwd<6>(L, g, qkv, P, dO, dP, dqkv); break;
    case 7: oz::bwd<7>(L, g, qkv, P, dO, dP, dqkv); break;
    default: throw Error(SLQ_EINVAL, "oz attention: S in 4..7");
  }
}

}  // namespace slq
