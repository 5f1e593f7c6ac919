// Row-wise and elementwise layers of the gradient passes:
// embeddings (deterministic, atomics-free backward), LayerNorm / RMSNorm (warp-shuffle row
// reductions, two-stage deterministic column reductions for the gains), causal softmax and its
// backward, token cross-entropy (online max / log-sum-exp), RoPE and SwiGLU.
#include <cuda_runtime.h>
#include <math.h>

#include "kernels.h"

namespace slq {

namespace {

constexpr int kWarp = 32;

template <class T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <class T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double dexp(double x) { return exp(x); }
__device__ __forceinline__ float dexp(float x) { return expf(x); }
__device__ __forceinline__ double dsqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float dsqrt(float x) { return sqrtf(x); }

// online softmax statistics: (m, s) with s = sum_j exp(x_j - m), m = max_j x_j
template <class T>
__device__ __forceinline__ void online_add(T& m, T& s, T x) {
  if (x > m) {
    s = s * dexp(m - x) + T(1);
    m = x;
  } else if (x > T(-INFINITY)) {  // (x = m = -inf would give exp(nan))
    s += dexp(x - m);
  } else if (x != x) {  // NaN: both comparisons are false; poison the row (the loss must be non-finite)
    m = x;
    s = x;
  }
}
template <class T>
__device__ __forceinline__ void online_merge(T& m, T& s, T m2, T s2) {
  const T mm = max(m, m2);
  s = (m == mm ? s : s * dexp(m - mm)) + (m2 == mm ? s2 : s2 * dexp(m2 - mm));
  m = mm;
}
template <class T>
__device__ __forceinline__ void warp_online(T& m, T& s) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const T m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, s, o);
    online_merge(m, s, m2, s2);
  }
}

inline int grid_for(int64_t n, int threads, int cap = 148 * 16) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), cap));
}

#define LAUNCH(cls, grid, block, kernel, ...)                          \
  do {                                                                 \
    LaunchScope scope_(L.prof, cls, L.stream);                         \
    kernel<<<grid, block, 0, L.stream>>>(__VA_ARGS__);                 \
    SLQ_CUDA(cudaGetLastError());                                      \
    ++*L.launches;                                                     \
  } while (0)

// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_convert(const float* __restrict__ x, T* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (T)x[i];
}

// x[b*T + t, :] = wte[tok[b][t], :] (+ wpe[t, :])
template <class T>
__global__ void k_embed_fwd(const int32_t* __restrict__ tok, int tok_stride, int nseq, int Tn,
                            const T* __restrict__ wte, const T* __restrict__ wpe, T* __restrict__ x, int D) {
  const int64_t total = (int64_t)nseq * Tn * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / D;
    const int c = (int)(i % D);
    const int b = (int)(row / Tn), t = (int)(row % Tn);
    const int id = tok[(int64_t)b * tok_stride + t];
    T v = wte[(int64_t)id * D + c];
    if (wpe) v += wpe[(int64_t)t * D + c];
    x[i] = v;
  }
}

// dW[v, :] (+)= sum over the rows listed for token v (CSR built once at init; fixed order)
// Embedding backward, stage 1: partial[c][col] = sum of dx rows over the <= kEmbedChunk token
// positions of chunk c (fixed order).  Stage 2: dW[v][col] (+)= sum of row v's chunk partials in
// chunk order.  Splitting the long token lists of frequent tokens (Zipf: the top token is ~14% of
// all positions) keeps every thread's dependent-load chain short.
template <class T>
__global__ void k_embed_bwd_chunks(const int32_t* __restrict__ pos, const int32_t* __restrict__ cbeg, int nchunks,
                                   const T* __restrict__ dx, T* __restrict__ part, int D) {
  const int64_t total = (int64_t)nchunks * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / D), col = (int)(i % D);
    const int s = cbeg[c], e = cbeg[c + 1];
    int p[kEmbedChunk];
#pragma unroll
    for (int j = 0; j < kEmbedChunk; ++j) p[j] = s + j < e ? pos[s + j] : -1;
    T acc = T(0);
#pragma unroll
    for (int j = 0; j < kEmbedChunk; ++j)
      if (p[j] >= 0) acc += dx[(int64_t)p[j] * D + col];
    part[i] = acc;
  }
}

template <class T>
__global__ void k_embed_bwd_rows(const int32_t* __restrict__ coff, const T* __restrict__ part, T* __restrict__ dW,
                                 int V, int D, bool accumulate) {
  const int64_t total = (int64_t)V * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(i / D), col = (int)(i % D);
    T acc = T(0);
    for (int c = coff[v]; c < coff[v + 1]; ++c) acc += part[(int64_t)c * D + col];
    T* dst = dW + i;
    *dst = accumulate ? *dst + acc : acc;
  }
}

template <class T>
__global__ void k_pos_bwd(const T* __restrict__ dx, T* __restrict__ dwpe, int nseq, int Tn, int D) {
  const int64_t total = (int64_t)Tn * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int b = 0; b < nseq; ++b) acc += dx[(int64_t)b * Tn * D + i];
    dwpe[i] = acc;
  }
}

// One warp per row.  V > 0: the row's values (D <= 32 V) are kept in registers across the passes
// (one global read per operand instead of two or three); the summation order is the same as the
// streaming V = 0 form, so both give identical results.
template <class T, int V>
__global__ void k_layernorm_fwd(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b,
                                T* __restrict__ y, T* __restrict__ mean, T* __restrict__ rstd, int rows, int D,
                                T eps) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const T* xr = x + (int64_t)row * D;
  T* yr = y + (int64_t)row * D;
  T mu, rs;
  if constexpr (V > 0) {
    T xv[V];
    T s = T(0);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      xv[i] = c < D ? xr[c] : T(0);
      if (c < D) s += xv[i];
    }
    mu = warp_sum(s) / T(D);
    T v = T(0);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      if (c < D) {
        const T d = xv[i] - mu;
        v += d * d;
      }
    }
    rs = T(1) / dsqrt(warp_sum(v) / T(D) + eps);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      if (c < D) yr[c] = (xv[i] - mu) * rs * g[c] + b[c];
    }
  } else {
    T s = T(0);
    for (int c = lane; c < D; c += kWarp) s += xr[c];
    mu = warp_sum(s) / T(D);
    T v = T(0);
    for (int c = lane; c < D; c += kWarp) {
      const T d = xr[c] - mu;
      v += d * d;
    }
    rs = T(1) / dsqrt(warp_sum(v) / T(D) + eps);
    for (int c = lane; c < D; c += kWarp) yr[c] = (xr[c] - mu) * rs * g[c] + b[c];
  }
  if (lane == 0) {
    mean[row] = mu;
    rstd[row] = rs;
  }
}

// dx = rstd * (dxhat - mean(dxhat) - xhat * mean(dxhat * xhat)) (+ dres),  dxhat = dy * g
template <class T, int V>
__global__ void __launch_bounds__(256, 2) k_layernorm_bwd(const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ mean,
                                const T* __restrict__ rstd, const T* __restrict__ g, const T* __restrict__ dres,
                                T* __restrict__ dx, int rows, int D) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int64_t o = (int64_t)row * D;
  const T mu = mean[row], rs = rstd[row];
  if constexpr (V > 0) {
    T dh[V], xh[V];
    T s1 = T(0), s2 = T(0);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      if (c < D) {
        dh[i] = dy[o + c] * g[c];
        xh[i] = (x[o + c] - mu) * rs;
        s1 += dh[i];
        s2 += dh[i] * xh[i];
      } else {
        dh[i] = xh[i] = T(0);
      }
    }
    s1 = warp_sum(s1) / T(D);
    s2 = warp_sum(s2) / T(D);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      if (c < D) {
        T v = rs * (dh[i] - s1 - xh[i] * s2);
        if (dres) v += dres[o + c];
        dx[o + c] = v;
      }
    }
  } else {
    T s1 = T(0), s2 = T(0);
    for (int c = lane; c < D; c += kWarp) {
      const T dxh = dy[o + c] * g[c];
      const T xh = (x[o + c] - mu) * rs;
      s1 += dxh;
      s2 += dxh * xh;
    }
    s1 = warp_sum(s1) / T(D);
    s2 = warp_sum(s2) / T(D);
    for (int c = lane; c < D; c += kWarp) {
      const T dxh = dy[o + c] * g[c];
      const T xh = (x[o + c] - mu) * rs;
      T v = rs * (dxh - s1 - xh * s2);
      if (dres) v += dres[o + c];
      dx[o + c] = v;
    }
  }
}

template <class T, int V>
__global__ void k_rmsnorm_fwd(const T* __restrict__ x, const T* __restrict__ g, T* __restrict__ y,
                              T* __restrict__ rstd, int rows, int D, T eps) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const T* xr = x + (int64_t)row * D;
  T* yr = y + (int64_t)row * D;
  T r;
  if constexpr (V > 0) {
    T xv[V];
    T s = T(0);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      xv[i] = c < D ? xr[c] : T(0);
      if (c < D) s += xv[i] * xv[i];
    }
    r = T(1) / dsqrt(warp_sum(s) / T(D) + eps);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      if (c < D) yr[c] = xv[i] * r * g[c];
    }
  } else {
    T s = T(0);
    for (int c = lane; c < D; c += kWarp) s += xr[c] * xr[c];
    r = T(1) / dsqrt(warp_sum(s) / T(D) + eps);
    for (int c = lane; c < D; c += kWarp) yr[c] = xr[c] * r * g[c];
  }
  if (lane == 0) rstd[row] = r;
}

// dx = r * dxhat - x * r^3 * mean(dxhat * x) (+ dres)
template <class T, int V>
__global__ void k_rmsnorm_bwd(const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ rstd,
                              const T* __restrict__ g, const T* __restrict__ dres, T* __restrict__ dx, int rows,
                              int D) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int64_t o = (int64_t)row * D;
  const T r = rstd[row];
  if constexpr (V > 0) {
    T dv[V], xv[V];
    T s = T(0);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      if (c < D) {
        dv[i] = dy[o + c] * g[c];
        xv[i] = x[o + c];
        s += dv[i] * xv[i];
      } else {
        dv[i] = xv[i] = T(0);
      }
    }
    s = warp_sum(s) / T(D);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int c = lane + kWarp * i;
      if (c < D) {
        T v = r * dv[i] - xv[i] * r * r * r * s;
        if (dres) v += dres[o + c];
        dx[o + c] = v;
      }
    }
  } else {
    T s = T(0);
    for (int c = lane; c < D; c += kWarp) s += dy[o + c] * g[c] * x[o + c];
    s = warp_sum(s) / T(D);
    for (int c = lane; c < D; c += kWarp) {
      T v = r * dy[o + c] * g[c] - x[o + c] * r * r * r * s;
      if (dres) v += dres[o + c];
      dx[o + c] = v;
    }
  }
}

// stage 1 of the column reductions: block (cx, cy) reduces rows [cy*rpb, (cy+1)*rpb) of
// columns [cx*blockDim, ...) into part[cy][col]
// block = 32 columns x 8 row lanes; rows [r0, r1) of this block's slab, reduced over the row
// lanes in shared memory in a fixed order
template <class T>
__global__ void k_colreduce1(int mode, const T* __restrict__ dy, int64_t lddy, const T* __restrict__ x,
                             const T* __restrict__ mean, const T* __restrict__ rstd, T* __restrict__ part0,
                             T* __restrict__ part1, int rows, int cols, int rpb, unsigned* __restrict__ counter,
                             T* __restrict__ out0, T* __restrict__ out1, bool accumulate) {
  __shared__ T s0[8][33], s1[8][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int c = blockIdx.x * 32 + tx;
  const int r0 = blockIdx.y * rpb, r1 = min(rows, r0 + rpb);
  T a0 = T(0), a1 = T(0);
  if (c < cols) {
    // four rows per iteration with every load issued before the first use (memory-level
    // parallelism: the loop is latency-bound otherwise); rows are summed in increasing order
    int r = r0 + ty;
    for (; r + 24 < r1; r += 32) {
      T d[4], xv[4], mu[4], rs[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int64_t rr = r + 8 * i;
        d[i] = dy[rr * lddy + c];
        if (mode != 0) {
          xv[i] = x[rr * cols + c];
          rs[i] = rstd[rr];
          mu[i] = mode == 1 ? mean[rr] : T(0);
        }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (mode == 0) {
          a0 += d[i];
        } else if (mode == 1) {
          a0 += d[i] * (xv[i] - mu[i]) * rs[i];
          a1 += d[i];
        } else {
          a0 += d[i] * xv[i] * rs[i];
        }
      }
    }
    for (; r < r1; r += 8) {
      const T d = dy[(int64_t)r * lddy + c];
      if (mode == 0) {
        a0 += d;
      } else if (mode == 1) {
        a0 += d * (x[(int64_t)r * cols + c] - mean[r]) * rstd[r];
        a1 += d;
      } else {
        a0 += d * x[(int64_t)r * cols + c] * rstd[r];
      }
    }
  }
  s0[ty][tx] = a0;
  s1[ty][tx] = a1;
  __syncthreads();
  if (ty == 0 && c < cols) {
    T b0 = T(0), b1 = T(0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      b0 += s0[i][tx];
      b1 += s1[i][tx];
    }
    part0[(int64_t)blockIdx.y * cols + c] = b0;
    if (mode == 1) part1[(int64_t)blockIdx.y * cols + c] = b1;
  }
  // stage 2 in the last block to finish (threadfence + counter): every column's partials are
  // summed in slab order, so the result does not depend on which block finishes last
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned nb = gridDim.x * gridDim.y;
    last = atomicAdd(counter, 1u) == nb - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int nparts = gridDim.y;
  for (int cc = threadIdx.x; cc < cols; cc += blockDim.x) {
    T s0v = T(0), s1v = T(0);
    int p = 0;
    // eight partial rows' loads in flight before the (in-order) additions
    for (; p + 8 <= nparts; p += 8) {
      T a[8], b[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        a[i] = __ldcg(part0 + (int64_t)(p + i) * cols + cc);
        b[i] = mode == 1 ? __ldcg(part1 + (int64_t)(p + i) * cols + cc) : T(0);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        s0v += a[i];
        if (mode == 1) s1v += b[i];
      }
    }
    for (; p < nparts; ++p) {
      s0v += __ldcg(part0 + (int64_t)p * cols + cc);
      if (mode == 1) s1v += __ldcg(part1 + (int64_t)p * cols + cc);
    }
    out0[cc] = accumulate ? out0[cc] + s0v : s0v;
    if (mode == 1) out1[cc] = accumulate ? out1[cc] + s1v : s1v;
  }
  if (threadIdx.x == 0) *counter = 0u;  // ready for the next call on this stream
}

// one warp per column

// causal softmax over rows of length Tn; row r is query position t = r % Tn (keys j <= t)
template <class T>
__global__ void k_softmax_causal(T* __restrict__ S, int64_t rows, int Tn) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int t = (int)(row % Tn);
  T* s = S + row * Tn;
  // one read for the (online) max and sum, one read + write for the probabilities
  T mx = -INFINITY, sum = T(0);
  for (int j = lane; j <= t; j += kWarp) online_add(mx, sum, s[j]);
  warp_online(mx, sum);
  const T inv = T(1) / sum;
  // entries j > t are zeroed only up to the end of t's 128-wide column block: the causal GEMMs that
  // read P (TRI_K_LE_M / TRI_K_GE_M, tiles <= 128 aligned on 128) never go further, and the tiles
  // entirely above the diagonal are neither computed nor read (TRI_SKIP_UPPER)
  const int jend = min(Tn, (t / 128 + 1) * 128);
  for (int j = lane; j < jend; j += kWarp) s[j] = (j <= t) ? dexp(s[j] - mx) * inv : T(0);
}

// register-resident variant for Tn <= 32 V: lane l holds s[l + 32 i]; one read of the causal part
// and one write of the row (same per-lane summation order as k_softmax_causal)
// One 128-thread block per row for long rows (Tn <= 128 V): the row is read once into registers
// (V values per thread), one exp per element, block reductions for the max and the sum, one write
// (up to the end of the diagonal 128-column block, as k_softmax_causal).  The warp-per-row kernels
// either read the row twice with two exps per element (online form) or hold 32 fp64 values per
// lane at low occupancy.
template <class T, int V>
__global__ void __launch_bounds__(128) k_softmax_causal_blk(T* __restrict__ S, int64_t rows, int Tn) {
  __shared__ T red[4];
  const int64_t row = blockIdx.x;
  const int t = (int)(row % Tn);
  T* s = S + row * Tn;
  const int tid = threadIdx.x, lane = tid % kWarp, wid = tid / kWarp;
  T v[V];
  T mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = tid + 128 * i;
    v[i] = j <= t ? s[j] : T(-INFINITY);
    mx = max(mx, v[i]);
  }
  mx = warp_max(mx);
  if (lane == 0) red[wid] = mx;
  __syncthreads();
  mx = max(max(red[0], red[1]), max(red[2], red[3]));
  __syncthreads();
  T sum = T(0);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (tid + 128 * i <= t) {
      v[i] = dexp(v[i] - mx);
      sum += v[i];
    }
  }
  sum = warp_sum(sum);
  if (lane == 0) red[wid] = sum;
  __syncthreads();
  const T inv = T(1) / ((red[0] + red[1]) + (red[2] + red[3]));
  const int jend = min(Tn, (t / 128 + 1) * 128);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = tid + 128 * i;
    if (j < jend) s[j] = j <= t ? v[i] * inv : T(0);
  }
}

template <class T, int V>
__global__ void k_softmax_causal_reg(T* __restrict__ S, int64_t rows, int Tn) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int t = (int)(row % Tn);
  T* s = S + row * Tn;
  T v[V];
  T mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + kWarp * i;
    v[i] = j <= t ? s[j] : T(-INFINITY);
    mx = max(mx, v[i]);
  }
  mx = warp_max(mx);
  T sum = T(0);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    if (lane + kWarp * i <= t) {
      v[i] = dexp(v[i] - mx);
      sum += v[i];
    }
  }
  const T inv = T(1) / warp_sum(sum);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + kWarp * i;
    if (j < Tn) s[j] = j <= t ? v[i] * inv : T(0);
  }
}

// dS = P * (dP - sum_j dP_j P_j), in place in dP
template <class T>
__global__ void k_softmax_bwd(const T* __restrict__ P, T* __restrict__ dP, int64_t rows, int Tn) {
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kWarp;
  const int lane = threadIdx.x % kWarp;
  if (row >= rows) return;
  const int t = (int)(row % Tn);
  const T* p = P + row * Tn;
  T* d = dP + row * Tn;
  T s = T(0);
  for (int j = lane; j <= t; j += kWarp) s += p[j] * d[j];  // entries j > t were never computed
  s = warp_sum(s);
  const int jend = min(Tn, (t / 128 + 1) * 128);  // (see k_softmax_causal)
  for (int j = lane; j < jend; j += kWarp) d[j] = (j <= t) ? p[j] * (d[j] - s) : T(0);
}

// one block per row: loss_row = lse - logit[tgt];  logits <- (softmax - onehot) * inv_ntok
template <class T>
__global__ void __launch_bounds__(1024, 1) k_cross_entropy(T* __restrict__ logits, const int32_t* __restrict__ tgt, int tgt_stride, int Tn,
                                double* __restrict__ loss_rows, int V, double inv_ntok) {
  const int row = blockIdx.x;
  T* z = logits + (int64_t)row * V;
  const int b = row / Tn, t = row % Tn;
  const int y = tgt[(int64_t)b * tgt_stride + t];
  __shared__ T red[32], red2[32];
  // Three sweeps over the row, one exp per element: the max; e_j = exp(z_j - max) stored in place
  // with their sum; the gradient e_j / sum - [j == y] (scaled).  1024-thread blocks, one per SM
  // (launch bounds): the rows in flight (148 x V x 8 B = 60 MB for V = 50257) stay in L2, so the
  // second and third sweeps cost no DRAM traffic; the kernel is bound by the fp64 exp (the online
  // (max, sum) form needed a second exp per element in the gradient sweep, serially dependent)
  const int bs = blockDim.x, nw = bs / kWarp, lane = threadIdx.x % kWarp, wid = threadIdx.x / kWarp;
  const T zy = z[y];  // (read before the second sweep overwrites the row)
  T mx = -INFINITY;
  bool bad = false;
  for (int j0 = threadIdx.x; j0 < V; j0 += 8 * bs) {
    T x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = j0 + i * bs < V ? z[j0 + i * bs] : T(-INFINITY);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      mx = max(mx, x[i]);
      bad |= x[i] != x[i];
    }
  }
  mx = warp_max(mx);
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) red[wid] = bad ? T(NAN) : mx;
  __syncthreads();
  if (threadIdx.x < kWarp) {
    T m = threadIdx.x < nw ? red[threadIdx.x] : T(-INFINITY);
    const bool b2 = __any_sync(0xffffffffu, m != m);
    m = warp_max(m);
    if (threadIdx.x == 0) red[0] = b2 ? T(NAN) : m;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  T sm = T(0);
  for (int j0 = threadIdx.x; j0 < V; j0 += 8 * bs) {
    T x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = j0 + i * bs < V ? z[j0 + i * bs] : T(0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (j0 + i * bs < V) {
        x[i] = dexp(x[i] - mx);
        sm += x[i];
        z[j0 + i * bs] = x[i];
      }
    }
  }
  sm = warp_sum(sm);
  if (lane == 0) red2[wid] = sm;
  __syncthreads();
  if (threadIdx.x < kWarp) {
    T s2 = threadIdx.x < nw ? red2[threadIdx.x] : T(0);
    s2 = warp_sum(s2);
    if (threadIdx.x == 0) red2[0] = s2;
  }
  __syncthreads();
  const T sum = red2[0];
  const T lse = mx + log(sum);
  if (threadIdx.x == 0) loss_rows[row] = (double)(lse - zy);
  __syncthreads();
  const T inv = T(1) / sum, scale = (T)inv_ntok;
  for (int j0 = threadIdx.x; j0 < V; j0 += 8 * bs) {
    T x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = j0 + i * bs < V ? z[j0 + i * bs] : T(0);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int j = j0 + i * bs;
      if (j < V) {
        T p = x[i] * inv;
        if (j == y) p -= T(1);
        z[j] = p * scale;
      }
    }
  }
}

// Register-resident variant for V <= 256 NV (one read and one write of the row): thread t holds
// z[t + 256 i]; the exact max, then the sum of exponentials, and the gradient are formed from
// registers.
template <class T, int NV>
__global__ void __launch_bounds__(256) k_cross_entropy_reg(T* __restrict__ logits, const int32_t* __restrict__ tgt,
                                                           int tgt_stride, int Tn, double* __restrict__ loss_rows,
                                                           int V, double inv_ntok) {
  const int row = blockIdx.x;
  T* z = logits + (int64_t)row * V;
  const int b = row / Tn, t = row % Tn;
  const int y = tgt[(int64_t)b * tgt_stride + t];
  __shared__ T red[32];
  T v[NV];
  T mx = -INFINITY;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = threadIdx.x + 256 * i;
    v[i] = j < V ? z[j] : T(-INFINITY);
    mx = max(mx, v[i]);
  }
  mx = warp_max(mx);
  if (threadIdx.x % kWarp == 0) red[threadIdx.x / kWarp] = mx;
  __syncthreads();
  if (threadIdx.x < kWarp) {
    T w = threadIdx.x < blockDim.x / kWarp ? red[threadIdx.x] : T(-INFINITY);
    w = warp_max(w);
    if (threadIdx.x == 0) red[0] = w;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  T s = T(0);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    if (threadIdx.x + 256 * i < V) {
      v[i] = dexp(v[i] - mx);
      s += v[i];
    }
  }
  s = warp_sum(s);
  if (threadIdx.x % kWarp == 0) red[threadIdx.x / kWarp] = s;
  __syncthreads();
  if (threadIdx.x < kWarp) {
    T w = threadIdx.x < blockDim.x / kWarp ? red[threadIdx.x] : T(0);
    w = warp_sum(w);
    if (threadIdx.x == 0) red[0] = w;
  }
  __syncthreads();
  const T sum = red[0];
  const T lse = mx + log(sum);
  if (threadIdx.x == 0) loss_rows[row] = (double)(lse - z[y]);
  __syncthreads();
  const T inv = T(1) / sum, scale = (T)inv_ntok;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int j = threadIdx.x + 256 * i;
    if (j < V) {
      T p = v[i] * inv;
      if (j == y) p -= T(1);
      z[j] = p * scale;
    }
  }
}

__global__ void k_sum_rows(const double* __restrict__ x, int n, double* out) {
  __shared__ double red[32];
  double s = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  s = warp_sum(s);
  if (threadIdx.x % kWarp == 0) red[threadIdx.x / kWarp] = s;
  __syncthreads();
  if (threadIdx.x < kWarp) {
    double v = threadIdx.x < blockDim.x / kWarp ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) *out = v;
  }
}

// RoPE on a [rows, ld] buffer holding `heads` heads of width hd starting at column 0; row r has
// position r % Tn.  Rotates pairs (i, i + hd/2) by +angle (inverse: -angle, the transpose).
template <class T>
__global__ void k_rope(T* __restrict__ x, int64_t ld, int rows, int Tn, int heads, int hd, const T* __restrict__ cs,
                       const T* __restrict__ sn, bool inverse) {
  const int half = hd / 2;
  const int64_t total = (int64_t)rows * heads * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(i % half);
    const int64_t rh = i / half;
    const int h = (int)(rh % heads);
    const int r = (int)(rh / heads);
    const int t = r % Tn;
    T* p = x + (int64_t)r * ld + (int64_t)h * hd;
    const T c = cs[(int64_t)t * half + j], s = inverse ? -sn[(int64_t)t * half + j] : sn[(int64_t)t * half + j];
    const T a = p[j], b = p[j + half];
    p[j] = a * c - b * s;
    p[j + half] = b * c + a * s;
  }
}

template <class T>
__global__ void k_swiglu_fwd(const T* __restrict__ ab, T* __restrict__ f, int rows, int F) {
  const int64_t n = (int64_t)rows * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F, j = i % F;
    const T a = ab[r * 2 * F + j], b = ab[r * 2 * F + F + j];
    const T s = T(1) / (T(1) + dexp(-a));
    f[i] = a * s * b;
  }
}

template <class T>
__global__ void k_swiglu_bwd(const T* __restrict__ df, const T* __restrict__ ab, T* __restrict__ dab, int rows, int F) {
  const int64_t n = (int64_t)rows * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / F, j = i % F;
    const T a = ab[r * 2 * F + j], b = ab[r * 2 * F + F + j];
    const T s = T(1) / (T(1) + dexp(-a));
    const T d = df[i];
    dab[r * 2 * F + j] = d * b * s * (T(1) + a * (T(1) - s));
    dab[r * 2 * F + F + j] = d * a * s;
  }
}

template <class T>
__global__ void k_add(T* __restrict__ y, const T* __restrict__ x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += x[i];
}

}  // namespace

template <class T>
void convert_f32(const Launch& L, const float* x, T* y, int64_t n) {
  if (n == 0) return;
  LAUNCH(KC_ELEM, grid_for(n, 256), 256, k_convert<T>, x, y, n);
}
template <class T>
void embed_fwd(const Launch& L, const int32_t* tok, int tok_stride, int nseq, int Tn, const T* wte, const T* wpe,
               T* x, int D) {
  const int64_t n = (int64_t)nseq * Tn * D;
  if (n == 0) return;
  LAUNCH(KC_EMBED, grid_for(n, 256), 256, k_embed_fwd<T>, tok, tok_stride, nseq, Tn, wte, wpe, x, D);
}
template <class T>
void embed_bwd_rows(const Launch& L, const EmbedCSR& csr, const T* dx, T* dW, int V, int D, bool accumulate) {
  T* part = (T*)L.ws->get(sizeof(T) * (size_t)std::max(csr.nchunks, 1) * D, L.stream);
  if (csr.nchunks > 0)
    LAUNCH(KC_EMBED, grid_for((int64_t)csr.nchunks * D, 256), 256, k_embed_bwd_chunks<T>, csr.pos, csr.cbeg,
           csr.nchunks, dx, part, D);
  LAUNCH(KC_EMBED, grid_for((int64_t)V * D, 256), 256, k_embed_bwd_rows<T>, csr.coff, part, dW, V, D, accumulate);
}

void build_embed_csr(const std::vector<int32_t>& tok, int nseq, int Tn, int V, std::vector<int32_t>& off,
                     std::vector<int32_t>& pos, std::vector<int32_t>& coff, std::vector<int32_t>& cbeg) {
  off.assign(V + 1, 0);
  for (int b = 0; b < nseq; ++b)
    for (int t = 0; t < Tn; ++t) off[tok[(size_t)b * (Tn + 1) + t] + 1]++;
  for (int v = 0; v < V; ++v) off[v + 1] += off[v];
  pos.assign((size_t)nseq * Tn, 0);
  std::vector<int32_t> fill(off.begin(), off.end() - 1);
  for (int b = 0; b < nseq; ++b)
    for (int t = 0; t < Tn; ++t) pos[fill[tok[(size_t)b * (Tn + 1) + t]]++] = b * Tn + t;
  coff.assign(V + 1, 0);
  cbeg.clear();
  for (int v = 0; v < V; ++v) {
    for (int s = off[v]; s < off[v + 1]; s += kEmbedChunk) cbeg.push_back(s);
    coff[v + 1] = (int32_t)cbeg.size();
  }
  cbeg.push_back(off[V]);
}
template <class T>
void pos_bwd(const Launch& L, const T* dx, T* dwpe, int nseq, int Tn, int D) {
  LAUNCH(KC_EMBED, grid_for((int64_t)Tn * D, 256), 256, k_pos_bwd<T>, dx, dwpe, nseq, Tn, D);
}
template <class T>
void layernorm_fwd(const Launch& L, const T* x, const T* g, const T* b, T* y, T* mean, T* rstd, int rows, int D,
                   double eps) {
  if (rows == 0) return;
  if (D <= 256)
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_layernorm_fwd<T, 8>), x, g, b, y, mean, rstd, rows, D, (T)eps);
  else if (D <= 768)
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_layernorm_fwd<T, 24>), x, g, b, y, mean, rstd, rows, D, (T)eps);
  else
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_layernorm_fwd<T, 0>), x, g, b, y, mean, rstd, rows, D, (T)eps);
}
template <class T>
void layernorm_bwd(const Launch& L, const T* dy, const T* x, const T* mean, const T* rstd, const T* g,
                   const T* dres, T* dx, int rows, int D) {
  if (rows == 0) return;
  // D > 256: the generic kernel (statistics pass, then a re-read pass; ~40 registers) -- at
  // D = 768 it runs 2.3x faster than the register-resident V = 24 variant, whose 128 registers
  // leave too few warps to hide the two load phases (c3: 81 -> 35 us per launch)
  static const int generic = getenv("SLQ_LN_GENERIC") ? atoi(getenv("SLQ_LN_GENERIC")) : 1;
  if (D <= 256)
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_layernorm_bwd<T, 8>), dy, x, mean, rstd, g, dres, dx, rows, D);
  else if (D <= 768 && !generic)
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_layernorm_bwd<T, 24>), dy, x, mean, rstd, g, dres, dx, rows, D);
  else
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_layernorm_bwd<T, 0>), dy, x, mean, rstd, g, dres, dx, rows, D);
}
template <class T>
void rmsnorm_fwd(const Launch& L, const T* x, const T* g, T* y, T* rstd, int rows, int D, double eps) {
  if (rows == 0) return;
  if (D <= 256)
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_rmsnorm_fwd<T, 8>), x, g, y, rstd, rows, D, (T)eps);
  else if (D <= 768)
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_rmsnorm_fwd<T, 24>), x, g, y, rstd, rows, D, (T)eps);
  else
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_rmsnorm_fwd<T, 0>), x, g, y, rstd, rows, D, (T)eps);
}
template <class T>
void rmsnorm_bwd(const Launch& L, const T* dy, const T* x, const T* rstd, const T* g, const T* dres, T* dx,
                 int rows, int D) {
  if (rows == 0) return;
  if (D <= 256)
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_rmsnorm_bwd<T, 8>), dy, x, rstd, g, dres, dx, rows, D);
  else if (D <= 768)
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_rmsnorm_bwd<T, 24>), dy, x, rstd, g, dres, dx, rows, D);
  else
    LAUNCH(KC_NORM, (int)ceil_div(rows, 8), 256, (k_rmsnorm_bwd<T, 0>), dy, x, rstd, g, dres, dx, rows, D);
}
template <class T>
void colreduce(const Launch& L, int mode, const T* dy, int64_t lddy, const T* x, const T* mean, const T* rstd,
               T* out0, T* out1, int rows, int cols, bool accumulate) {
  if (cols == 0) return;
  const int cblocks = (int)ceil_div(cols, 32);
  int rblocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows, 64), ceil_div(2 * 148, cblocks)));
  const int rpb = (int)ceil_div(std::max(rows, 1), rblocks);
  rblocks = (int)ceil_div(std::max(rows, 1), rpb);
  T* part = (T*)L.ws->get(sizeof(T) * 2 * (size_t)rblocks * cols, L.stream);
  T* part1 = part + (size_t)rblocks * cols;
  unsigned* counter = L.ws->counters(1);  // zero on entry, reset by the last block
  LAUNCH(KC_NORM, dim3(cblocks, rblocks), 256, k_colreduce1<T>, mode, dy, lddy, x, mean, rstd, part, part1, rows,
         cols, rpb, counter, out0, out1, accumulate);
}
template <class T>
void softmax_causal_fwd(const Launch& L, T* S, int64_t rows, int Tn) {
  if (rows == 0) return;
  // (at Tn = 1024 the 32-value register variant is slower than the generic kernel: 500 vs 429 us
  // per c3 launch -- its 107 registers halve the resident warps)
  if (Tn <= 256)
    LAUNCH(KC_ATTN, (int)ceil_div(rows, 8), 256, (k_softmax_causal_reg<T, 8>), S, rows, Tn);
  else if (Tn <= 1024)
    LAUNCH(KC_ATTN, (int)rows, 128, (k_softmax_causal_blk<T, 8>), S, rows, Tn);
  else if (Tn <= 2048)
    LAUNCH(KC_ATTN, (int)rows, 128, (k_softmax_causal_blk<T, 16>), S, rows, Tn);
  else
    LAUNCH(KC_ATTN, (int)ceil_div(rows, 8), 256, k_softmax_causal<T>, S, rows, Tn);
}
template <class T>
void softmax_bwd(const Launch& L, const T* P, T* dP, int64_t rows, int Tn) {
  if (rows == 0) return;
  LAUNCH(KC_ATTN, (int)ceil_div(rows, 8), 256, k_softmax_bwd<T>, P, dP, rows, Tn);
}
template <class T>
void cross_entropy(const Launch& L, T* logits, const int32_t* tgt, int tgt_stride, int Tn, double* loss_rows,
                   int rows, int V, double inv_ntok) {
  if (rows == 0) return;
  if (V <= 256 * 16)
    LAUNCH(KC_CE, rows, 256, (k_cross_entropy_reg<T, 16>), logits, tgt, tgt_stride, Tn, loss_rows, V, inv_ntok);
  else
    LAUNCH(KC_CE, rows, 1024, k_cross_entropy<T>, logits, tgt, tgt_stride, Tn, loss_rows, V, inv_ntok);
}
void sum_rows_f64(const Launch& L, const double* x, int n, double* out) {
  LAUNCH(KC_VEC, 1, 1024, k_sum_rows, x, n, out);
}
template <class T>
void rope(const Launch& L, T* x, int64_t ld, int rows, int Tn, int heads, int hd, const T* cs, const T* sn,
          bool inverse) {
  const int64_t n = (int64_t)rows * heads * (hd / 2);
  if (n == 0) return;
  LAUNCH(KC_ELEM, grid_for(n, 256), 256, k_rope<T>, x, ld, rows, Tn, heads, hd, cs, sn, inverse);
}
template <class T>
void swiglu_fwd(const Launch& L, const T* ab, T* f, int rows, int F) {
  const int64_t n = (int64_t)rows * F;
  if (n == 0) return;
  LAUNCH(KC_ELEM, grid_for(n, 256), 256, k_swiglu_fwd<T>, ab, f, rows, F);
}
template <class T>
void swiglu_bwd(const Launch& L, const T* df, const T* ab, T* dab, int rows, int F) {
  const int64_t n = (int64_t)rows * F;
  if (n == 0) return;
  LAUNCH(KC_ELEM, grid_for(n, 256), 256, k_swiglu_bwd<T>, df, ab, dab, rows, F);
}
template <class T>
void add_inplace(const Launch& L, T* y, const T* x, int64_t n) {
  if (n == 0) return;
  LAUNCH(KC_ELEM, grid_for(n, 256), 256, k_add<T>, y, x, n);
}

#define INST(T)                                                                                                 \
  template void convert_f32<T>(const Launch&, const float*, T*, int64_t);                                       \
  template void embed_fwd<T>(const Launch&, const int32_t*, int, int, int, const T*, const T*, T*, int);        \
  template void embed_bwd_rows<T>(const Launch&, const EmbedCSR&, const T*, T*, int, int, bool);             \
  template void pos_bwd<T>(const Launch&, const T*, T*, int, int, int);                                         \
  template void layernorm_fwd<T>(const Launch&, const T*, const T*, const T*, T*, T*, T*, int, int, double);    \
  template void layernorm_bwd<T>(const Launch&, const T*, const T*, const T*, const T*, const T*, const T*, T*, \
                                 int, int);                                                                     \
  template void rmsnorm_fwd<T>(const Launch&, const T*, const T*, T*, T*, int, int, double);                    \
  template void rmsnorm_bwd<T>(const Launch&, const T*, const T*, const T*, const T*, const T*, T*, int, int);   \
  template void colreduce<T>(const Launch&, int, const T*, int64_t, const T*, const T*, const T*, T*, T*, int,  \
                             int, bool);                                                                        \
  template void softmax_causal_fwd<T>(const Launch&, T*, int64_t, int);                                         \
  template void softmax_bwd<T>(const Launch&, const T*, T*, int64_t, int);                                      \
  template void cross_entropy<T>(const Launch&, T*, const int32_t*, int, int, double*, int, int, double);       \
  template void rope<T>(const Launch&, T*, int64_t, int, int, int, int, const T*, const T*, bool);              \
  template void swiglu_fwd<T>(const Launch&, const T*, T*, int, int);                                           \
  template void swiglu_bwd<T>(const Launch&, const T*, const T*, T*, int, int);                                 \
  template void add_inplace<T>(const Launch&, T*, const T*, int64_t);

INST(double)
INST(float)

}  // namespace slq
