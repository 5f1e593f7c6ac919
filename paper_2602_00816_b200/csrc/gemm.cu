// Dense contractions of the two gradient passes for the fp64 / fp32 pass
// modes.  tcgen05 has no fp64 kind, so the fp64 parity passes run on the FP64 pipe: a
// register-blocked SIMT GEMM, double-buffered through shared memory, with the layer epilogues
// fused (bias, residual add, GELU / tanh and their derivatives) and a deterministic split-K for
// the weight-gradient contractions over tokens (K = tokens >> M, N).
#include <cuda_runtime.h>
#include <stdlib.h>

#include "kernels.h"

namespace slq {

namespace {

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

// BM x BN tile per CTA, BK-deep k-slices double-buffered in smem, TM x TN outputs per thread.
// AK: A is K-contiguous (sAk == 1) else M-contiguous;  BKm: B is K-contiguous else N-contiguous.
template <class T, int BM, int BN, int BK, int TM, int TN, bool AK, bool BKm>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    gemm_kernel(GemmArgs<T> p, int splits, int kchunk, T* __restrict__ ws) {
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int ALD = BM * BK / NT;
  constexpr int BLD = BN * BK / NT;
  static_assert(ALD * NT == BM * BK && BLD * NT == BN * BK, "tile/threads");
  __shared__ T As[2][BK][BM + 1];
  __shared__ T Bs[2][BK][BN + 1];

  const int tid = threadIdx.x;
  const int tx = tid % (BN / TN), ty = tid / (BN / TN);
  const int z = blockIdx.z / splits, split = blockIdx.z % splits;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (p.tri == TRI_SKIP_UPPER && n0 > m0 + BM - 1) return;
  const T* __restrict__ A = p.A + boff(p.offA, z);
  const T* __restrict__ B = p.B + boff(p.offB, z);
  int kb = split * kchunk;
  int ke = min(p.K, kb + kchunk);
  if (p.tri == TRI_K_LE_M) ke = min(ke, m0 + BM);
  if (p.tri == TRI_K_GE_M) kb = max(kb, m0);

  T ra[ALD], rb[BLD];
  auto gload = [&](int k0) {
#pragma unroll
    for (int i = 0; i < ALD; ++i) {
      const int idx = tid + i * NT;
      int m, k;
      if (AK) { m = idx / BK; k = idx % BK; } else { m = idx % BM; k = idx / BM; }
      const int gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < p.M && gk < ke) ? A[(int64_t)gm * p.sAm + (int64_t)gk * p.sAk] : T(0);
    }
#pragma unroll
    for (int i = 0; i < BLD; ++i) {
      const int idx = tid + i * NT;
      int n, k;
      if (BKm) { n = idx / BK; k = idx % BK; } else { n = idx % BN; k = idx / BN; }
      const int gn = n0 + n, gk = k0 + k;
      rb[i] = (gn < p.N && gk < ke) ? B[(int64_t)gk * p.sBk + (int64_t)gn * p.sBn] : T(0);
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int i = 0; i < ALD; ++i) {
      const int idx = tid + i * NT;
      int m, k;
      if (AK) { m = idx / BK; k = idx % BK; } else { m = idx % BM; k = idx / BM; }
      As[buf][k][m] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < BLD; ++i) {
      const int idx = tid + i * NT;
      int n, k;
      if (BKm) { n = idx / BK; k = idx % BK; } else { n = idx % BN; k = idx / BN; }
      Bs[buf][k][n] = rb[i];
    }
  };

  T acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = T(0);

  if (kb < ke) {
    gload(kb);
    sstore(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = kb; k0 < ke; k0 += BK) {
      const bool more = k0 + BK < ke;
      if (more) gload(k0 + BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        T a[TM], b[TN];
#pragma unroll
        for (int i = 0; i < TM; ++i) a[i] = As[buf][kk][ty * TM + i];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[j] = Bs[buf][kk][tx * TN + j];
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
      }
      if (more) sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  if (splits > 1) {
    T* W = ws + (int64_t)split * p.M * p.N;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int m = m0 + ty * TM + i;
      if (m >= p.M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int n = n0 + tx * TN + j;
        if (n < p.N) W[(int64_t)m * p.N + n] = acc[i][j];
      }
    }
    return;
  }
  T* C = p.C + boff(p.offC, z);
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + ty * TM + i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tx * TN + j;
      if (n < p.N) epilogue_store(p, C, m, n, acc[i][j]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// fp64 tensor-core path: mma.sync m8n8k4 f64 (DMMA; measured 37 TFLOP/s on B200 vs 34 for DFMA).
// CTA tile BM x BN, 4 warps in 2 x 2, warp tile (BM/2) x (BN/2) of 8x8 DMMA tiles; BK = 16;
// STAGES-deep cp.async pipeline.  Each operand is staged in smem in its global layout (so the
// copies are straight, coalesced 8-byte cp.async) with a 4-double row pad that makes the
// fragment reads bank-conflict free: K-contiguous -> [row][k] ld 20, else [k][row] ld BM+4.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int bytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BM, int BN, bool AK, bool BKm, int NSTAGE>
struct DmmaCfg {
  static constexpr int BK = 16, STAGES = NSTAGE, THREADS = 128;
  static constexpr int LDA = AK ? BK + 4 : BM + 4;   // [m][k] or [k][m]
  static constexpr int LDB = BKm ? BK + 4 : BN + 4;  // [n][k] or [k][n]
  static constexpr int A_ELEMS = AK ? BM * LDA : BK * LDA;
  static constexpr int B_ELEMS = BKm ? BN * LDB : BK * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = sizeof(double) * STAGE * STAGES;
};

template <int BM, int BN, bool AK, bool BKm, int NSTAGE>
__global__ void __launch_bounds__(128) gemm_dmma_kernel(GemmArgs<double> p, int splits, int kchunk,
                                                        double* __restrict__ ws) {
  using C = DmmaCfg<BM, BN, AK, BKm, NSTAGE>;
  constexpr int BK = C::BK, S = C::STAGES;
  constexpr int WM = BM / 2, WN = BN / 2, TM = WM / 8, TN = WN / 8;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane / 4, t = lane % 4;
  const int wm = warp / 2, wn = warp % 2;
  const int z = blockIdx.z / splits, split = blockIdx.z % splits;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  if (p.tri == TRI_SKIP_UPPER && n0 > m0 + BM - 1) return;
  const double* __restrict__ A = p.A + boff(p.offA, z);
  const double* __restrict__ B = p.B + boff(p.offB, z);
  int kb = split * kchunk;
  int ke = min(p.K, kb + kchunk);
  if (p.tri == TRI_K_LE_M) ke = min(ke, m0 + BM);
  if (p.tri == TRI_K_GE_M) kb = max(kb, m0);
  const int nk = kb < ke ? (ke - kb + BK - 1) / BK : 0;

  auto load_tile = [&](int kt, int stage) {
    double* As = smem + stage * C::STAGE;
    double* Bs = As + C::A_ELEMS;
    const int k0 = kb + kt * BK;
#pragma unroll
    for (int i = tid; i < BM * BK; i += C::THREADS) {
      int m, k;
      if (AK) { m = i / BK; k = i % BK; } else { m = i % BM; k = i / BM; }
      const int gm = m0 + m, gk = k0 + k;
      const bool ok = gm < p.M && gk < ke;
      const double* src = ok ? A + (int64_t)gm * p.sAm + (int64_t)gk * p.sAk : A;
      cp_async8(AK ? &As[m * C::LDA + k] : &As[k * C::LDA + m], src, ok);
    }
#pragma unroll
    for (int i = tid; i < BN * BK; i += C::THREADS) {
      int n, k;
      if (BKm) { n = i / BK; k = i % BK; } else { n = i % BN; k = i / BN; }
      const int gn = n0 + n, gk = k0 + k;
      const bool ok = gn < p.N && gk < ke;
      const double* src = ok ? B + (int64_t)gk * p.sBk + (int64_t)gn * p.sBn : B;
      cp_async8(BKm ? &Bs[n * C::LDB + k] : &Bs[k * C::LDB + n], src, ok);
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < nk) load_tile(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<S - 2>();
    __syncthreads();
    if (kt + S - 1 < nk) load_tile(kt + S - 1, (kt + S - 1) % S);
    cp_async_commit();
    const double* As = smem + (kt % S) * C::STAGE;
    const double* Bs = As + C::A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int m = wm * WM + i * 8 + g, k = ks + t;
        a[i] = AK ? As[m * C::LDA + k] : As[k * C::LDA + m];
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int n = wn * WN + j * 8 + g, k = ks + t;
        b[j] = BKm ? Bs[n * C::LDB + k] : Bs[k * C::LDB + n];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  double* C_ = splits > 1 ? ws + (int64_t)split * p.M * p.N : p.C + boff(p.offC, z);
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = m0 + wm * WM + i * 8 + g;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int n = n0 + wn * WN + j * 8 + 2 * t + h;
        if (n >= p.N) continue;
        if (splits > 1)
          C_[(int64_t)m * p.N + n] = acc[i][j][h];
        else
          epilogue_store(p, C_, m, n, acc[i][j][h]);
      }
    }
  }
}

template <class T>
__global__ void splitk_reduce(GemmArgs<T> p, int splits, const T* __restrict__ ws) {
  const int64_t mn = (int64_t)p.M * p.N;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < mn; i += (int64_t)gridDim.x * blockDim.x) {
    T s = T(0);
    for (int k = 0; k < splits; ++k) s += ws[k * mn + i];
    epilogue_store(p, p.C, (int)(i / p.N), (int)(i % p.N), s);
  }
}

template <class T, bool AK, bool BKm>
void launch_cfg(const Launch& L, const GemmArgs<T>& a) {
  constexpr int BM = 64, BN = 64, BK = 16, TM = 4, TN = 4;
  const int tiles_m = (int)ceil_div(a.M, BM), tiles_n = (int)ceil_div(a.N, BN);
  const int tiles = tiles_m * tiles_n * a.batch;
  int splits = 1;
  if (a.batch == 1 && a.tri == TRI_NONE && tiles < 2 * 148 && a.K >= 512) {
    splits = (int)ceil_div(2 * 148, tiles);
    splits = std::min<int>(splits, (int)(a.K / 256));
    splits = std::max(1, std::min(splits, 32));
  }
  int kchunk = (int)ceil_div(ceil_div(a.K, splits), BK) * BK;
  splits = (int)ceil_div(a.K, kchunk);
  T* ws = nullptr;
  if (splits > 1) ws = (T*)L.ws->get(sizeof(T) * (size_t)splits * a.M * a.N, L.stream);
  dim3 grid(tiles_n, tiles_m, a.batch * splits);
  LaunchScope scope(L.prof, KC_GEMM, L.stream, 2.0 * a.M * a.N * (double)a.K * a.batch,
                    sizeof(T) * ((double)a.M * a.K + (double)a.K * a.N + (double)a.M * a.N) * a.batch);
  gemm_kernel<T, BM, BN, BK, TM, TN, AK, BKm><<<grid, (BM / TM) * (BN / TN), 0, L.stream>>>(a, splits, kchunk, ws);
  SLQ_CUDA(cudaGetLastError());
  ++*L.launches;
  if (splits > 1) {
    const int64_t mn = (int64_t)a.M * a.N;
    int blocks = (int)std::min<int64_t>(ceil_div(mn, 256), 148 * 8);
    splitk_reduce<T><<<blocks, 256, 0, L.stream>>>(a, splits, ws);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
}

// algorithmic FLOPs of a (possibly causal-structured) GEMM
double gemm_flops(const GemmArgs<double>& a, int BM) {
  double f = 2.0 * a.M * a.N * (double)a.K * a.batch;
  if (a.tri != TRI_NONE && a.M > 0) f *= std::min(1.0, (a.M + (double)BM) / (2.0 * a.M));
  return f;
}

template <int BM, int BN, bool AK, bool BKm, int NSTAGE>
void launch_dmma(const Launch& L, const GemmArgs<double>& a) {
  using C = DmmaCfg<BM, BN, AK, BKm, NSTAGE>;
  static bool attr_set = false;
  if (!attr_set) {
    SLQ_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel<BM, BN, AK, BKm, NSTAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)C::SMEM));
    attr_set = true;
  }
  const int tiles_m = (int)ceil_div(a.M, BM), tiles_n = (int)ceil_div(a.N, BN);
  const int tiles = tiles_m * tiles_n * a.batch;
  int splits = 1;
  if (a.batch == 1 && a.tri == TRI_NONE && tiles < 2 * 148 && a.K >= 256) {
    splits = (int)ceil_div(2 * 148, tiles);
    splits = std::min<int>(splits, (int)(a.K / 128));
    splits = std::max(1, std::min(splits, 32));
  }
  const int kchunk = (int)ceil_div(ceil_div(a.K, splits), C::BK) * C::BK;
  splits = std::max(1, (int)ceil_div(a.K, kchunk));
  double* ws = nullptr;
  if (splits > 1) ws = (double*)L.ws->get(sizeof(double) * (size_t)splits * a.M * a.N, L.stream);
  dim3 grid(tiles_n, tiles_m, a.batch * splits);
  LaunchScope scope(L.prof, KC_GEMM, L.stream, gemm_flops(a, BM),
                    8.0 * ((double)a.M * a.K + (double)a.K * a.N + (double)a.M * a.N) * a.batch);
  gemm_dmma_kernel<BM, BN, AK, BKm, NSTAGE><<<grid, C::THREADS, C::SMEM, L.stream>>>(a, splits, kchunk, ws);
  SLQ_CUDA(cudaGetLastError());
  ++*L.launches;
  if (splits > 1) {
    const int64_t mn = (int64_t)a.M * a.N;
    int blocks = (int)std::min<int64_t>(ceil_div(mn, 256), 148 * 8);
    splitk_reduce<double><<<blocks, 256, 0, L.stream>>>(a, splits, ws);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
}

int dmma_stages() {
  static int s = [] {
    const char* e = getenv("SLQ_DMMA_STAGES");
    return (e && atoi(e) == 2) ? 2 : 3;
  }();
  return s;
}

template <bool AK, bool BKm>
void dmma_dispatch(const Launch& L, const GemmArgs<double>& a) {
  const int stages = dmma_stages();
  const int64_t t64 = ceil_div(a.M, 64) * ceil_div(a.N, 64) * a.batch;
  if (t64 >= 148 || (a.batch == 1 && a.K >= 256)) {
    if (stages == 2) launch_dmma<64, 64, AK, BKm, 2>(L, a);
    else launch_dmma<64, 64, AK, BKm, 3>(L, a);
  } else if (a.N >= a.M) {
    if (stages == 2) launch_dmma<32, 64, AK, BKm, 2>(L, a);
    else launch_dmma<32, 64, AK, BKm, 3>(L, a);
  } else {
    if (stages == 2) launch_dmma<64, 32, AK, BKm, 2>(L, a);
    else launch_dmma<64, 32, AK, BKm, 3>(L, a);
  }
}

}  // namespace

template <>
void gemm<double>(const Launch& L, const GemmArgs<double>& a) {
  SLQ_CHECK_ARG(a.M >= 0 && a.N >= 0 && a.K >= 0 && a.batch >= 1, "gemm dims");
  if (a.M == 0 || a.N == 0) return;
  SLQ_CHECK_ARG(a.sAk == 1 || a.sAm == 1, "gemm A layout");
  SLQ_CHECK_ARG(a.sBk == 1 || a.sBn == 1, "gemm B layout");
  SLQ_CHECK_ARG(a.batch == 1 || (!a.resid && !a.aux && !a.C2), "batched gemm epilogue");
  SLQ_CHECK_ARG(a.act != ACT_GELU || a.C2, "GELU epilogue needs C2");
  SLQ_CHECK_ARG((a.act != ACT_DGELU && a.act != ACT_DTANH) || a.aux, "derivative epilogue needs aux");
  const bool ak = a.sAk == 1 && !(a.sAm == 1 && a.K == 1);
  const bool bk = a.sBk == 1 && !(a.sBn == 1 && a.K == 1);
  if (ak && bk) dmma_dispatch<true, true>(L, a);
  else if (ak && !bk) dmma_dispatch<true, false>(L, a);
  else if (!ak && bk) dmma_dispatch<false, true>(L, a);
  else dmma_dispatch<false, false>(L, a);
}

template <class T>
void gemm(const Launch& L, const GemmArgs<T>& a) {
  SLQ_CHECK_ARG(a.M >= 0 && a.N >= 0 && a.K >= 0 && a.batch >= 1, "gemm dims");
  if (a.M == 0 || a.N == 0) return;
  SLQ_CHECK_ARG(a.sAk == 1 || a.sAm == 1, "gemm A layout");
  SLQ_CHECK_ARG(a.sBk == 1 || a.sBn == 1, "gemm B layout");
  SLQ_CHECK_ARG(a.batch == 1 || (!a.resid && !a.aux && !a.C2), "batched gemm epilogue");
  SLQ_CHECK_ARG(a.act != ACT_GELU || a.C2, "GELU epilogue needs C2");
  SLQ_CHECK_ARG((a.act != ACT_DGELU && a.act != ACT_DTANH) || a.aux, "derivative epilogue needs aux");
  const bool ak = a.sAk == 1 && !(a.sAm == 1 && a.K == 1);
  const bool bk = a.sBk == 1 && !(a.sBn == 1 && a.K == 1);
  if (ak && bk) launch_cfg<T, true, true>(L, a);
  else if (ak && !bk) launch_cfg<T, true, false>(L, a);
  else if (!ak && bk) launch_cfg<T, false, true>(L, a);
  else launch_cfg<T, false, false>(L, a);
}

template void gemm<float>(const Launch&, const GemmArgs<float>&);

}  // namespace slq
