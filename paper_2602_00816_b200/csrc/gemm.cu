// Dense contractions of the fp32 pass mode: a register-blocked SIMT GEMM, double-buffered
// through shared memory, with the layer epilogues fused and a deterministic split-K.  (The fp64
// parity passes use the DMMA kernels in gemm_f64.cu.)
#include <cuda_runtime.h>

#include "gemm_common.cuh"

namespace slq {

namespace {

using namespace gemm_detail;

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

}  // namespace

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
  if constexpr (sizeof(T) == 4) {
    if ((L.gemm_mode == 1 || L.gemm_mode == 3) && a.batch == 1 && a.K > 0) {
      gemm_tc_bf16x3(L, a, L.gemm_mode == 3 ? 1 : 3);
      return;
    }
  }
  if (ak && bk) launch_cfg<T, true, true>(L, a);
  else if (ak && !bk) launch_cfg<T, true, false>(L, a);
  else if (!ak && bk) launch_cfg<T, false, true>(L, a);
  else launch_cfg<T, false, false>(L, a);
}

template void gemm<float>(const Launch&, const GemmArgs<float>&);

template <>
size_t gemm_ws_bytes<float>(const Launch& L, const GemmArgs<float>& a) {
  if (a.M == 0 || a.N == 0) return 0;
  if ((L.gemm_mode == 1 || L.gemm_mode == 3) && a.batch == 1 && a.K > 0)
    return tc_ws_bytes(a.M, a.N, a.K, L.gemm_mode == 3 ? 1 : 3);
  constexpr int BM = 64, BN = 64, BK = 16;  // launch_cfg's decisions
  const int tiles = (int)(ceil_div(a.M, BM) * ceil_div(a.N, BN)) * a.batch;
  int splits = 1;
  if (a.batch == 1 && a.tri == TRI_NONE && tiles < 2 * 148 && a.K >= 512) {
    splits = (int)ceil_div(2 * 148, tiles);
    splits = std::min<int>(splits, (int)(a.K / 256));
    splits = std::max(1, std::min(splits, 32));
  }
  const int kchunk = (int)ceil_div(ceil_div(a.K, splits), BK) * BK;
  splits = (int)ceil_div(a.K, kchunk);
  return splits > 1 ? sizeof(float) * (size_t)splits * a.M * a.N : 0;
}

}  // namespace slq
