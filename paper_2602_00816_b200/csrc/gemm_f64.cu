// fp64 contractions of the parity gradient passes on the FP64 tensor core:
// mma.sync.m8n8k4.f64 (DMMA; measured 37 TFLOP/s on B200 vs 34 for DFMA; tcgen05 has no fp64 kind).
//
// CTA tile BM x BN, WGM x WGN warps, warp tile (BM/WGM) x (BN/WGN) of 8x8 DMMA tiles; BK-deep
// k-slices through a STAGES-deep cp.async pipeline.  Each operand is staged in shared memory in
// its global layout (straight, coalesced 8-byte cp.async) with a row pitch = 4 (mod 16) doubles,
// which makes the DMMA fragment reads bank-conflict free: K-contiguous -> [row][k], else [k][row].
// Epilogues (bias, residual, GELU / tanh and derivatives, accumulate) are fused; the weight-
// gradient contractions over tokens (K >> M, N) use a deterministic split-K.
#include <cuda_runtime.h>
#include <stdlib.h>

#include <vector>

#include "gemm_common.cuh"

namespace slq {

namespace {

using namespace gemm_detail;

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
// 16-byte variant: copies `bytes` (0, 8 or 16) and zero-fills the rest of the 16-byte destination
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BM_, int BN_, int BK_, int WGM_, int WGN_, int STAGES_>
struct Tile {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WGM = WGM_, WGN = WGN_, STAGES = STAGES_;
  static constexpr int THREADS = 32 * WGM * WGN;
  static constexpr int WM = BM / WGM, WN = BN / WGN, TM = WM / 8, TN = WN / 8;
  static_assert(TM >= 1 && TN >= 1 && WM % 8 == 0 && WN % 8 == 0, "warp tile");
};

template <class TL, bool AK, bool BKm>
struct Smem {
  static constexpr int LDA = AK ? TL::BK + 4 : TL::BM + 4;
  static constexpr int LDB = BKm ? TL::BK + 4 : TL::BN + 4;
  static constexpr int A_ELEMS = AK ? TL::BM * LDA : TL::BK * LDA;
  static constexpr int B_ELEMS = BKm ? TL::BN * LDB : TL::BK * LDB;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr int PIPE = STAGE * TL::STAGES;
  static constexpr int CTILE = TL::BM * (TL::BN + 1);  // epilogue staging tile
  static constexpr size_t BYTES = sizeof(double) * (PIPE > CTILE ? PIPE : CTILE);
};

template <class TL, bool AK, bool BKm>
__global__ void __launch_bounds__(TL::THREADS, TL::THREADS == 128 ? (TL::BK >= 32 ? 2 : TL::BM * TL::BN >= 4096 ? 3 : 4) : (TL::THREADS == 256 && TL::BM * TL::BN <= 4096 ? 3 : 1)) gemm_dmma_kernel(GemmArgs<double> p, int splits, int kchunk,
                                                                double* __restrict__ ws, unsigned* __restrict__ cnt) {
  using SM = Smem<TL, AK, BKm>;
  constexpr int BM = TL::BM, BN = TL::BN, BK = TL::BK, S = TL::STAGES;
  constexpr int WM = TL::WM, WN = TL::WN, TM = TL::TM, TN = TL::TN;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int g = lane / 4, t = lane % 4;
  const int wm = warp / TL::WGN, wn = warp % TL::WGN;
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

  // 16-byte copies of element pairs along each operand's contiguous axis when the global strides
  // and bases allow it (pairs are aligned and a pair's validity is a prefix: first, or both)
  const bool vecA = AK ? ((p.sAm % 2) == 0 && ((uintptr_t)A % 16) == 0)
                       : ((p.sAk % 2) == 0 && ((uintptr_t)A % 16) == 0);
  const bool vecB = BKm ? ((p.sBn % 2) == 0 && ((uintptr_t)B % 16) == 0)
                        : ((p.sBk % 2) == 0 && ((uintptr_t)B % 16) == 0);
  auto load_tile = [&](int kt, int stage) {
    double* As = smem + stage * SM::STAGE;
    double* Bs = As + SM::A_ELEMS;
    const int k0 = kb + kt * BK;
    if (vecA) {
#pragma unroll
      for (int i = tid; i < BM * BK / 2; i += TL::THREADS) {
        int m, k;
        if (AK) { m = i / (BK / 2); k = 2 * (i % (BK / 2)); } else { m = 2 * (i % (BM / 2)); k = i / (BM / 2); }
        const int gm = m0 + m, gk = k0 + k;
        // elements (gm, gk) and the next along the contiguous axis
        const int n_ok = AK ? (gm < p.M ? max(0, min(2, ke - gk)) : 0) : (gk < ke ? max(0, min(2, p.M - gm)) : 0);
        const double* src = n_ok ? A + (int64_t)gm * p.sAm + (int64_t)gk * p.sAk : A;
        cp_async16(AK ? &As[m * SM::LDA + k] : &As[k * SM::LDA + m], src, 8 * n_ok);
      }
    } else {
#pragma unroll
      for (int i = tid; i < BM * BK; i += TL::THREADS) {
        int m, k;
        if (AK) { m = i / BK; k = i % BK; } else { m = i % BM; k = i / BM; }
        const int gm = m0 + m, gk = k0 + k;
        const bool ok = gm < p.M && gk < ke;
        const double* src = ok ? A + (int64_t)gm * p.sAm + (int64_t)gk * p.sAk : A;
        cp_async8(AK ? &As[m * SM::LDA + k] : &As[k * SM::LDA + m], src, ok);
      }
    }
    if (vecB) {
#pragma unroll
      for (int i = tid; i < BN * BK / 2; i += TL::THREADS) {
        int n, k;
        if (BKm) { n = i / (BK / 2); k = 2 * (i % (BK / 2)); } else { n = 2 * (i % (BN / 2)); k = i / (BN / 2); }
        const int gn = n0 + n, gk = k0 + k;
        const int n_ok = BKm ? (gn < p.N ? max(0, min(2, ke - gk)) : 0) : (gk < ke ? max(0, min(2, p.N - gn)) : 0);
        const double* src = n_ok ? B + (int64_t)gk * p.sBk + (int64_t)gn * p.sBn : B;
        cp_async16(BKm ? &Bs[n * SM::LDB + k] : &Bs[k * SM::LDB + n], src, 8 * n_ok);
      }
    } else {
#pragma unroll
      for (int i = tid; i < BN * BK; i += TL::THREADS) {
        int n, k;
        if (BKm) { n = i / BK; k = i % BK; } else { n = i % BN; k = i / BN; }
        const int gn = n0 + n, gk = k0 + k;
        const bool ok = gn < p.N && gk < ke;
        const double* src = ok ? B + (int64_t)gk * p.sBk + (int64_t)gn * p.sBn : B;
        cp_async8(BKm ? &Bs[n * SM::LDB + k] : &Bs[k * SM::LDB + n], src, ok);
      }
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
    const double* As = smem + (kt % S) * SM::STAGE;
    const double* Bs = As + SM::A_ELEMS;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int m = wm * WM + i * 8 + g, k = ks + t;
        a[i] = AK ? As[m * SM::LDA + k] : As[k * SM::LDA + m];
      }
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int n = wn * WN + j * 8 + g, k = ks + t;
        b[j] = BKm ? Bs[n * SM::LDB + k] : Bs[k * SM::LDB + n];
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // Epilogue: stage the accumulator tile in shared memory (reusing the pipeline buffers), then
  // one compact loop applies the fused epilogue with row-contiguous, coalesced global stores.
  // (Inlining the epilogue per accumulator register blew the kernel up to ~15k instructions and
  // made instruction fetch the top stall.)
  constexpr int LDC = BN + 1;
  double* Cs = smem;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int r = wm * WM + i * 8 + g, c = wn * WN + j * 8 + 2 * t;
      Cs[r * LDC + c] = acc[i][j][0];
      Cs[r * LDC + c + 1] = acc[i][j][1];
    }
  __syncthreads();
  double* C_ = splits > 1 ? ws + ((int64_t)z * splits + split) * p.M * p.N : p.C + boff(p.offC, z);
  const int rows = min(BM, p.M - m0), cols = min(BN, p.N - n0);
  // column pairs; 16-byte accesses when every pitch is even and every base 16-byte aligned
  const int64_t ldo = splits > 1 ? p.N : p.ldc;
  auto al = [](const void* q) { return ((uintptr_t)q & 15) == 0; };
  const bool plain = splits > 1 || (!p.bias && !p.resid && !p.aux && !p.accumulate && p.act == ACT_NONE &&
                                    p.alpha == 1.0);
  const bool vec = (ldo % 2) == 0 && al(C_) && (!p.bias || al(p.bias)) &&
                   (splits > 1 || ((!p.resid || ((p.ldr % 2) == 0 && al(p.resid))) &&
                                   (!p.aux || ((p.ldaux % 2) == 0 && al(p.aux))) &&
                                   (!p.C2 || ((p.ldc2 % 2) == 0 && al(p.C2)))));
  if (plain) {
#pragma unroll 4
    for (int e = tid; e < BM * BN / 2; e += TL::THREADS) {
      const int r = e / (BN / 2), c = 2 * (e % (BN / 2));
      if (r >= rows || c >= cols) continue;
      double* dst = C_ + (int64_t)(m0 + r) * ldo + n0 + c;
      const double v0 = Cs[r * LDC + c], v1 = Cs[r * LDC + c + 1];
      if (c + 1 < cols && vec) {
        *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
      } else {
        dst[0] = v0;
        if (c + 1 < cols) dst[1] = v1;
      }
    }
    if (splits == 1 || !cnt) return;
    // split-K reduction in the last CTA of the tile to arrive (threadfence + per-tile counter):
    // it sums the splits' partials in split order 0..splits-1 -- the order of splitk_reduce, so
    // the result does not depend on which CTA arrives last -- and applies the fused epilogue
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    const int64_t tile = ((int64_t)z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    if (tid == 0) last = atomicAdd(cnt + tile, 1u) == (unsigned)splits - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int64_t mn = (int64_t)p.M * p.N;
    const double* part = ws + (int64_t)z * splits * mn;
    double* Cz = p.C + boff(p.offC, z);
    const bool vc = (p.ldc % 2) == 0 && al(Cz) && (!p.bias || al(p.bias)) &&
                    (!p.resid || ((p.ldr % 2) == 0 && al(p.resid))) &&
                    (!p.aux || ((p.ldaux % 2) == 0 && al(p.aux))) &&
                    (!p.C2 || ((p.ldc2 % 2) == 0 && al(p.C2)));
#pragma unroll 1
    for (int e = tid; e < BM * BN / 2; e += TL::THREADS) {
      const int r = e / (BN / 2), c = 2 * (e % (BN / 2));
      if (r >= rows || c >= cols) continue;
      const int64_t o = (int64_t)(m0 + r) * p.N + n0 + c;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll 4
      for (int k = 0; k < splits; ++k) {
        s0 += __ldcg(part + k * mn + o);
        if (c + 1 < cols) s1 += __ldcg(part + k * mn + o + 1);
      }
      if (c + 1 < cols) epilogue_store2(p, Cz, m0 + r, n0 + c, s0, s1, vc);
      else epilogue_store(p, Cz, m0 + r, n0 + c, s0);
    }
    if (tid == 0) cnt[tile] = 0u;  // ready for the next launch on this stream
    return;
  }
#pragma unroll 1
  for (int e = tid; e < BM * BN / 2; e += TL::THREADS) {
    const int r = e / (BN / 2), c = 2 * (e % (BN / 2));
    if (r >= rows || c >= cols) continue;
    if (c + 1 < cols) {
      epilogue_store2(p, C_, m0 + r, n0 + c, Cs[r * LDC + c], Cs[r * LDC + c + 1], vec);
    } else {
      epilogue_store(p, C_, m0 + r, n0 + c, Cs[r * LDC + c]);
    }
  }
}

// algorithmic FLOPs of a (possibly causal-structured) GEMM
double gemm_flops(const GemmArgs<double>& a) {
  double f = 2.0 * a.M * a.N * (double)a.K * a.batch;
  if (a.tri != TRI_NONE && a.M > 0) f *= std::min(1.0, (a.M + 64.0) / (2.0 * a.M));
  return f;
}

// auto split-K: fill ~2 waves of CTAs when the tile grid is small and K is long
int choose_splits(const GemmArgs<double>& a, int tiles, int forced, int BK) {
  if (forced > 0) return forced;
  static const int min_k = getenv("SLQ_DMMA_SPLIT_MIN_K") ? atoi(getenv("SLQ_DMMA_SPLIT_MIN_K")) : 256;
  static const int waves = getenv("SLQ_DMMA_SPLIT_WAVES") ? atoi(getenv("SLQ_DMMA_SPLIT_WAVES")) : 2;
  // batched: only the long-K weight-gradient batches (attention batches keep their tuned plans)
  if ((a.batch != 1 && a.K < 2048) || a.tri != TRI_NONE || a.K < min_k || tiles >= waves * 148) return 1;
  int s = (int)ceil_div(waves * 148, tiles);
  s = std::min<int>(s, (int)(a.K / (4 * BK)));
  return std::max(1, std::min(s, 32));
}

template <class TL, bool AK, bool BKm>
void launch(const Launch& L, const GemmArgs<double>& a, int forced_splits) {
  using SM = Smem<TL, AK, BKm>;
  static bool attr_set = false;
  if (!attr_set) {
    SLQ_CUDA(cudaFuncSetAttribute(gemm_dmma_kernel<TL, AK, BKm>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)SM::BYTES));
    attr_set = true;
  }
  const int tiles_m = (int)ceil_div(a.M, TL::BM), tiles_n = (int)ceil_div(a.N, TL::BN);
  int splits = choose_splits(a, tiles_m * tiles_n * a.batch, forced_splits, TL::BK);
  const int kchunk = (int)ceil_div(ceil_div(a.K, splits), TL::BK) * TL::BK;
  splits = std::max(1, (int)ceil_div(a.K, kchunk));
  double* ws = nullptr;
  unsigned* cnt = nullptr;
  if (splits > 1) {
    ws = (double*)L.ws->get(sizeof(double) * (size_t)splits * a.M * a.N * a.batch, L.stream);
    static const bool ext = getenv("SLQ_DMMA_SPLIT_EXT") && atoi(getenv("SLQ_DMMA_SPLIT_EXT"));
    if (!ext) cnt = L.ws->counters((size_t)tiles_m * tiles_n * a.batch);
  }
  dim3 grid(tiles_n, tiles_m, a.batch * splits);
  LaunchScope scope(L.prof, KC_GEMM, L.stream, gemm_flops(a),
                    8.0 * ((double)a.M * a.K + (double)a.K * a.N + (double)a.M * a.N) * a.batch);
  gemm_dmma_kernel<TL, AK, BKm><<<grid, TL::THREADS, SM::BYTES, L.stream>>>(a, splits, kchunk, ws, cnt);
  SLQ_CUDA(cudaGetLastError());
  ++*L.launches;
  if (splits > 1 && !cnt) {
    const int64_t mn = (int64_t)a.M * a.N * a.batch;
    int blocks = (int)std::min<int64_t>(ceil_div(mn, 256), 148 * 8);
    splitk_reduce<double><<<blocks, 256, 0, L.stream>>>(a, splits, ws);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
}

// tile variants (the sweep in tools/gemm_sweep.py picks the heuristic below)
using V0 = Tile<64, 64, 16, 2, 2, 3>;
using V1 = Tile<64, 64, 16, 2, 2, 2>;
using V2 = Tile<64, 64, 32, 2, 2, 2>;
using V3 = Tile<128, 64, 16, 4, 2, 3>;
using V4 = Tile<64, 128, 16, 2, 4, 3>;
using V5 = Tile<128, 128, 16, 2, 4, 2>;
using V6 = Tile<32, 64, 16, 2, 2, 3>;
using V7 = Tile<64, 32, 16, 2, 2, 3>;
using V8 = Tile<128, 64, 32, 4, 2, 2>;
using V9 = Tile<64, 64, 16, 4, 2, 2>;
using V10 = Tile<64, 64, 16, 4, 4, 2>;
using V11 = Tile<64, 32, 16, 4, 2, 3>;
using V12 = Tile<32, 64, 16, 2, 4, 3>;
using V13 = Tile<128, 64, 16, 8, 2, 2>;
using V14 = Tile<64, 64, 32, 4, 4, 2>;
constexpr int kVariants = 15;
constexpr int kVarDims[kVariants][3] = {{64, 64, 16}, {64, 64, 16}, {64, 64, 32}, {128, 64, 16}, {64, 128, 16},
                                        {128, 128, 16}, {32, 64, 16}, {64, 32, 16}, {128, 64, 32}, {64, 64, 16},
                                        {64, 64, 16}, {64, 32, 16}, {32, 64, 16}, {128, 64, 16}, {64, 64, 32}};

template <bool AK, bool BKm>
void launch_variant(const Launch& L, const GemmArgs<double>& a, int v, int splits) {
  switch (v) {
    case 0: launch<V0, AK, BKm>(L, a, splits); break;
    case 1: launch<V1, AK, BKm>(L, a, splits); break;
    case 2: launch<V2, AK, BKm>(L, a, splits); break;
    case 3: launch<V3, AK, BKm>(L, a, splits); break;
    case 4: launch<V4, AK, BKm>(L, a, splits); break;
    case 5: launch<V5, AK, BKm>(L, a, splits); break;
    case 6: launch<V6, AK, BKm>(L, a, splits); break;
    case 7: launch<V7, AK, BKm>(L, a, splits); break;
    case 8: launch<V8, AK, BKm>(L, a, splits); break;
    case 9: launch<V9, AK, BKm>(L, a, splits); break;
    case 10: launch<V10, AK, BKm>(L, a, splits); break;
    case 11: launch<V11, AK, BKm>(L, a, splits); break;
    case 12: launch<V12, AK, BKm>(L, a, splits); break;
    case 13: launch<V13, AK, BKm>(L, a, splits); break;
    default: launch<V14, AK, BKm>(L, a, splits); break;
  }
}

int forced_variant() {
  static int v = [] {
    const char* e = getenv("SLQ_DMMA_VARIANT");
    return e ? atoi(e) : -1;
  }();
  return v;
}

int pick_variant(const GemmArgs<double>& a) {
  const int fv = forced_variant();
  if (fv >= 0 && fv < kVariants) return fv;
  const int64_t t64 = ceil_div(a.M, 64) * ceil_div(a.N, 64) * a.batch;
  if (t64 >= 148 || (a.batch == 1 && a.K >= 256)) return 1;
  return a.N >= a.M ? 6 : 7;
}

// Per-shape plan for the dense (batch 1, non-causal) GEMMs, from the B200 sweep of every tile
// variant x split count on the c2 shapes (tools/gemm_sweep2.py): 64 x 32 tiles with 8 warps and
// no split for the N <= 256, K <= 1024 chain GEMMs (+50% on 2048 x 256 x 256); split-K 8 for
// the token-contracting weight gradients; 32-wide tiles for 2048 x 1024 x 256.  Returns the
// variant and sets *splits (0 = automatic).
int plan_variant(const GemmArgs<double>& a, int* splits) {
  *splits = 0;
  const int fv = forced_variant();
  if (fv >= 0 && fv < kVariants) return fv;
  if (a.batch != 1 || a.tri != TRI_NONE) {
    // batched causal attention GEMMs at T <= 256 (tools/gemm_sweep_attn.py on B200: +12..28%)
    if (a.M <= 256 && a.N <= 256 && a.K <= 64) return 7;
    if (a.M <= 256 && a.N <= 64) return 11;
    // T = 1024 (c3): the K = T contractions (P V, P^T dO, dS K, dS^T Q) on 32 x 64 tiles (+8%,
    // tools/gemm_sweep_attn.py with T=1024 NB=96)
    if (a.N <= 64 && a.K >= 512) return 6;
    return pick_variant(a);
  }
  const double mn = (double)a.M * a.N;
  if (a.K >= 2048) {
    if (mn <= 65536.0) { *splits = 8; return 11; }    // 256 x 256
    if (mn <= 200000.0) { *splits = 3; return 11; }   // 768 x 256
    if (mn <= 300000.0) { *splits = 8; return 7; }    // 1024 x 256, 256 x 1024
    if (mn <= 600000.0) { *splits = 8; return 0; }    // 2048 x 256
    *splits = 4;
    return 1;
  }
  if (a.N <= 256 && a.K <= 1024) { *splits = 1; return 11; }
  if (a.N >= 1024 && a.N <= 2048 && a.K <= 256) { *splits = 1; return 6; }
  return pick_variant(a);
}

void check(const GemmArgs<double>& a) {
  SLQ_CHECK_ARG(a.M >= 0 && a.N >= 0 && a.K >= 0 && a.batch >= 1, "gemm dims");
  SLQ_CHECK_ARG(a.sAk == 1 || a.sAm == 1, "gemm A layout");
  SLQ_CHECK_ARG(a.sBk == 1 || a.sBn == 1, "gemm B layout");
  SLQ_CHECK_ARG(a.batch == 1 || (!a.resid && !a.aux && !a.C2), "batched gemm epilogue");
  SLQ_CHECK_ARG(a.act != ACT_GELU || a.C2, "GELU epilogue needs C2");
  SLQ_CHECK_ARG((a.act != ACT_DGELU && a.act != ACT_DTANH) || a.aux, "derivative epilogue needs aux");
}

// split-K workspace bytes the DMMA launch of variant v takes (the same decisions as launch<>)
size_t dmma_ws_bytes(const GemmArgs<double>& a, int v, int forced) {
  const int BM = kVarDims[v][0], BN = kVarDims[v][1], BK = kVarDims[v][2];
  const int tiles = (int)(ceil_div(a.M, BM) * ceil_div(a.N, BN)) * a.batch;
  int splits = choose_splits(a, tiles, forced, BK);
  const int kchunk = (int)ceil_div(ceil_div(a.K, splits), BK) * BK;
  splits = std::max(1, (int)ceil_div(a.K, kchunk));
  return splits > 1 ? sizeof(double) * (size_t)splits * a.M * a.N * a.batch : 0;
}

void run(const Launch& L, const GemmArgs<double>& a, int v, int splits) {
  const bool ak = a.sAk == 1 && !(a.sAm == 1 && a.K == 1);
  const bool bk = a.sBk == 1 && !(a.sBn == 1 && a.K == 1);
  if (ak && bk) launch_variant<true, true>(L, a, v, splits);
  else if (ak && !bk) launch_variant<true, false>(L, a, v, splits);
  else if (!ak && bk) launch_variant<false, true>(L, a, v, splits);
  else launch_variant<false, false>(L, a, v, splits);
}

__global__ void k_fill(double* x, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    x[i] = (double)((z >> 11) & 0xFFFFF) / 1048576.0 - 0.5;
  }
}

}  // namespace

// Ozaki GEMMs whose digit planes + split-K partials would exceed the workspace caps are cut into
// blocks computed one after the other in the same workspace (the c5 head GEMMs ask for up to 8 GB
// otherwise).  K blocks (plain, scaled or accumulating epilogue only: the blocks accumulate into C)
// cost nothing extra -- every block slices its own K range -- so they are used above 1 GiB; M / N
// blocks (any epilogue) re-slice the other operand for every block, so they are used only above
// 4 GiB (on c3 the M blocks of the head's dgrad re-sliced its 50257 x 768 weight four times,
// 4 ms per step).
constexpr size_t kOzWsCapK = (size_t)1 << 30, kOzWsCapMN = (size_t)4 << 30;
struct OzBlocks {
  int mb, nb, kb;  // block extents
};
bool oz_k_splittable(const GemmArgs<double>& a) {
  return !a.bias && !a.resid && !a.aux && !a.C2 && a.act == ACT_NONE;
}
OzBlocks oz_blocks(const GemmArgs<double>& a, int S) {
  OzBlocks b{a.M, a.N, a.K};
  auto half = [](int x, int q) { return (int)(ceil_div(ceil_div(x, 2), q) * q); };
  const bool ksplit = oz_k_splittable(a);
  for (int it = 0; it < 64; ++it) {
    const size_t ws = oz_ws_bytes(b.mb, b.nb, b.kb, S);
    if (ws <= kOzWsCapK) break;
    if (ksplit && b.kb >= 256) {
      b.kb = half(b.kb, 64);
    } else if (ws > kOzWsCapMN && std::max(b.mb, b.nb) >= 256) {
      if (b.mb >= b.nb) b.mb = half(b.mb, 128);
      else b.nb = half(b.nb, 128);
    } else {
      break;
    }
  }
  return b;
}
// The activation of an int8 Ozaki GEMM runs as a separate elementwise pass: inside the GEMM's
// epilogue the fp64 tanh of GELU cost ~200 instructions per output and made the c3 fc-forward
// GEMM epilogue-bound (22% INT8-pipe activity, 0.63 ms); as a streaming pass it is ~0.06 ms.
//   GELU:  C2 = y (pre-activation, written by the GEMM), C = gelu(C2)
//   TANH:  C = tanh(y)                       DGELU: C = y gelu'(aux)      DTANH: C = y (1 - aux^2)
// the activation pass of the Ozaki GEMMs: each thread owns 4 columns of a row, 256 apart
// (coalesced), and issues all its loads before the first fp64 activation (four independent loads
// in flight per thread: the pass is HBM-bound, and one load per thread left it at ~3.5 TB/s)
template <int ACT>
__global__ void __launch_bounds__(256) k_oz_act(int M, int N, const double* __restrict__ Y, int64_t ldy,
                                                double* __restrict__ C, int64_t ldc, const double* __restrict__ aux,
                                                int64_t ldaux) {
  constexpr bool kAux = ACT == ACT_DGELU || ACT == ACT_DTANH;
  for (int64_t m = blockIdx.y; m < M; m += gridDim.y) {
    const int n0 = blockIdx.x * 1024 + threadIdx.x;
    double y[4], x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = n0 + 256 * i;
      y[i] = n < N ? Y[m * ldy + n] : 0.0;
      x[i] = (kAux && n < N) ? aux[m * ldaux + n] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int n = n0 + 256 * i;
      if (n >= N) continue;
      double out;
      if constexpr (ACT == ACT_GELU) out = gelu_tanh(y[i]);
      else if constexpr (ACT == ACT_TANH) out = tanh(y[i]);
      else if constexpr (ACT == ACT_DGELU) out = y[i] * gelu_tanh_grad(x[i]);
      else out = y[i] * (1.0 - x[i] * x[i]);
      C[m * ldc + n] = out;
    }
  }
}

void gemm_oz_core(const Launch& L, const GemmArgs<double>& a);

void gemm_oz_blocked(const Launch& L, const GemmArgs<double>& a) {
  if (a.act == ACT_NONE) {
    gemm_oz_core(L, a);
    return;
  }
  SLQ_CHECK_ARG(!a.accumulate, "oz gemm: accumulate with an activation");
  GemmArgs<double> c = a;
  c.act = ACT_NONE;
  c.aux = nullptr;
  c.C2 = nullptr;
  const double* Y = a.C;
  int64_t ldy = a.ldc;
  if (a.act == ACT_GELU) {  // the pre-activation is an output of its own
    c.C = a.C2;
    c.ldc = a.ldc2;
    Y = a.C2;
    ldy = a.ldc2;
  }
  gemm_oz_core(L, c);
  const int64_t total = (int64_t)a.M * a.N;
  LaunchScope scope(L.prof, KC_ELEM, L.stream, 0,
                    8.0 * total * ((a.act == ACT_DGELU || a.act == ACT_DTANH) ? 3 : 2));
  const dim3 grid((unsigned)ceil_div(a.N, 1024), (unsigned)std::min(a.M, 65535));
  switch (a.act) {
    case ACT_GELU: k_oz_act<ACT_GELU><<<grid, 256, 0, L.stream>>>(a.M, a.N, Y, ldy, a.C, a.ldc, a.aux, a.ldaux); break;
    case ACT_TANH: k_oz_act<ACT_TANH><<<grid, 256, 0, L.stream>>>(a.M, a.N, Y, ldy, a.C, a.ldc, a.aux, a.ldaux); break;
    case ACT_DGELU: k_oz_act<ACT_DGELU><<<grid, 256, 0, L.stream>>>(a.M, a.N, Y, ldy, a.C, a.ldc, a.aux, a.ldaux); break;
    default: k_oz_act<ACT_DTANH><<<grid, 256, 0, L.stream>>>(a.M, a.N, Y, ldy, a.C, a.ldc, a.aux, a.ldaux);
  }
  SLQ_CUDA(cudaGetLastError());
  ++*L.launches;
}

void gemm_oz_core(const Launch& L, const GemmArgs<double>& a) {
  const OzBlocks b = oz_blocks(a, L.oz_S);
  if (b.mb == a.M && b.nb == a.N && b.kb == a.K) {
    gemm_oz(L, a, L.oz_S);
    return;
  }
  for (int k0 = 0; k0 < a.K; k0 += b.kb)
    for (int m0 = 0; m0 < a.M; m0 += b.mb)
      for (int n0 = 0; n0 < a.N; n0 += b.nb) {
        GemmArgs<double> c = a;
        c.M = std::min(b.mb, a.M - m0);
        c.N = std::min(b.nb, a.N - n0);
        c.K = std::min(b.kb, a.K - k0);
        c.A = a.A + (int64_t)m0 * a.sAm + (int64_t)k0 * a.sAk;
        c.B = a.B + (int64_t)k0 * a.sBk + (int64_t)n0 * a.sBn;
        c.C = a.C + (int64_t)m0 * a.ldc + n0;
        if (a.bias) c.bias = a.bias + n0;
        if (a.resid) c.resid = a.resid + (int64_t)m0 * a.ldr + n0;
        if (a.aux) c.aux = a.aux + (int64_t)m0 * a.ldaux + n0;
        if (a.C2) c.C2 = a.C2 + (int64_t)m0 * a.ldc2 + n0;
        c.accumulate = a.accumulate || k0 > 0;
        gemm_oz(L, c, L.oz_S);
      }
}

template <>
size_t gemm_ws_bytes<double>(const Launch& L, const GemmArgs<double>& a) {
  if (a.M == 0 || a.N == 0) return 0;
  if (L.gemm_mode == 2 && a.batch == 1 && a.tri == TRI_NONE && a.K > 0 &&
      (double)a.M * a.N * (double)a.K >= L.oz_min_mnk) {
    const OzBlocks b = oz_blocks(a, L.oz_S);
    return oz_ws_bytes(b.mb, b.nb, b.kb, L.oz_S);
  }
  int splits = 0;
  const int v = plan_variant(a, &splits);
  return dmma_ws_bytes(a, v, splits);
}

template <>
void gemm<double>(const Launch& L, const GemmArgs<double>& a) {
  check(a);
  if (a.M == 0 || a.N == 0) return;
  if (L.gemm_mode == 2 && a.batch == 1 && a.tri == TRI_NONE && a.K > 0 &&
      (double)a.M * a.N * (double)a.K >= L.oz_min_mnk) {
    gemm_oz_blocked(L, a);
    return;
  }
  int splits = 0;
  const int v = plan_variant(a, &splits);
  // experiment knob: divide the planned split counts (the plan was swept on an otherwise idle
  // GPU; inside the step two or three kernels share it)
  static const int div = getenv("SLQ_DMMA_SPLIT_DIV") ? std::max(1, atoi(getenv("SLQ_DMMA_SPLIT_DIV"))) : 1;
  if (div > 1 && splits > 0) splits = std::max(1, splits / div);
  run(L, a, v, splits);
}

}  // namespace slq

// Diagnostic (not on the hot path): time one fp64 GEMM shape with a given tile variant
// (-1 = the production heuristic) and split count (0 = auto).  A is [M x K] (K-contiguous when
// a_kmajor) and B is [K x N] given as [N x K] when b_kmajor.  Returns TFLOP/s and a checksum
// of C (all batch entries) so that variants can be compared for equality.
extern "C" slq_status slq_diag_gemm_f64(int32_t device, int32_t M, int32_t N, int32_t K, int32_t a_kmajor,
                                        int32_t b_kmajor, int32_t variant, int32_t splits, int32_t iters,
                                        double* tflops, double* checksum) {
  using namespace slq;
  double *A = nullptr, *B = nullptr, *C = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // diagnostic knobs: SLQ_DIAG_BATCH = b (contiguous batches), SLQ_DIAG_TRI = causal structure
  const int nb = getenv("SLQ_DIAG_BATCH") ? std::max(1, atoi(getenv("SLQ_DIAG_BATCH"))) : 1;
  const int tri = getenv("SLQ_DIAG_TRI") ? atoi(getenv("SLQ_DIAG_TRI")) : TRI_NONE;
  try {
    SLQ_CUDA(cudaSetDevice(device));
    SLQ_CUDA(cudaMalloc(&A, sizeof(double) * (size_t)M * K * nb));
    SLQ_CUDA(cudaMalloc(&B, sizeof(double) * (size_t)N * K * nb));
    SLQ_CUDA(cudaMalloc(&C, sizeof(double) * (size_t)M * N * nb));
    k_fill<<<1024, 256>>>(A, (int64_t)M * K * nb, 1);
    k_fill<<<1024, 256>>>(B, (int64_t)N * K * nb, 2);
    Workspace ws;
    int64_t launches = 0;
    Launch L{0, nullptr, &ws, &launches};
    GemmArgs<double> a;
    a.M = M; a.N = N; a.K = K;
    a.A = A; a.sAm = a_kmajor ? K : 1; a.sAk = a_kmajor ? 1 : M;
    a.B = B; a.sBk = b_kmajor ? 1 : N; a.sBn = b_kmajor ? K : 1;
    a.C = C; a.ldc = N;
    a.batch = nb;
    a.tri = tri;
    a.offA = BatchOff{(int64_t)M * K, 0, 1, 1};
    a.offB = BatchOff{(int64_t)N * K, 0, 1, 1};
    a.offC = BatchOff{(int64_t)M * N, 0, 1, 1};
    // variant <= -4: the tcgen05 int8 Ozaki path with S = -variant digit planes
    int planned_splits = 0;
    const int v = variant < 0 ? plan_variant(a, &planned_splits) : variant;
    if (variant < 0 && splits == 0) splits = planned_splits;
    auto go = [&] {
      if (variant <= -4) gemm_oz(L, a, -variant);
      else run(L, a, v, splits);
    };
    go();  // warm-up (also sets the smem attribute)
    SLQ_CUDA(cudaEventCreate(&e0));
    SLQ_CUDA(cudaEventCreate(&e1));
    SLQ_CUDA(cudaEventRecord(e0));
    for (int i = 0; i < iters; ++i) go();
    SLQ_CUDA(cudaEventRecord(e1));
    SLQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SLQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *tflops = gemm_flops(a) * iters / (ms * 1e-3) / 1e12;
    std::vector<double> h((size_t)M * N * nb);
    SLQ_CUDA(cudaMemcpy(h.data(), C, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
    double s = 0;
    for (size_t i = 0; i < h.size(); ++i) s += h[i] * (double)((i % 7) + 1);
    *checksum = s;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
    return SLQ_OK;
  } catch (const Error& e) {
    if (A) cudaFree(A);
    if (B) cudaFree(B);
    if (C) cudaFree(C);
    return e.status;
  }
}
