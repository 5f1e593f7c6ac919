// fp64 GEMM emulated exactly-accumulated on the tcgen05 INT8 tensor cores (Ozaki scheme, int8
// slices; pass mode SLQ_PASS_FP64_OZ).
//
//   C[M x N] = epilogue( A[M x K] . B[K x N] ),  A, B, C fp64.
//
// Every row i of A (every column j of B) is scaled by a power of two 2^e_i with |A_ik| < 2^e_i and
// cut into S signed 7-bit digits (truncation, exact in fp64):
//     A_ik = 2^e_i * sum_{p<S} a_p(i,k) 2^{-7(p+1)} + r,   |a_p| <= 127,  |r| < 2^{e_i - 7S}
// so   A.B ~= 2^{e_i + f_j} sum_{g<S} 2^{-7(g+2)} sum_{p+q=g} (a_p . b_q)
// Each a_p . b_q is an exact INT8 x INT8 -> INT32 tensor-core product; the products of one digit
// weight g share one INT32 TMEM accumulator (no rounding anywhere in the contraction; |acc| <=
// S K 127^2 < 2^31 is enforced by capping K per split).  The only error is the dropped digits,
// |error| <~ (S + 2) 2^{-7S} K max|A_i.| max|B_.j|.  S = 7 (default) meets the fp32 alpha/beta
// gate on c2 (S = 6: HVP 1.2e-6 but alpha drifts to 1.9e-4 by step 32; measured on B200).
//
// Kernel: BM = 128 x BN = 64 output tile per CTA, K in 64-byte k-tiles (SWIZZLE_64B TMA boxes);
// one pipeline stage holds all S digit planes of the A and B k-tiles, and the MMA issuer runs the
// S(S+1)/2 products from them (each plane is read from L2 once per k-tile, not once per product).
// Warp-specialised: warp 0 TMA producer, warp 1 TMEM allocator + single-thread MMA issuer, warps
// 2..9 epilogue (TMEM -> fp64 combine -> shared tile -> fused epilogue with coalesced stores).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "common.h"
#include "gemm_common.cuh"
#include "kernels.h"
#include "tc_common.cuh"
#include "oz_common.cuh"

namespace slq {
namespace oz {

using namespace tc;

constexpr int BM = 128, BK = 64, UMMA_K = 32;

// KT: k-tile width in bytes = int8 elements (64: SWIZZLE_64B, two MMAs per product per k-tile;
// 32: SWIZZLE_32B, one MMA per product, twice the stages in the same shared memory)
// NE = BN / 8 epilogue warps: four TMEM lane quadrants x BN / 32 groups of 32 columns
// TS: plain-epilogue output through per-warp 128B-swizzled shared tiles and TMA stores (8 KB per
// epilogue warp; the single-k-tile attention GEMMs, whose fp64 stores otherwise bound them)
template <int S, int BN, int KT = BK, bool TS = false>
struct Cfg {
  static constexpr int NE = BN / 8;
  static_assert(BN % 32 == 0 && BN >= 64 && BN <= 128, "BN in {64, 96, 128}");
  static constexpr int A_PLANE = BM * KT, B_PLANE = BN * KT;  // bytes
  static constexpr int A_BYTES = S * A_PLANE, B_BYTES = S * B_PLANE;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int OUTB = TS ? 8192 : 128 * 8;  // epilogue staging bytes per warp
  static constexpr int STAGES_FIT = (227 * 1024 - 2048 - NE * OUTB) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static_assert(STAGES >= (TS ? 1 : 2), "pipeline stages");
  static constexpr int BAR_BYTES = TS ? 1024 : 256;  // (TS: keeps the staging tiles 1024-byte aligned)
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + BAR_BYTES + NE * OUTB;
  static_assert(SMEM <= 232448, "dynamic shared memory per CTA");
  static constexpr int TMEM_COLS = S * BN <= 128 ? 128 : (S * BN <= 256 ? 256 : 512);
  static constexpr int NPROD = S * (S + 1) / 2;
  static_assert(S * BN <= 512, "S accumulators of BN columns must fit TMEM");
};

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(map),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}

// instruction descriptor, kind::i8: D s32, A and B signed 8-bit, both K-major, M x N
__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

struct OzArgs {
  int M, N, nk;          // nk: k-tiles of the whole K
  int kt_per_split, splits;
  const int* ea;         // [nbA][M] row exponents of A (nullptr: 0)
  const int* eb;         // [nbB][N] column exponents of B (nullptr: 0)
  int debug;  // diagnostic only (SLQ_OZ_DEBUG bits): 1 no MMAs, 2 no TMA loads, 4 no stores, 8 no TMEM drain
  int mfast;  // tile order: 1 = m fastest (the B tile is shared by the CTAs in flight and streamed
              // from DRAM once; the smaller A planes are re-read from L2), 0 = n fastest
  // batched (attention) GEMMs over pre-sliced planes: GEMM z reads plane batch zA(z) of A (planes
  // [S][nbA][M][Kp]) and zB(z) of B; tri: TRI_SKIP_UPPER tiles are not enumerated, TRI_K_LE_M /
  // TRI_K_GE_M clip the tile's k range to the causal part (splits == 1 then)
  int batch = 1, tri = 0, tiles_b = 0, nbA = 1, nbB = 1, z0A = 0, z0B = 0;
  BatchOff zA, zB;
};

__device__ __forceinline__ int64_t boff(const BatchOff& b, int z) {
  return (int64_t)(z / b.div) * b.outer + (int64_t)((z % b.div) / b.rep) * b.inner;
}

// 32 consecutive TMEM columns of the warp's 32 lanes (one 32-bit value per lane per column)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// Persistent kernel: grid <= #SMs, CTA c processes work units c, c + grid, ... (unit = output
// tile x K split).  The TMA producer runs ahead across unit boundaries (ring of STAGES k-tiles);
// the epilogue drains the S accumulators from TMEM into registers, releases TMEM (the next unit's
// MMAs start), then does the scaling and the global stores while the next unit computes.
// NI > 1 (S = 7): the digit weights are split over NI MMA-issuing warps (warp 1, then warps 10,
// 11), each a single issuing thread: NI = 2 -> {0, 5, 6} / {1..4} (14 + 14 products), NI = 3 ->
// {1, 6} / {2, 5} / {0, 3, 4} (9 + 9 + 10).  One thread cannot issue 128 x 64 x 32 MMAs as fast as
// the tensor pipe retires them; several threads can.
// Digit weight g has g + 1 products.  S = 7: NI = 2 -> {0, 5, 6} / {1..4} (14 + 14), NI = 3 ->
// {1, 6} / {2, 5} / {0, 3, 4} (9 + 9 + 10); S = 6: NI = 2 -> {0, 1, 2, 5} / {3, 4} (12 + 9); S = 5:
// NI = 2 -> {0, 1, 4} / {2, 3} (8 + 7).
__host__ __device__ constexpr int oz_owner(int S, int NI, int g) {
  return NI == 1   ? 0
         : S == 7  ? (NI == 2 ? (g >= 1 && g <= 4 ? 1 : 0) : (g == 1 || g == 6 ? 0 : (g == 2 || g == 5 ? 1 : 2)))
         : S == 6  ? (g == 3 || g == 4 ? 1 : 0)
                   : (g == 2 || g == 3 ? 1 : 0);
}
// warps: 0 TMA producer, 1 MMA issuer 0 + TMEM allocator, 2 .. NE + 1 epilogue, NE + 2 .. NE + NI
// the other MMA issuers
template <int S, int BN, int KT = BK, int NI = 1, bool TS = false>
__global__ void __launch_bounds__(32 * (Cfg<S, BN, KT, TS>::NE + NI + 1), 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, OzArgs o,
              const __grid_constant__ GemmArgs<double> p, double* __restrict__ ws,
              const __grid_constant__ CUtensorMap tmC) {
  static_assert(NI == 1 || (NI == 2 && S >= 5) || (NI == 3 && S == 7), "issuer split defined for S = 5..7");
  using CF = Cfg<S, BN, KT, TS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::STAGES * CF::STAGE_BYTES);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* tmem_full = empty + CF::STAGES;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  double* stage_t = reinterpret_cast<double*>(smem + CF::STAGES * CF::STAGE_BYTES + CF::BAR_BYTES);  // NE x OUTB
  constexpr int NE = CF::NE;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles_n = (p.N + BN - 1) / BN, tiles_m = (p.M + BM - 1) / BM;
  const int nwork = o.batch * o.tiles_b * o.splits;
  // unit w -> (batch z, split, tile_m, tile_n): the larger operand's tile is the one the CTAs in
  // flight share (o.mfast), so its digit planes stream from DRAM once and the smaller operand's
  // planes are the ones re-read (from L2); TRI_SKIP_UPPER enumerates the lower tiles row by row
  auto decode = [&](int w, int& z, int& m0, int& n0, int& sp, int& kt0, int& nloc) {
    sp = w % o.splits;
    int t = w / o.splits;
    z = t / o.tiles_b;
    t -= z * o.tiles_b;
    if (o.tri == TRI_K_LE_M || o.tri == TRI_K_GE_M) {
      // k-clipped causal tiles differ in length (1 .. nk k-tiles): longest first across the whole
      // batch, so the static round-robin hands every CTA a similar mix (largest-first balancing)
      t = w / o.splits;
      const int bn = o.batch * tiles_n;
      const int rank = t / bn, rem = t - rank * bn;
      z = rem / tiles_n;
      n0 = (rem - z * tiles_n) * BN;
      m0 = (o.tri == TRI_K_LE_M ? tiles_m - 1 - rank : rank) * BM;
    } else if (o.tri == TRI_SKIP_UPPER) {
      int mt = 0;
      for (;;) {
        const int c = min(tiles_n, (mt * BM + BM - 1) / BN + 1);
        if (t < c) break;
        t -= c;
        ++mt;
      }
      m0 = mt * BM;
      n0 = t * BN;
    } else if (o.mfast) {
      m0 = (t % tiles_m) * BM;
      n0 = (t / tiles_m) * BN;
    } else {
      n0 = (t % tiles_n) * BN;
      m0 = (t / tiles_n) * BM;
    }
    int kb = 0, ke = o.nk;
    if (o.tri == TRI_K_LE_M) ke = min(ke, (m0 + BM + KT - 1) / KT);
    else if (o.tri == TRI_K_GE_M) kb = m0 / KT;
    kt0 = kb + sp * o.kt_per_split;
    const int kt1 = min(ke, kt0 + o.kt_per_split);
    nloc = kt1 > kt0 ? kt1 - kt0 : 0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NI);  // one commit per issuing warp
    }
    mbar_init(tmem_full, NI);
    mbar_init(tmem_empty, NE);  // one arrive per epilogue warp
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_holder)),
                 "n"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: all S digit planes of A and B for one k-tile per stage ----
      int it = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        int z, m0, n0, sp, kt0, nloc;
        decode(w, z, m0, n0, sp, kt0, nloc);
        const int ra = (o.z0A + (int)boff(o.zA, z)) * o.M + m0, rb = (o.z0B + (int)boff(o.zB, z)) * o.N + n0;
        for (int i = 0; i < nloc; ++i, ++it) {
          const int kt = kt0 + i, s = it % CF::STAGES;
          const uint32_t ph = (it / CF::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * CF::STAGE_BYTES;
          uint8_t* sb = sa + CF::A_BYTES;
          if (o.debug & 2) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&full[s])));
            continue;
          }
          mbar_expect_tx(&full[s], CF::STAGE_BYTES);
#pragma unroll
          for (int q = 0; q < S; ++q) {
            tma_load_2d(sa + q * CF::A_PLANE, &tmA, &full[s], kt * KT, q * o.nbA * o.M + ra);
            tma_load_2d(sb + q * CF::B_PLANE, &tmB, &full[s], kt * KT, q * o.nbB * o.N + rb);
          }
        }
      }
    }
  } else if (warp == 1 || warp >= NE + 2) {
    if (lane == 0) {  // ---- MMA issuer(s): S(S+1)/2 digit products per k-tile ----
      const int iss = warp == 1 ? 0 : warp - (NE + 1);
      constexpr uint32_t idesc = make_idesc_i8(BM, BN);
      int it = 0, tl = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++tl) {
        int z, m0, n0, sp, kt0, nloc;
        decode(w, z, m0, n0, sp, kt0, nloc);
        mbar_wait(tmem_empty, (tl & 1) ^ 1);  // the previous unit's accumulators have been drained
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        uint32_t started = 0;  // the unit's accumulators have been initialised
        for (int i = 0; i < nloc; ++i, ++it) {
          const int s = it % CF::STAGES;
          const uint32_t ph = (it / CF::STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          const uint32_t sa = smem_u32(smem + s * CF::STAGE_BYTES);
          const uint32_t sb = sa + CF::A_BYTES;
          // descriptors: one base per operand and stage, plane / k offsets added to the 14-bit
          // address field (16-byte units; every address stays below 256 KB, so no carry out)
          const uint64_t da0 = KT == 64 ? make_desc_sw64(sa) : make_desc_sw32(sa);
          const uint64_t db0 = KT == 64 ? make_desc_sw64(sb) : make_desc_sw32(sb);
          const uint32_t first = started == 0u;  // first k-tile of the unit: overwrite
          if (!(o.debug & 1)) {
#pragma unroll
            for (int g = 0; g < S; ++g) {
              if (NI > 1 && oz_owner(S, NI, g) != iss) continue;
#pragma unroll
              for (int pa = 0; pa <= g; ++pa) {
                const int qb = g - pa;
#pragma unroll
                for (int kk = 0; kk < KT / UMMA_K; ++kk) {
                  const uint64_t da = da0 + (uint64_t)((pa * CF::A_PLANE + kk * UMMA_K) >> 4);
                  const uint64_t db = db0 + (uint64_t)((qb * CF::B_PLANE + kk * UMMA_K) >> 4);
                  const uint32_t acc = (pa == 0 && kk == 0) ? (first ^ 1u) : 1u;
                  asm volatile(
                      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)(g * BN)),
                      "l"(da), "l"(db), "r"(idesc), "r"(acc));
                }
              }
            }
          }
          started = 1u;
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              smem_u32(&empty[s])));
        }
        if (nloc > 0) {
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              smem_u32(tmem_full)));
        } else {
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_full)));
        }
      }
    }
  } else {
    // ---- epilogue (warps 2 .. NE + 1): warp w drains TMEM lanes 32 (w % 4) .. +31 (its quadrant),
    // columns [32 h, 32 h + 32) with h = (w - 2) / 4, combining the S digit weights in fp64 ----
    const int lg = (warp % 4) * 32;
    const int c0 = ((warp - 2) / 4) * 32;
    int tl = 0;
    for (int w = blockIdx.x; w < nwork; w += gridDim.x, ++tl) {
      int z, m0, n0, sp, kt0, nloc;
      decode(w, z, m0, n0, sp, kt0, nloc);
      // scales first (their global-load latency overlaps the wait for the accumulators):
      // lane l holds 2^f for column n0 + c0 + l and 2^e for row m0 + lg + l; alpha folds into the
      // row scale (an exact power-of-two product, so alpha * (v 2^e 2^f) rounds identically)
      const int n_l = n0 + c0 + lane, row_l = m0 + lg + lane;
      const double sc_l = n_l < p.N ? (o.eb ? scale_of(o.eb[(o.batch > 1 || o.z0B ? o.z0B + boff(o.zB, z) : 0) * p.N + n_l]) : 1.0) : 0.0;
      const bool fold = o.splits == 1 && !p.bias && !p.resid && !p.accumulate;
      double sr = (nloc > 0 && row_l < p.M) ? (o.ea ? scale_of(o.ea[(o.batch > 1 || o.z0A ? o.z0A + boff(o.zA, z) : 0) * p.M + row_l]) : 1.0) : 0.0;
      if (fold) sr *= p.alpha;
      mbar_wait(tmem_full, tl & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      double v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = 0.0;
      if constexpr (S <= 5) {
        // Drain for S <= 5: the S accumulators are combined EXACTLY in int64 by Horner's rule in
        // base 2^7, h = ((a_0 2^7 + a_1) 2^7 + ...) 2^7 + a_{S-1} (|a_g| < 2^31, so |h| < 2^60), and
        // h is converted to fp64 only after TMEM is released -- the fp64 pipe work (the top stall of
        // the short-K GEMMs) leaves the section in which the next tile's MMAs wait for the
        // accumulators.  (S = 6, 7 would overflow int64 and keep the fp64 drain below.)
        // Short units (K of the unit < kLim): |h| <= K 127^2 2^(7(S-1)) sum_g (g+1) 2^(-7g) < 2^53, so
        // the same Horner combination is exact in fp64 (one i2d + one DFMA per accumulator value,
        // about half the int64 instruction count -- the drain is the per-tile period of the
        // K = 64 attention GEMMs); both branches give the identical integer h.
        constexpr double kLim = 9007199254740992.0 / (16129.0 * 1.0158 * (double)(1ll << (7 * (S - 1))));
        const double wl = exp2i(-7 * (S + 1));
        if ((double)nloc * KT < kLim) {
          double hd[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) hd[i] = 0.0;
#pragma unroll 1
          for (int g = 0; g < ((o.debug & 8) ? 0 : S); ++g) {
            uint32_t r0[32];
            tmem_ld32(tmem + ((uint32_t)lg << 16) + (uint32_t)(g * BN + c0), r0);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
            for (int i = 0; i < 32; ++i) hd[i] = fma(hd[i], 128.0, i2d(r0[i]));
          }
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_empty)));
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = hd[i] * wl;
        } else {
          long long h[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) h[i] = 0;
#pragma unroll 1
          for (int g = 0; g < ((o.debug & 8) ? 0 : S); ++g) {
            uint32_t r0[32];
            tmem_ld32(tmem + ((uint32_t)lg << 16) + (uint32_t)(g * BN + c0), r0);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
            for (int i = 0; i < 32; ++i) h[i] = h[i] * 128 + (long long)(int)r0[i];
          }
          asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
          __syncwarp();
          if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_empty)));
          // v = h 2^(-7(S + 1)): hi 2^32 + lo exactly from two i2d conversions, one rounding in the fma
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const double hi = i2d((uint32_t)(int)(h[i] >> 32));
            const double lo = __hiloint2double(0x43300000, (int)(uint32_t)h[i]) - 4503599627370496.0;
            v[i] = fma(hi, 4294967296.0, lo) * wl;
          }
        }
      } else {
        // two digit-weight groups per TMEM round trip (2 x 32 columns, one wait); the g loop stays
        // rolled (the 32-wide bodies are unrolled) to keep the kernel inside the instruction cache
        // (more than 8 epilogue warps: one group per round trip, within the smaller register budget)
        constexpr int GS = NE > 8 ? 1 : 2;
#pragma unroll 1
        for (int g = 0; g < ((o.debug & 8) ? 0 : S); g += GS) {
          uint32_t r0[32], r1[GS > 1 ? 32 : 1];
          tmem_ld32(tmem + ((uint32_t)lg << 16) + (uint32_t)(g * BN + c0), r0);
          if (GS > 1 && g + 1 < S) tmem_ld32(tmem + ((uint32_t)lg << 16) + (uint32_t)((g + 1) * BN + c0), r1);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
          const double w0 = exp2i(-7 * (g + 2)), w1 = exp2i(-7 * (g + 3));
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fma(i2d(r0[i]), w0, v[i]);
          if (GS > 1 && g + 1 < S) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fma(i2d(r1[GS > 1 ? i : 0]), w1, v[i]);
          }
        }
        // accumulators drained: release TMEM to the next unit's MMAs
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_empty)));
      }
      if constexpr (TS) {
        // plain epilogue through TMA stores (host-checked: one split, no bias / residual /
        // accumulate, the C rows of batch z contiguous at z M): the warp's 32 x 32 block goes to
        // two [32 rows][16 columns] 128B-swizzled shared tiles (16-byte chunk j of row r at
        // r 128 + (j ^ (r % 8)) 16), one lane issues the two bulk tensor stores; the tiles are reused
        // once the previous unit's stores have read them
        uint8_t* stg = reinterpret_cast<uint8_t*>(stage_t) + (warp - 2) * CF::OUTB;
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 32; c += 2) {
          const double s0 = __shfl_sync(0xffffffffu, sc_l, c), s1 = __shfl_sync(0xffffffffu, sc_l, c + 1);
          const int box = c >> 4, ch = (c & 15) >> 1;
          *reinterpret_cast<double2*>(stg + box * 4096 + lane * 128 + ((ch ^ (lane & 7)) << 4)) =
              make_double2(v[c] * sr * s0, v[c + 1] * sr * s1);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0 && !(o.debug & 4)) {
          const int rowg = (o.batch > 1 ? z * p.M : 0) + m0 + lg;
#pragma unroll
          for (int box = 0; box < 2; ++box)
            if (n0 + c0 + 16 * box < p.N) tma_store_2d(&tmC, stg + box * 4096, n0 + c0 + 16 * box, rowg);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        continue;
      }
      // Row scale in registers (lane = row); then 4-column chunks go through a per-warp 32 x 4
      // shared tile so that each store instruction writes 8 rows x 32 contiguous bytes (full
      // sectors) instead of 32 rows x 8-16 bytes (register-direct row stores measured 14% slower on
      // the write-heavy c3 logits GEMM).  Lane l stores rows 8 j + l / 4 of column l % 4.  Plain
      // stores: split-K partials, or no bias / residual / accumulate (alpha folded into the row
      // scale).  Otherwise y = alpha (x sc) + bias (+ residual) (+ old C): the bias comes from a
      // register loaded with the scales, and each chunk's residual / old-C values are loaded one
      // chunk ahead (the out-of-line per-chunk function this replaces serialised 8 dependent global
      // round trips per tile, which made the bias / residual forward GEMMs epilogue-bound).
      const int ncol = p.N - (n0 + c0);  // valid columns of this warp's 32 (may be <= 0)
      const bool plain = o.splits > 1 || fold;
      double* Wd = o.splits > 1 ? ws + (int64_t)sp * p.M * p.N : p.C + (o.batch > 1 ? boff(p.offC, z) : 0);
      const int64_t ldw = o.splits > 1 ? p.N : p.ldc;
      double* T = stage_t + (warp - 2) * 128;
      const int cc = lane & 3, r0 = lane >> 2;
      const int mmax = p.M - (m0 + lg) - r0;  // rows 8 j + r0 with 8 j < mmax are valid
      double* dst = Wd + (int64_t)(m0 + lg + r0) * ldw + (n0 + c0 + cc);
      const double* rsd = (!plain && p.resid) ? p.resid + (int64_t)(m0 + lg + r0) * p.ldr + (n0 + c0 + cc) : nullptr;
      const double* bsp = (!plain && p.bias) ? p.bias + (n0 + c0 + cc) : nullptr;
      double rn[4], bn = 0.0;
      auto fetch = [&](int c) {
        const bool okc = c + cc < ncol;
        bn = (bsp && okc) ? bsp[c] : 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) rn[j] = (rsd && okc && 8 * j < mmax) ? rsd[(int64_t)(8 * j) * p.ldr + c] : 0.0;
      };
      if (!plain) fetch(0);
#pragma unroll
      for (int c = 0; c < ((o.debug & 4) ? 0 : 32); c += 4) {
        if (c >= ncol) break;  // (warp-uniform)
        __syncwarp();
        *reinterpret_cast<double2*>(&T[lane * 4]) = make_double2(v[c] * sr, v[c + 1] * sr);
        *reinterpret_cast<double2*>(&T[lane * 4 + 2]) = make_double2(v[c + 2] * sr, v[c + 3] * sr);
        __syncwarp();
        const double sc = __shfl_sync(0xffffffffu, sc_l, c + cc);
        if (plain) {
          if (c + cc < ncol) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (8 * j < mmax) dst[(int64_t)(8 * j) * ldw + c] = T[(8 * j + r0) * 4 + cc] * sc;
          }
        } else {
          double y[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            y[j] = p.alpha * (T[(8 * j + r0) * 4 + cc] * sc) + bn;
            if (rsd) y[j] += rn[j];
          }
          if (c + 4 < 32 && c + 4 < ncol) fetch(c + 4);  // next chunk's loads in flight during these stores
          if (c + cc < ncol) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (8 * j < mmax) {
                double* d = dst + (int64_t)(8 * j) * ldw + c;
                *d = p.accumulate ? *d + y[j] : y[j];
              }
            }
          }
        }
      }
    }
    if constexpr (TS) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(CF::TMEM_COLS));
  }
}

// ---- wide variant: S = 7, 128 x 128 tiles, accumulators in two phases ----
// The INT8 pipe runs far closer to its peak with N = 128 MMAs than with N = 64 (75% vs 41% pipe
// activity), but 7 accumulators of 128 columns exceed the 512 TMEM columns.  So each
// tile is computed in two phases over its k-range: digit weights g = 0..3 (4 x 128 columns, digit
// planes 0..3 of both operands, 10 products), drained into fp64 registers, then g = 4..6 (3 x 128
// columns, planes 0..6, 18 products) -- the same 28 products, with the phase-0 planes re-streamed.
// 32-byte k-tiles (SWIZZLE_32B, one MMA per product per k-tile) keep three 56 KB stages.
constexpr int WBN = 128, WBK = 32, WS = 7;
struct CfgW {
  static constexpr int PLANE = BM * WBK;  // bytes (A and B planes are both 128 x 32)
  static constexpr int STAGE_BYTES = 2 * WS * PLANE;
  static constexpr int STAGES = 3;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256 + 8 * 128 * 8;
  static_assert(SMEM <= 232448, "dynamic shared memory per CTA");
};

__global__ void __launch_bounds__(320, 1)
    k_oz_gemm_w(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, OzArgs o,
                GemmArgs<double> p, double* __restrict__ ws) {
  using CF = CfgW;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + CF::STAGES * CF::STAGE_BYTES);
  uint64_t* empty = full + CF::STAGES;
  uint64_t* tmem_full = empty + CF::STAGES;
  uint64_t* tmem_empty = tmem_full + 1;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_empty + 1);
  double* stage_t = reinterpret_cast<double*>(smem + CF::STAGES * CF::STAGE_BYTES + 256);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int tiles_n = (p.N + WBN - 1) / WBN, tiles_m = (p.M + BM - 1) / BM;
  const int nwork = tiles_n * tiles_m * o.splits;
  auto decode = [&](int w, int& m0, int& n0, int& sp, int& kt0, int& nloc) {
    sp = w % o.splits;
    const int t = w / o.splits;
    n0 = (t % tiles_n) * WBN;
    m0 = (t / tiles_n) * BM;
    kt0 = sp * o.kt_per_split;
    const int kt1 = min(o.nk, kt0 + o.kt_per_split);
    nloc = kt1 > kt0 ? kt1 - kt0 : 0;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < CF::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    mbar_init(tmem_empty, 8);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_holder)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: per tile, phase 0 (planes 0..3) then phase 1 (planes 0..6) ----
      int it = 0;
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        int m0, n0, sp, kt0, nloc;
        decode(w, m0, n0, sp, kt0, nloc);
        for (int ph = 0; ph < 2; ++ph) {
          const int np = ph == 0 ? 4 : WS;
          for (int i = 0; i < nloc; ++i, ++it) {
            const int kt = kt0 + i, s = it % CF::STAGES;
            mbar_wait(&empty[s], ((it / CF::STAGES) & 1) ^ 1);
            uint8_t* sa = smem + s * CF::STAGE_BYTES;
            uint8_t* sb = sa + WS * CF::PLANE;
            mbar_expect_tx(&full[s], 2 * np * CF::PLANE);
            for (int q = 0; q < np; ++q) {
              tma_load_2d(sa + q * CF::PLANE, &tmA, &full[s], kt * WBK, q * o.M + m0);
              tma_load_2d(sb + q * CF::PLANE, &tmB, &full[s], kt * WBK, q * o.N + n0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = make_idesc_i8(BM, WBN);
      int it = 0, use = 0;  // use: tmem_full / tmem_empty handshakes so far
      for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
        int m0, n0, sp, kt0, nloc;
        decode(w, m0, n0, sp, kt0, nloc);
        for (int ph = 0; ph < 2; ++ph, ++use) {
          mbar_wait(tmem_empty, (use & 1) ^ 1);  // the epilogue drained the previous phase
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
          uint32_t started = 0;
          for (int i = 0; i < nloc; ++i, ++it) {
            const int s = it % CF::STAGES;
            mbar_wait(&full[s], (it / CF::STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
            const uint32_t sa = smem_u32(smem + s * CF::STAGE_BYTES);
            const uint32_t sb = sa + WS * CF::PLANE;
            // descriptors: one base per operand and stage plus constant plane offsets (16-byte
            // units); fully unrolled per phase, accumulate flag constant after the first k-tile
            const uint64_t da0 = make_desc_sw32(sa), db0 = make_desc_sw32(sb);
            const uint32_t first = started == 0u;
            auto mma = [&](int g, int pa, int qb, int gl) {
              const uint64_t da = da0 + (uint64_t)((pa * CF::PLANE) >> 4);
              const uint64_t db = db0 + (uint64_t)((qb * CF::PLANE) >> 4);
              const uint32_t acc = pa == 0 ? (first ^ 1u) : 1u;
              asm volatile(
                  "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                  "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (uint32_t)(gl * WBN)),
                  "l"(da), "l"(db), "r"(idesc), "r"(acc));
            };
            if (ph == 0) {
#pragma unroll
              for (int g = 0; g < 4; ++g)
#pragma unroll
                for (int pa = 0; pa <= g; ++pa) mma(g, pa, g - pa, g);
            } else {
#pragma unroll
              for (int g = 4; g < WS; ++g)
#pragma unroll
                for (int pa = 0; pa <= g; ++pa) mma(g, pa, g - pa, g - 4);
            }
            started = 1u;
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(&empty[s])));
          }
          if (nloc > 0) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                smem_u32(tmem_full)));
          } else {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_full)));
          }
        }
      }
    }
  } else {
    // ---- epilogue (warps 2..9): lanes 32 (w % 4) .. +31, columns [64 h, 64 h + 64) with h = (w-2)/4 ----
    const int lg = (warp % 4) * 32;
    const int ch = ((warp - 2) / 4) * 64;
    int use = 0;
    for (int w = blockIdx.x; w < nwork; w += gridDim.x) {
      int m0, n0, sp, kt0, nloc;
      decode(w, m0, n0, sp, kt0, nloc);
      const int row_l = m0 + lg + lane;
      const double sr = (nloc > 0 && row_l < p.M) ? scale_of(o.ea[row_l]) : 0.0;
      double sc_l[2];
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        const int n_l = n0 + ch + 32 * jb + lane;
        sc_l[jb] = n_l < p.N ? scale_of(o.eb[n_l]) : 0.0;
      }
      double v[64];
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = 0.0;
#pragma unroll 1
      for (int ph = 0; ph < 2; ++ph, ++use) {
        mbar_wait(tmem_full, use & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const int g0 = ph == 0 ? 0 : 4, g1 = ph == 0 ? 4 : WS;
#pragma unroll 1
        for (int g = g0; g < g1; ++g) {
          uint32_t r0[32], r1[32];
          const uint32_t base = tmem + ((uint32_t)lg << 16) + (uint32_t)((g - g0) * WBN + ch);
          tmem_ld32(base, r0);
          tmem_ld32(base + 32, r1);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
          const double wg = exp2i(-7 * (g + 2));
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v[i] = fma(i2d(r0[i]), wg, v[i]);
            v[32 + i] = fma(i2d(r1[i]), wg, v[32 + i]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(tmem_empty)));
      }
      double* T = stage_t + (warp - 2) * 128;
      const bool plain = o.splits > 1 || (!p.bias && !p.resid && !p.aux && !p.accumulate && p.act == ACT_NONE &&
                                          p.alpha == 1.0);
      double* Wd = o.splits > 1 ? ws + (int64_t)sp * p.M * p.N : p.C;
      const int64_t ldw = o.splits > 1 ? p.N : p.ldc;
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        const int c0 = ch + 32 * jb;
        const int ncol = p.N - (n0 + c0);
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          __syncwarp();
          *reinterpret_cast<double2*>(&T[lane * 4]) = make_double2(v[32 * jb + c] * sr, v[32 * jb + c + 1] * sr);
          *reinterpret_cast<double2*>(&T[lane * 4 + 2]) =
              make_double2(v[32 * jb + c + 2] * sr, v[32 * jb + c + 3] * sr);
          __syncwarp();
          const int cc = c + (lane & 3);
          const int n = n0 + c0 + cc;
          const bool colok = cc < ncol;
          const double sc = __shfl_sync(0xffffffffu, sc_l[jb], cc);
          double x[4], bs = 0.0, rs[4], ax[4], cold[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int m = m0 + lg + 8 * j + (lane >> 2);
            const bool ok = colok && m < p.M;
            x[j] = T[(8 * j + (lane >> 2)) * 4 + (lane & 3)] * sc;
            if (!plain) {
              rs[j] = (ok && p.resid) ? p.resid[(int64_t)m * p.ldr + n] : 0.0;
              ax[j] = (ok && p.aux) ? p.aux[(int64_t)m * p.ldaux + n] : 0.0;
              cold[j] = (ok && p.accumulate) ? p.C[(int64_t)m * p.ldc + n] : 0.0;
            }
          }
          if (!plain && colok && p.bias) bs = p.bias[n];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int m = m0 + lg + 8 * j + (lane >> 2);
            if (!colok || m >= p.M) continue;
            if (plain) {
              Wd[(int64_t)m * ldw + n] = x[j];
              continue;
            }
            const double y = p.alpha * x[j] + bs + rs[j];
            double out;
            switch (p.act) {
              case ACT_GELU:
                p.C2[(int64_t)m * p.ldc2 + n] = y;
                out = gemm_detail::gelu_tanh(y);
                break;
              case ACT_TANH: out = tanh(y); break;
              case ACT_DGELU: out = y * gemm_detail::gelu_tanh_grad(ax[j]); break;
              case ACT_DTANH: out = y * (1.0 - ax[j] * ax[j]); break;
              default: out = y;
            }
            p.C[(int64_t)m * p.ldc + n] = p.accumulate ? cold[j] + out : out;
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(512));
  }
}

// ---- merged slicing of both GEMM operands (one or two launches per GEMM) ----
// A job slices one operand into S digit planes [S][rows][Kp] and row exponents ex[rows].
// kmajor: element (r, k) at X[r * ld + k]; else at X[k * ld + r] (the exponent pass then writes
// one partial exponent per 256-deep k block into xp[kb * rows + r], combined by the slice pass).
struct SliceJob {
  const double* X;
  int64_t ld;
  int rows, K, Kp, kmajor;
  int8_t* out;
  int* ex;
  int* xp;       // [ceil(K / kcol)][rows] partial exponents (cols path)
  int blocks0;   // first block of this job in the launch
  int kcol;      // k extent of one exponent-pass block (cols path)
};
struct SliceJobs {
  SliceJob j[2];
  int n;
  int regrow = 1;  // rows path with Kp <= 1024: the row held in registers (0: re-read through L1, A/B)
};
constexpr int kColK = 256;     // k extent of one exponent-pass block
constexpr int kColKMin = 64;   // ... for operands whose exponent pass would not fill two waves of SMs
static int col_kblk(int rows, int K) { return ceil_div(rows, 32) * ceil_div(K, kColK) >= 2 * 148 ? kColK : kColKMin; }

__device__ __forceinline__ const SliceJob& job_of(const SliceJobs& js, int b) {
  return (js.n > 1 && b >= js.j[1].blocks0) ? js.j[1] : js.j[0];
}

// exponent pass of the cols-path jobs: block (32 rows, 256 k) -> xp[kb][r]
__global__ void __launch_bounds__(256) k_oz_colexp2(const __grid_constant__ SliceJobs js) {
  const SliceJob& jb = job_of(js, blockIdx.x);
  const int b = blockIdx.x - jb.blocks0;
  const int rb = (jb.rows + 31) / 32;
  const int r0 = (b % rb) * 32, kb = b / rb;
  __shared__ double red[8][33];
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int r = r0 + tx;
  const int k0 = kb * jb.kcol, k1 = min(jb.K, k0 + jb.kcol);
  double mx = 0.0;
  bool nf = false;
  if (r < jb.rows) {
#pragma unroll 8
    for (int k = k0 + ty; k < k1; k += 8) {
      const double x = jb.X[(int64_t)k * jb.ld + r];
      mx = fmax(mx, fabs(x));
      nf |= nonfinite(x);
    }
  }
  red[ty][tx] = nf ? __longlong_as_double(0x7ff8000000000000ll) : mx;
  __syncthreads();
  if (ty == 0 && r < jb.rows) {
    double m = 0.0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      bad |= red[i][tx] != red[i][tx];
      m = fmax(m, red[i][tx]);
    }
    jb.xp[(int64_t)kb * jb.rows + r] = bad ? kExNaN : (m > 0.0 ? exp_of(m) : kExNone);
  }
}

// slice pass: rows-path job = one warp per row (the max pass issues 32 independent loads per lane
// per 1024-wide sweep; the digit pass re-reads the row from L1/L2); cols-path job = 32 rows x 128 k
// per block through a shared tile, exponent = max of the row's partial exponents
template <int S>
__global__ void __launch_bounds__(256) k_oz_slice2(const __grid_constant__ SliceJobs js) {
  const SliceJob& jb = job_of(js, blockIdx.x);
  const int b = blockIdx.x - jb.blocks0;
  const int64_t plane = (int64_t)jb.rows * jb.Kp;
  if (jb.kmajor) {
    const int row = b * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
    if (row >= jb.rows) return;
    const double* xr = jb.X + (int64_t)row * jb.ld;
    // 16-byte loads when the row base is 16-byte aligned (even pitch, aligned base)
    const bool v2 = (jb.ld % 2) == 0 && ((uintptr_t)jb.X & 15) == 0;
    if (v2 && jb.Kp <= 1024 && js.regrow) {
      // the whole row in registers (4 consecutive k per lane per 128-wide sweep): one read of X
      double x[8][4];
      double mx = 0.0;
      bool nf = false;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k4 = 128 * i + 4 * lane;
        if (k4 + 3 < jb.K) {
          const double2 p0 = *reinterpret_cast<const double2*>(xr + k4);
          const double2 p1 = *reinterpret_cast<const double2*>(xr + k4 + 2);
          x[i][0] = p0.x; x[i][1] = p0.y; x[i][2] = p1.x; x[i][3] = p1.y;
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) x[i][j] = (k4 + j < jb.K) ? xr[k4 + j] : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          mx = fmax(mx, fabs(x[i][j]));
          nf |= nonfinite(x[i][j]);
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      nf = __any_sync(0xffffffffu, nf);
      if (lane == 0) jb.ex[row] = exp_of(mx, nf);
      const int e = nf ? 0 : exp_of(mx);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int k4 = 128 * i + 4 * lane;
        if (k4 >= jb.Kp) break;
        uint32_t w[S];
        digits4<S>(x[i], e, w);
#pragma unroll
        for (int q = 0; q < S; ++q) *reinterpret_cast<uint32_t*>(jb.out + q * plane + (int64_t)row * jb.Kp + k4) = w[q];
      }
      return;
    }
    constexpr int V = 32;  // values per lane per sweep (1024-wide sweeps)
    double mx = 0.0;
    bool nf = false;
    for (int k0 = 0; k0 < jb.K; k0 += 32 * V) {
#pragma unroll
      for (int i = 0; i < V; ++i) {
        const int k = k0 + i * 32 + lane;
        if (k < jb.K) {
          mx = fmax(mx, fabs(xr[k]));
          nf |= nonfinite(xr[k]);
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    nf = __any_sync(0xffffffffu, nf);
    if (lane == 0) jb.ex[row] = exp_of(mx, nf);
    const int e = nf ? 0 : exp_of(mx);  // (digits of a non-finite row are never used)
    for (int k4 = lane * 4; k4 < jb.Kp; k4 += 128) {
      double x[4];
      if (v2 && k4 + 3 < jb.K) {
        const double2 p0 = *reinterpret_cast<const double2*>(xr + k4);
        const double2 p1 = *reinterpret_cast<const double2*>(xr + k4 + 2);
        x[0] = p0.x; x[1] = p0.y; x[2] = p1.x; x[3] = p1.y;
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = (k4 + j < jb.K) ? xr[k4 + j] : 0.0;
      }
      uint32_t w[S];
      digits4<S>(x, e, w);
#pragma unroll
      for (int q = 0; q < S; ++q) *reinterpret_cast<uint32_t*>(jb.out + q * plane + (int64_t)row * jb.Kp + k4) = w[q];
    }
    return;
  }
  // the block's whole 32-row x 128-k tile in one sweep (16 loads in flight per thread), then the
  // digits of 4 x 4 consecutive k per thread
  __shared__ double tile[128][33];
  __shared__ int es[32];
  const int rb = (jb.rows + 31) / 32;
  const int r0 = (b % rb) * 32, kblk = b / rb;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
  const int r = r0 + tx;
  const int kb0 = kblk * 128, kb1 = min(jb.Kp, kb0 + 128);
  {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k = kb0 + ty + 8 * i;
      x[i] = (r < jb.rows && k < jb.K) ? jb.X[(int64_t)k * jb.ld + r] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) tile[ty + 8 * i][tx] = x[i];
  }
  if (threadIdx.x < 32) {
    int e = kExNone;
    if (r < jb.rows) {
      const int nkb = (jb.K + jb.kcol - 1) / jb.kcol;
      for (int kb = 0; kb < nkb; ++kb) e = max(e, jb.xp[(int64_t)kb * jb.rows + r]);
    }
    if (kblk == 0 && r < jb.rows) jb.ex[r] = e == kExNone ? 0 : e;
    es[threadIdx.x] = (e == kExNone || e == kExNaN) ? 0 : e;  // (digits of a non-finite row are never used)
  }
  __syncthreads();
  const int wr = threadIdx.x / 8, kq = threadIdx.x % 8;
  if (r0 + wr >= jb.rows) return;
  const int ew = es[wr];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const int kl = 32 * g + 4 * kq;
    if (kb0 + kl >= kb1) break;
    const double x[4] = {tile[kl][wr], tile[kl + 1][wr], tile[kl + 2][wr], tile[kl + 3][wr]};
    uint32_t w[S];
    digits4<S>(x, ew, w);
#pragma unroll
    for (int q = 0; q < S; ++q)
      *reinterpret_cast<uint32_t*>(jb.out + q * plane + (int64_t)(r0 + wr) * jb.Kp + kb0 + kl) = w[q];
  }
}

// cols-path jobs in ONE pass (exponent and digits together; X read from HBM once instead of twice):
// a cluster of kSlCS CTAs covers 8 rows x all of K.  CTA c stages k in [c kc, (c + 1) kc) of its 8
// rows in shared memory with 8-byte cp.async (each 8-row k line is a 64-byte coalesced read), the
// cluster combines the per-CTA row maxima through distributed shared memory, and every CTA emits the
// digits of its staged slab, 32 lanes x 4 consecutive k = 128 contiguous bytes of one row per plane.
// Shared tile [kc][8] with the row slot XOR-swizzled by (k >> 2) & 7 (the digit reads of 16 lanes
// then hit 8 distinct slots: at most 2-way conflicts).  8 rows (64 KB at kc = 1024) keep three CTAs
// per SM, so one CTA's digit phase overlaps the others' loads (16 rows / 128 KB ran at 1.7 TB/s).
// Exponents and digits are those of k_oz_colexp2 + k_oz_slice2 (max of |x| over the row, frexp exponent, kExNaN for non-finite rows).
constexpr int kSlCS = 8, kSlRows = 8, kSlKcMax = 1024;
static int slcl_kc(int Kp) { return (int)ceil_div(ceil_div(Kp, kSlCS), 16) * 16; }

template <int S, int kSlRows, int kSlCS>
__device__ __forceinline__ void slicecl_body(const SliceJobs& js, int kc) {
  extern __shared__ double tile[];  // [kc][kSlRows]
  __shared__ double red[256 / kSlRows][kSlRows + 1];
  __shared__ double pm[kSlRows];
  __shared__ int es[kSlRows];
  const SliceJob& jb = job_of(js, blockIdx.x);
  const int b = blockIdx.x - jb.blocks0;  // (blocks0 is a multiple of kSlCS: c is the cluster rank)
  const int c = b % kSlCS, r0 = (b / kSlCS) * kSlRows, k0 = c * kc;
  constexpr int NY = 256 / kSlRows;  // k lines per sweep
  const int tx = threadIdx.x % kSlRows, ty = threadIdx.x / kSlRows;
  const int r = r0 + tx;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(tile);
  for (int k = ty; k < kc; k += NY) {
    const int kg = k0 + k;
    const bool ok = r < jb.rows && kg < jb.K;
    const double* src = ok ? jb.X + (int64_t)kg * jb.ld + r : jb.X;
    const uint32_t dst = sb + 8u * (uint32_t)(k * kSlRows + (tx ^ ((k >> 2) & (kSlRows - 1))));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(ok ? 8 : 0) : "memory");
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  double mx = 0.0;
  bool nf = false;
  for (int k = ty; k < kc; k += NY) {  // (this thread's own copies)
    const double x = tile[k * kSlRows + (tx ^ ((k >> 2) & (kSlRows - 1)))];
    mx = fmax(mx, fabs(x));
    nf |= nonfinite(x);
  }
  const double qnan = __longlong_as_double(0x7ff8000000000000ll);
  red[ty][tx] = nf ? qnan : mx;
  __syncthreads();
  if (threadIdx.x < kSlRows) {
    double m = 0.0;
    bool bad = false;
#pragma unroll
    for (int i = 0; i < NY; ++i) {
      bad |= red[i][threadIdx.x] != red[i][threadIdx.x];
      m = fmax(m, red[i][threadIdx.x]);
    }
    pm[threadIdx.x] = bad ? qnan : m;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (threadIdx.x < kSlRows) {
    double m = 0.0;
    bool bad = false;
    const uint32_t la = (uint32_t)__cvta_generic_to_shared(&pm[threadIdx.x]);
#pragma unroll
    for (int q = 0; q < kSlCS; ++q) {
      uint32_t ra;
      double v;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(q));
      asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(ra) : "memory");
      bad |= v != v;
      m = fmax(m, v);
    }
    const int e = exp_of(m, bad);
    if (c == 0 && r0 + (int)threadIdx.x < jb.rows) jb.ex[r0 + threadIdx.x] = e;
    es[threadIdx.x] = bad ? 0 : e;  // (digits of a non-finite row are never used)
  }
  __syncthreads();
  const int64_t plane = (int64_t)jb.rows * jb.Kp;
  const int nq = min(kc, jb.Kp - k0) / 4;  // quads of this CTA's slab inside Kp (Kp, kc multiples of 16)
  for (int idx = threadIdx.x; idx < kSlRows * nq; idx += 256) {
    const int rr = idx / nq, q = idx - rr * nq;
    if (r0 + rr >= jb.rows) break;
    const int sw = rr ^ (q & (kSlRows - 1));
    const double x[4] = {tile[(4 * q) * kSlRows + sw], tile[(4 * q + 1) * kSlRows + sw],
                         tile[(4 * q + 2) * kSlRows + sw], tile[(4 * q + 3) * kSlRows + sw]};
    uint32_t w[S];
    digits4<S>(x, es[rr], w);
#pragma unroll
    for (int p = 0; p < S; ++p)
      *reinterpret_cast<uint32_t*>(jb.out + p * plane + (int64_t)(r0 + rr) * jb.Kp + k0 + 4 * q) = w[p];
  }
  // no CTA exits while a peer may still read its pm
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int S>
__global__ void __cluster_dims__(kSlCS, 1, 1) __launch_bounds__(256)
    k_oz_slicecl(const __grid_constant__ SliceJobs js, int kc) {
  slicecl_body<S, kSlRows, kSlCS>(js, kc);
}

// opt-in form (SLQ_OZ_SLICE_CS16=1): 16 rows (128-byte k-line segments) over a non-portable cluster of
// 16 CTAs, 64 KB slabs at K = 8192; cluster dimension given at launch
constexpr int kSl16Rows = 16, kSl16CS = 16, kSl16KcMax = 512;
template <int S>
__global__ void __launch_bounds__(256) k_oz_slicecl16(const __grid_constant__ SliceJobs js, int kc) {
  slicecl_body<S, kSl16Rows, kSl16CS>(js, kc);
}

// 2-D int8 tensor [rows x cols] (row pitch ld bytes), box {64, box_rows}, 64-byte swizzle
static CUtensorMap make_map_i8(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                               int box_cols = BK) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_cols == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(SLQ_ECUDA, "cuTensorMapEncodeTiled (int8) failed: " + std::to_string((int)r));
  return m;
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// split-K: one CTA per SM (the stage ring fills the shared memory), so fill the 148 SMs with
// tiles x splits <= 148; every split's K range keeps |acc| <= S * Ksplit * 127^2 < 2^31
static void plan_splits(int S, int tiles, int nk, int KT, int& splits, int& ktps) {
  const int kt_cap = (int)std::max<int64_t>(1, ((int64_t)2147483647 / ((int64_t)S * 127 * 127)) / KT);
  splits = tiles < 148 ? std::max(1, std::min(148 / tiles, nk / 2)) : 1;
  splits = std::max<int>(splits, (int)ceil_div(nk, kt_cap));
  ktps = (int)ceil_div(nk, splits);
  splits = (int)ceil_div(nk, ktps);
}

// W: the wide two-phase kernel (S = 7, BN = 128, 32-byte k-tiles)
template <int S, int BN, bool W = false, int KTN = BK, int NI = 1>
void run(const Launch& L, const GemmArgs<double>& a) {
  using CF = Cfg<S, W ? 64 : BN, KTN>;  // (the wide kernel has its own CfgW; NPROD is the same)
  constexpr int KT = W ? WBK : KTN;
  static bool attr = false;
  if (!attr) {
    if constexpr (W)
      SLQ_CUDA(cudaFuncSetAttribute(k_oz_gemm_w, cudaFuncAttributeMaxDynamicSharedMemorySize, CfgW::SMEM));
    else
      SLQ_CUDA(cudaFuncSetAttribute(k_oz_gemm<S, BN, KTN, NI>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    attr = true;
  }
  const int M = a.M, N = a.N, K = a.K;
  const int Kp = (int)ceil_div(K, 16) * 16;
  const int nk = (int)ceil_div(K, KT);
  const int tiles = (int)(ceil_div(M, BM) * ceil_div(N, BN));
  int splits, ktps;
  plan_splits(S, tiles, nk, KT, splits, ktps);
  const size_t a_bytes = align256((size_t)S * M * Kp), b_bytes = align256((size_t)S * N * Kp);
  const size_t e_bytes = align256(4 * (size_t)(M + N));
  const int nkb = (int)ceil_div(K, kColKMin);  // (sized for the finer exponent blocks)
  const size_t xp_bytes = align256(4 * (size_t)(M + N) * nkb);
  const size_t w_bytes = splits > 1 ? align256(8 * (size_t)M * N * splits) : 0;
  uint8_t* base = (uint8_t*)L.ws->get(a_bytes + b_bytes + e_bytes + xp_bytes + w_bytes, L.stream);
  int8_t* as = (int8_t*)base;
  int8_t* bs = (int8_t*)(base + a_bytes);
  int* ea = (int*)(base + a_bytes + b_bytes);
  int* eb = ea + M;
  int* xpa = (int*)(base + a_bytes + b_bytes + e_bytes);
  int* xpb = xpa + (size_t)M * nkb;
  double* ws = splits > 1 ? (double*)(base + a_bytes + b_bytes + e_bytes + xp_bytes) : nullptr;
  {
    LaunchScope scope(L.prof, KC_OZ_SLICE, L.stream, 0, (8.0 + S) * ((double)M * K + (double)N * K));
    // A(m, k): K-contiguous when sAk == 1 (rows = M, pitch sAm), else stored [K x M] with pitch sAk;
    // B(k, n) = B[k * sBk + n * sBn]: K-contiguous rows per n when sBk == 1 (pitch sBn)
    static const int regrow = getenv("SLQ_OZ_SLICE_L1") ? 0 : 1;  // A/B switch
    SliceJobs js;
    js.n = 2;
    js.regrow = regrow;
    js.j[0] = SliceJob{a.A, a.sAk == 1 ? a.sAm : a.sAk, M, K, Kp, a.sAk == 1 ? 1 : 0, as, ea, xpa, 0, col_kblk(M, K)};
    js.j[1] = SliceJob{a.B, a.sBk == 1 ? a.sBn : a.sBk, N, K, Kp, a.sBk == 1 ? 1 : 0, bs, eb, xpb, 0, col_kblk(N, K)};
    static const bool twopass = getenv("SLQ_OZ_SLICE_TWOPASS") != nullptr;  // A/B switch
    const int kc = slcl_kc(Kp);
    if (!twopass && kc <= kSlKcMax) {
      // cols-path jobs: one fused cluster launch; rows-path jobs: k_oz_slice2
      static bool cl_attr = false;
      if (!cl_attr) {
        SLQ_CUDA(cudaFuncSetAttribute(k_oz_slicecl<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kSlKcMax * kSlRows * 8));
        cl_attr = true;
      }
      SliceJobs jc, jr;
      jc.n = jr.n = 0;
      jr.regrow = regrow;
      int ncl = 0, nr = 0;
      for (int i = 0; i < 2; ++i) {
        SliceJob jj = js.j[i];
        if (jj.kmajor) {
          jj.blocks0 = nr;
          nr += (int)ceil_div(jj.rows, 8);
          jr.j[jr.n++] = jj;
        } else {
          jj.blocks0 = ncl;
          ncl += (int)ceil_div(jj.rows, kSlRows) * kSlCS;
          jc.j[jc.n++] = jj;
        }
      }
      if (ncl > 0) {
        if (jc.n == 1) jc.j[1] = jc.j[0];
        static const bool cs16 = getenv("SLQ_OZ_SLICE_CS16") && atoi(getenv("SLQ_OZ_SLICE_CS16")) != 0;
        static int cs16_ok = -1;  // the 16-CTA cluster of 64 KB slabs fits (cudaOccupancyMaxActiveClusters)
        const int kc16 = (int)ceil_div(ceil_div(Kp, kSl16CS), 16) * 16;
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        if (cs16 && kc16 <= kSl16KcMax) {
          cfg.blockDim = dim3(256);
          cfg.dynamicSmemBytes = (size_t)kc16 * kSl16Rows * 8;
          cfg.stream = L.stream;
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = kSl16CS;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          if (cs16_ok < 0) {
            SLQ_CUDA(cudaFuncSetAttribute(k_oz_slicecl16<S>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            SLQ_CUDA(cudaFuncSetAttribute(k_oz_slicecl16<S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          kSl16KcMax * kSl16Rows * 8));
            cfg.gridDim = dim3(kSl16CS);
            cfg.dynamicSmemBytes = (size_t)kSl16KcMax * kSl16Rows * 8;
            int nclu = 0;
            cs16_ok = cudaOccupancyMaxActiveClusters(&nclu, k_oz_slicecl16<S>, &cfg) == cudaSuccess && nclu > 0;
            (void)cudaGetLastError();
            cfg.dynamicSmemBytes = (size_t)kc16 * kSl16Rows * 8;
          }
        }
        if (cs16 && kc16 <= kSl16KcMax && cs16_ok == 1) {
          SliceJobs j16 = jc;
          int n16 = 0;
          for (int i = 0; i < j16.n; ++i) {
            j16.j[i].blocks0 = n16;
            n16 += (int)ceil_div(j16.j[i].rows, kSl16Rows) * kSl16CS;
          }
          if (j16.n == 1) j16.j[1] = j16.j[0];
          cfg.gridDim = dim3(n16);
          SLQ_CUDA(cudaLaunchKernelEx(&cfg, k_oz_slicecl16<S>, j16, kc16));
        } else {
          k_oz_slicecl<S><<<ncl, 256, (size_t)kc * kSlRows * 8, L.stream>>>(jc, kc);
        }
        SLQ_CUDA(cudaGetLastError());
        ++*L.launches;
      }
      if (nr > 0) {
        if (jr.n == 1) jr.j[1] = jr.j[0];
        k_oz_slice2<S><<<nr, 256, 0, L.stream>>>(jr);
        SLQ_CUDA(cudaGetLastError());
        ++*L.launches;
      }
    } else {
    // exponent pass (cols-path jobs only)
    int nexp = 0;
    SliceJobs je;
    je.n = 0;
    for (int i = 0; i < 2; ++i)
      if (!js.j[i].kmajor) {
        SliceJob jj = js.j[i];
        jj.blocks0 = nexp;
        nexp += (int)(ceil_div(jj.rows, 32) * ceil_div(K, jj.kcol));
        je.j[je.n++] = jj;
      }
    if (je.n == 1) je.j[1] = je.j[0];
    if (nexp > 0) {
      k_oz_colexp2<<<nexp, 256, 0, L.stream>>>(je);
      SLQ_CUDA(cudaGetLastError());
      ++*L.launches;
    }
    int nsl = 0;
    for (int i = 0; i < 2; ++i) {
      js.j[i].blocks0 = nsl;
      nsl += js.j[i].kmajor ? (int)ceil_div(js.j[i].rows, 8) : (int)(ceil_div(js.j[i].rows, 32) * ceil_div(Kp, 128));
    }
    k_oz_slice2<S><<<nsl, 256, 0, L.stream>>>(js);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
    }
  }
  const CUtensorMap ta = make_map_i8(as, (int64_t)S * M, Kp, Kp, BM, KT);
  const CUtensorMap tb = make_map_i8(bs, (int64_t)S * N, Kp, Kp, BN, KT);
  static const int dbg = getenv("SLQ_OZ_DEBUG") ? atoi(getenv("SLQ_OZ_DEBUG")) : 0;
  static const int order = getenv("SLQ_OZ_ORDER") ? atoi(getenv("SLQ_OZ_ORDER")) : -1;  // 0 n-fast, 1 m-fast
  OzArgs o{M, N, nk, ktps, splits, ea, eb, dbg, order >= 0 ? order : (N > M ? 1 : 0)};
  o.tiles_b = tiles;
  {
    LaunchScope scope(L.prof, KC_GEMM_I8, L.stream, 2.0 * M * N * (double)K * CF::NPROD,
                      (double)S * ((double)M * K + (double)N * K) + 8.0 * M * N);
    const int nwork = tiles * splits;
    if constexpr (W)
      k_oz_gemm_w<<<std::min(nwork, 148), 320, CfgW::SMEM, L.stream>>>(ta, tb, o, a, ws);
    else
      k_oz_gemm<S, BN, KTN, NI><<<std::min(nwork, 148), 32 * (CF::NE + NI + 1), CF::SMEM, L.stream>>>(ta, tb, o, a, ws,
                                                                                                   ta);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
  if (splits > 1) {
    LaunchScope scope(L.prof, KC_GEMM, L.stream, 0, 8.0 * (double)M * N * (splits + 1));
    const int64_t mn = (int64_t)M * N;
    int blocks = (int)std::min<int64_t>(ceil_div(mn, 256), 148 * 8);
    gemm_detail::splitk_reduce<double><<<blocks, 256, 0, L.stream>>>(a, splits, ws);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
}

// 2-D fp64 tensor [rows x cols] (row pitch ld elements), box {16, 32}, 128-byte swizzle: the TS
// epilogue's store map
static CUtensorMap make_map_f64_store(const double* base, int64_t rows, int64_t cols, int64_t ld) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  cuuint32_t box[2] = {16, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(SLQ_ECUDA, "cuTensorMapEncodeTiled (fp64 store) failed: " + std::to_string((int)r));
  return m;
}

// batched / causal GEMM over pre-sliced digit planes (the attention path): no slicing, no split-K.
// TS: the TMA-store epilogue (one pipeline stage; only for plain outputs with contiguous batches)
template <int S, int BN, int NI, bool TS>
void run_planes(const Launch& L, const OzPlanes& A, const OzPlanes& B, const GemmArgs<double>& a) {
  using CF = Cfg<S, BN, BK, TS>;
  static bool attr = false;
  if (!attr) {
    SLQ_CUDA(cudaFuncSetAttribute(k_oz_gemm<S, BN, BK, NI, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    attr = true;
  }
  const int M = a.M, N = a.N, K = a.K;
  const int nk = (int)ceil_div(K, BK);
  const int tm = (int)ceil_div(M, BM), tn = (int)ceil_div(N, BN);
  int tiles_b = tm * tn;
  if (a.tri == TRI_SKIP_UPPER) {
    tiles_b = 0;
    for (int mt = 0; mt < tm; ++mt) tiles_b += std::min(tn, (mt * BM + BM - 1) / BN + 1);
  }
  const CUtensorMap ta = make_map_i8(A.d, (int64_t)S * A.nb * M, A.Kp, A.Kp, BM, BK);
  const CUtensorMap tb = make_map_i8(B.d, (int64_t)S * B.nb * N, B.Kp, B.Kp, BN, BK);
  const CUtensorMap tc = TS ? make_map_f64_store(a.C, (int64_t)a.batch * M, N, a.ldc) : ta;
  static const int dbg = getenv("SLQ_OZ_DEBUG") ? atoi(getenv("SLQ_OZ_DEBUG")) : 0;  // diagnostic only
  OzArgs o{M, N, nk, nk, 1, A.ex, B.ex, dbg, 0};
  o.batch = a.batch; o.tri = a.tri; o.tiles_b = tiles_b;
  o.nbA = A.nb; o.nbB = B.nb; o.z0A = A.z0; o.z0B = B.z0; o.zA = A.z; o.zB = B.z;
  // algorithmic work: the causal half (T + 1) / 2T of the square for the triangular contractions
  const double frac = a.tri == TRI_NONE ? 1.0 : (a.tri == TRI_SKIP_UPPER ? (M + 1.0) / (2.0 * M) : (K + 1.0) / (2.0 * K));
  LaunchScope scope(L.prof, KC_ATTN_I8, L.stream, 2.0 * M * N * (double)K * a.batch * CF::NPROD * frac,
                    (double)S * ((double)M * K + (double)N * K) * a.batch * frac + 8.0 * M * N * a.batch);
  const int64_t nwork = (int64_t)a.batch * tiles_b;
  k_oz_gemm<S, BN, BK, NI, TS><<<(int)std::min<int64_t>(nwork, 148), 32 * (CF::NE + NI + 1), CF::SMEM, L.stream>>>(
      ta, tb, o, a, nullptr, tc);
  SLQ_CUDA(cudaGetLastError());
  ++*L.launches;
}

template <int S, int BN, int NI>
void run_planes_sel(const Launch& L, const OzPlanes& A, const OzPlanes& B, const GemmArgs<double>& a) {
  static const bool ts_off = getenv("SLQ_OZ_NO_TMA_STORE") && atoi(getenv("SLQ_OZ_NO_TMA_STORE")) != 0;  // A/B
  const bool ts = !ts_off && a.K <= 2 * BK && !a.accumulate && !a.bias && !a.resid && a.offC.inner == 0 &&
                  a.offC.div == 1 && (a.batch == 1 || (a.offC.outer == (int64_t)a.M * a.ldc && a.M % BM == 0)) &&
                  (a.ldc % 2) == 0 && (((uintptr_t)a.C) & 15) == 0;
  if (ts) run_planes<S, BN, NI, true>(L, A, B, a);
  else run_planes<S, BN, NI, false>(L, A, B, a);
}

}  // namespace oz

// output tile width of the production kernel for S digit planes: the S accumulators of BN columns
// share the 512 TMEM columns (S = 5: 5 x 96 = 480; S = 6, 7: 64)
static int oz_bn(int S) { return S == 5 ? 96 : 64; }

// workspace of the production configuration (BN = oz_bn(S), 64-byte k-tiles; the diagnostic wide /
// 32-byte variants size their own)
size_t oz_ws_bytes(int M, int N, int K, int S) {
  using namespace oz;
  const int Kp = (int)ceil_div(K, 16) * 16, nk = (int)ceil_div(K, BK);
  const int tiles = (int)(ceil_div(M, BM) * ceil_div(N, oz_bn(S)));
  int splits, ktps;
  plan_splits(S, tiles, nk, BK, splits, ktps);
  const int nkb = (int)ceil_div(K, kColKMin);
  return align256((size_t)S * M * Kp) + align256((size_t)S * N * Kp) + align256(4 * (size_t)(M + N)) +
         align256(4 * (size_t)(M + N) * nkb) + (splits > 1 ? align256(8 * (size_t)M * N * splits) : 0);
}

void gemm_oz(const Launch& L, const GemmArgs<double>& a, int S) {
  SLQ_CHECK_ARG(a.batch == 1 && a.tri == TRI_NONE && a.M > 0 && a.N > 0 && a.K > 0, "oz gemm: batch 1, dense");
  static const bool wide = getenv("SLQ_OZ_BN") && atoi(getenv("SLQ_OZ_BN")) == 128;  // diagnostic
  switch (S) {
    case 4:
      if (wide) oz::run<4, 128>(L, a);
      else oz::run<4, 64>(L, a);
      break;
    // S = 5 / 6 (the bf16 models' default is 5): two issuers as for S = 7; S = 5 on 128 x 96 tiles
    case 5: oz::run<5, 96, false, oz::BK, 2>(L, a); break;
    case 6: oz::run<6, 64, false, oz::BK, 2>(L, a); break;
    default: {
      // the wide two-phase kernel when it has enough 128 x 128 tiles to fill the GPU
      static const int wide_env = getenv("SLQ_OZ_WIDE") ? atoi(getenv("SLQ_OZ_WIDE")) : 0;
      const int64_t t128 = ceil_div(a.M, oz::BM) * ceil_div(a.N, oz::WBN);
      static const int kt_env = getenv("SLQ_OZ_BK") ? atoi(getenv("SLQ_OZ_BK")) : 64;
      static const int ni_env = getenv("SLQ_OZ_ISSUERS") ? atoi(getenv("SLQ_OZ_ISSUERS")) : 2;
      if (wide_env == 2 || (wide_env == 1 && t128 >= 148))
        oz::run<7, 128, true>(L, a);
      else if (kt_env == 32)
        oz::run<7, 64, false, 32>(L, a);
      else if (ni_env == 3)
        oz::run<7, 64, false, oz::BK, 3>(L, a);
      else if (ni_env == 1)
        oz::run<7, 64>(L, a);
      else
        oz::run<7, 64, false, oz::BK, 2>(L, a);
      break;
    }
  }
}

void gemm_oz_planes(const Launch& L, int S, const OzPlanes& A, const OzPlanes& B, const GemmArgs<double>& a) {
  SLQ_CHECK_ARG(a.M > 0 && a.N > 0 && a.K > 0 && a.batch >= 1 && A.Kp == B.Kp && A.Kp % 16 == 0 && A.Kp >= a.K,
                "oz planes gemm: shapes");
  // head-dimension outputs (N <= 128): 128 x 64 tiles; S = 5 otherwise on 128 x 96
  const bool narrow = a.N <= 128;
  switch (S) {
    case 4: oz::run_planes_sel<4, 64, 1>(L, A, B, a); break;
    case 5:
      if (narrow) oz::run_planes_sel<5, 64, 2>(L, A, B, a);
      else oz::run_planes_sel<5, 96, 2>(L, A, B, a);
      break;
    case 6: oz::run_planes_sel<6, 64, 2>(L, A, B, a); break;
    case 7: oz::run_planes_sel<7, 64, 2>(L, A, B, a); break;
    default: throw Error(SLQ_EINVAL, "oz planes gemm: S in 4..7");
  }
}

}  // namespace slq

namespace slq {
namespace oz {
__global__ void k_fill_f64(double* x, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    // wide dynamic range: mantissa in [-1, 1) times 2^(-8 .. 7)
    const double m = (double)(int64_t)(z >> 11) / 4503599627370496.0 - 1.0;
    x[i] = ldexp(m, (int)((z >> 3) & 15) - 8);
  }
}
}  // namespace oz
}  // namespace slq

extern "C" slq_status slq_diag_oz_check(int32_t device, int32_t M, int32_t N, int32_t K, int32_t a_kmajor,
                                        int32_t b_kmajor, int32_t S, int32_t iters, double* max_err,
                                        double* tflops) {
  using namespace slq;
  double *A = nullptr, *B = nullptr, *C1 = nullptr, *C2 = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto cleanup = [&] {
    if (A) cudaFree(A);
    if (B) cudaFree(B);
    if (C1) cudaFree(C1);
    if (C2) cudaFree(C2);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
  };
  try {
    SLQ_CHECK_ARG(M > 0 && N > 0 && K > 0 && S >= 4 && S <= 7 && iters >= 1 && max_err && tflops, "arguments");
    SLQ_CUDA(cudaSetDevice(device));
    SLQ_CUDA(cudaMalloc(&A, sizeof(double) * (size_t)M * K));
    SLQ_CUDA(cudaMalloc(&B, sizeof(double) * (size_t)N * K));
    SLQ_CUDA(cudaMalloc(&C1, sizeof(double) * (size_t)M * N));
    SLQ_CUDA(cudaMalloc(&C2, sizeof(double) * (size_t)M * N));
    oz::k_fill_f64<<<1024, 256>>>(A, (int64_t)M * K, 11);
    oz::k_fill_f64<<<1024, 256>>>(B, (int64_t)N * K, 12);
    Workspace ws;
    int64_t launches = 0;
    Launch L{0, nullptr, &ws, &launches};
    GemmArgs<double> a;
    a.M = M; a.N = N; a.K = K;
    a.A = A; a.sAm = a_kmajor ? K : 1; a.sAk = a_kmajor ? 1 : M;
    a.B = B; a.sBk = b_kmajor ? 1 : N; a.sBn = b_kmajor ? K : 1;
    a.ldc = N;
    a.C = C1;
    gemm<double>(L, a);  // DMMA reference (gemm_mode 0)
    a.C = C2;
    gemm_oz(L, a, S);
    SLQ_CUDA(cudaDeviceSynchronize());
    SLQ_CUDA(cudaEventCreate(&e0));
    SLQ_CUDA(cudaEventCreate(&e1));
    SLQ_CUDA(cudaEventRecord(e0));
    for (int i = 0; i < iters; ++i) gemm_oz(L, a, S);
    SLQ_CUDA(cudaEventRecord(e1));
    SLQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SLQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *tflops = 2.0 * M * N * (double)K * iters / (ms * 1e-3) / 1e12;
    std::vector<double> hA((size_t)M * K), hB((size_t)N * K), h1((size_t)M * N), h2((size_t)M * N);
    SLQ_CUDA(cudaMemcpy(hA.data(), A, sizeof(double) * hA.size(), cudaMemcpyDeviceToHost));
    SLQ_CUDA(cudaMemcpy(hB.data(), B, sizeof(double) * hB.size(), cudaMemcpyDeviceToHost));
    SLQ_CUDA(cudaMemcpy(h1.data(), C1, sizeof(double) * h1.size(), cudaMemcpyDeviceToHost));
    SLQ_CUDA(cudaMemcpy(h2.data(), C2, sizeof(double) * h2.size(), cudaMemcpyDeviceToHost));
    std::vector<double> ra(M, 0.0), cb(N, 0.0);
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k) ra[m] = std::max(ra[m], fabs(hA[a_kmajor ? (size_t)m * K + k : (size_t)k * M + m]));
    for (int n = 0; n < N; ++n)
      for (int k = 0; k < K; ++k) cb[n] = std::max(cb[n], fabs(hB[b_kmajor ? (size_t)n * K + k : (size_t)k * N + n]));
    double worst = 0.0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        const double den = (double)K * ra[m] * cb[n];
        const double d = fabs(h1[(size_t)m * N + n] - h2[(size_t)m * N + n]);
        if (!std::isfinite(h2[(size_t)m * N + n])) worst = INFINITY;
        else if (den > 0) worst = std::max(worst, d / den);
      }
    *max_err = worst;
    cleanup();
    return SLQ_OK;
  } catch (const Error& e) {
    cleanup();
    return e.status;
  }
}
