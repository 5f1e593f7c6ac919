// bf16 GEMM on the 5th-generation tensor cores (tcgen05.mma, accumulators in TMEM), operands
// streamed by TMA (cp.async.bulk.tensor, 128B swizzle) through an mbarrier pipeline.
//
//   C[M x N] (fp32) = A[M x K] . B[N x K]^T      A, B bf16, both K-contiguous ("TN")
//
// Warp-specialised CTA (192 threads): warp 0 = TMA producer (one elected lane), warp 1 = TMEM
// allocator + MMA issuer (one elected lane issues tcgen05.mma for the whole CTA), warps 2..5 =
// epilogue (tcgen05.ld from TMEM -> registers -> global).  Tile 128 x BN x 64, STAGES-deep ring of
// {full, empty} mbarriers; tcgen05.commit releases a stage when the MMAs that read it complete.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <vector>

#include "common.h"
#include "gemm_common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace slq {
namespace tc {

constexpr int BM = 128, BK = 64, UMMA_K = 16;

// instruction descriptor for kind::f16: D f32, A/B bf16, both K-major, shape M x N
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4)                    // D format F32
         | (1u << 7)                  // A format BF16
         | (1u << 10)                 // B format BF16
         | ((uint32_t)(N >> 3) << 17)  // N
         | ((uint32_t)(M >> 4) << 24);  // M
}

template <int BN, int STAGES>
struct Cfg {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;  // power of two >= 32
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_tc_gemm(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, float* __restrict__ C,
              int M, int N, int K, int64_t ldc) {
  using CF = Cfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
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
    if (lane == 0) {  // ---- TMA producer ----
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % STAGES;
        const uint32_t ph = (kt / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * CF::STAGE_BYTES;
        uint8_t* sb = sa + CF::A_BYTES;
        mbar_expect_tx(&full[s], CF::STAGE_BYTES);
        tma_load_2d(sa, &tmA, &full[s], kt * BK, m0);
        tma_load_2d(sb, &tmB, &full[s], kt * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      constexpr uint32_t idesc = make_idesc(BM, BN);
      for (int kt = 0; kt < nk; ++kt) {
        const int s = kt % STAGES;
        const uint32_t ph = (kt / STAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const uint32_t sa = smem_u32(smem + s * CF::STAGE_BYTES);
        const uint32_t sb = sa + CF::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
          const uint64_t da = make_desc_sw128(sa + kk * UMMA_K * 2);
          const uint64_t db = make_desc_sw128(sb + kk * UMMA_K * 2);
          const uint32_t acc = (kt | kk) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&empty[s])));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
          smem_u32(tmem_full)));
    }
  } else {  // ---- epilogue: warps 2..5, warp w owns TMEM lanes 32*(w%4) .. +31 ----
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    const int lg = (warp % 4) * 32;
    const int row = m0 + lg + lane;
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      const uint32_t taddr = tmem + ((uint32_t)lg << 16) + (uint32_t)c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
      if (row < M) {
        float* dst = C + (int64_t)row * ldc + n0 + c;
        if (n0 + c + 16 <= N && (ldc % 4) == 0) {
#pragma unroll
          for (int i = 0; i < 16; i += 4)
            *reinterpret_cast<float4*>(dst + i) =
                make_float4(__uint_as_float(r[i]), __uint_as_float(r[i + 1]), __uint_as_float(r[i + 2]),
                            __uint_as_float(r[i + 3]));
        } else {
          for (int i = 0; i < 16; ++i)
            if (n0 + c + i < N) dst[i] = __uint_as_float(r[i]);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(CF::TMEM_COLS));
  }
}

// 2-D bf16 tensor [rows x cols] with row pitch `ld` elements, K (=cols) innermost; box {64, box_rows}
static CUtensorMap make_map_bf16(const void* base, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(SLQ_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

template <int BN, int STAGES>
void launch(cudaStream_t s, const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc, int M,
            int N, int K) {
  using CF = Cfg<BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    SLQ_CUDA(cudaFuncSetAttribute(k_tc_gemm<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    attr = true;
  }
  SLQ_CHECK_ARG((lda * 2) % 16 == 0 && (ldb * 2) % 16 == 0, "TMA needs 16-byte row pitches");
  SLQ_CHECK_ARG(((uintptr_t)A % 16) == 0 && ((uintptr_t)B % 16) == 0, "TMA needs 16-byte aligned bases");
  const CUtensorMap ta = make_map_bf16(A, M, K, lda, BM);
  const CUtensorMap tb = make_map_bf16(B, N, K, ldb, BN);
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM));
  k_tc_gemm<BN, STAGES><<<grid, 192, CF::SMEM, s>>>(ta, tb, C, M, N, K, ldc);
  SLQ_CUDA(cudaGetLastError());
}

// ------------------------------------------------------------------------------------------
// Multi-product variant: C = epilogue( sum_p A[ai_p] . B[bi_p]^T ), all products accumulated in
// one TMEM accumulator; the K loop runs over (product, k-tile) pairs, so a split-operand GEMM is
// one long-K tensor-core GEMM.  Optional split-K over that sequence (partials to a workspace,
// deterministic reduce).
constexpr int kMaxTerms = 6, kMaxPairs = 12;
struct MultiOps {
  CUtensorMap a[kMaxTerms];
  CUtensorMap b[kMaxTerms];
  int npairs;
  int ai[kMaxPairs], bi[kMaxPairs];
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(192, 1)
    k_tc_multi(const __grid_constant__ MultiOps ops, GemmArgs<float> p, int nk, int tiles_per_split, int splits,
               float* __restrict__ ws) {
  using CF = Cfg<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * CF::STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int split = blockIdx.z;
  const int total = ops.npairs * nk;
  const int t0 = split * tiles_per_split;
  const int t1 = min(total, t0 + tiles_per_split);
  const int nloc = t1 > t0 ? t1 - t0 : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
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
    if (lane == 0) {
      for (int i = 0; i < nloc; ++i) {
        const int t = t0 + i, pr = t / nk, kt = t % nk;
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * CF::STAGE_BYTES;
        uint8_t* sb = sa + CF::A_BYTES;
        mbar_expect_tx(&full[s], CF::STAGE_BYTES);
        tma_load_2d(sa, &ops.a[ops.ai[pr]], &full[s], kt * BK, m0);
        tma_load_2d(sb, &ops.b[ops.bi[pr]], &full[s], kt * BK, n0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc(BM, BN);
      for (int i = 0; i < nloc; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const uint32_t sa = smem_u32(smem + s * CF::STAGE_BYTES);
        const uint32_t sb = sa + CF::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
          const uint64_t da = make_desc_sw128(sa + kk * UMMA_K * 2);
          const uint64_t db = make_desc_sw128(sb + kk * UMMA_K * 2);
          const uint32_t acc = (i | kk) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
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
  } else {
    // Epilogue: TMEM -> registers -> shared tile (the pipeline buffers are free once the last
    // MMA committed) -> coalesced row-contiguous global stores with the fused epilogue.
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    const int lg = (warp % 4) * 32;
    constexpr int LDS = BN + 1;
    float* Cs = reinterpret_cast<float*>(smem);
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      uint32_t r[16];
      const uint32_t taddr = tmem + ((uint32_t)lg << 16) + (uint32_t)c;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
      for (int i = 0; i < 16; ++i) Cs[(lg + lane) * LDS + c + i] = nloc > 0 ? __uint_as_float(r[i]) : 0.0f;
    }
    asm volatile("bar.sync 1, 128;\n" ::);  // the four epilogue warps only
    float* W = splits > 1 ? ws + (int64_t)split * p.M * p.N : nullptr;
    const int et = threadIdx.x - 64;
    const int rows = min(BM, p.M - m0), cols = min(BN, p.N - n0);
#pragma unroll 1
    for (int e = et; e < BM * BN; e += 128) {
      const int rr = e / BN, cc = e % BN;
      if (rr >= rows || cc >= cols) continue;
      const float v = Cs[rr * LDS + cc];
      if (W)
        W[(int64_t)(m0 + rr) * p.N + n0 + cc] = v;
      else
        gemm_detail::epilogue_store(p, p.C, m0 + rr, n0 + cc, v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(CF::TMEM_COLS));
  }
}

// x = t0 + t1 + t2 in bf16 terms (each residual is exact in fp32); optional transpose through a
// 32 x 32 shared tile so that every operand reaches the tensor core K-contiguous
template <bool TRANS, int NT = 3>
__global__ void k_split3(const float* __restrict__ X, int64_t R, int64_t C, int64_t ld, __nv_bfloat16* __restrict__ o0,
                         __nv_bfloat16* __restrict__ o1, __nv_bfloat16* __restrict__ o2, int64_t ldo) {
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8 threads
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    tile[i][tx] = (r < R && c < C) ? X[r * ld + c] : 0.0f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    float x;
    int64_t orow, ocol;
    if (TRANS) {
      x = tile[tx][i];
      orow = c0 + i;
      ocol = r0 + tx;
      if (orow >= C || ocol >= R) continue;
    } else {
      x = tile[i][tx];
      orow = r0 + i;
      ocol = c0 + tx;
      if (orow >= R || ocol >= C) continue;
    }
    const __nv_bfloat16 b0 = __float2bfloat16_rn(x);
    const int64_t o = orow * ldo + ocol;
    o0[o] = b0;
    if constexpr (NT == 3) {
      const float e1 = x - __bfloat162float(b0);
      const __nv_bfloat16 b1 = __float2bfloat16_rn(e1);
      const float e2 = e1 - __bfloat162float(b1);
      o1[o] = b1;
      o2[o] = __float2bfloat16_rn(e2);
    }
  }
}

template <int BN>
void launch_multi(const Launch& L, const MultiOps& ops, const GemmArgs<float>& a, int nk, int splits, int tps,
                  float* ws) {
  // two CTAs per SM (one's epilogue overlaps the other's MMAs); the smem also hosts the fp32
  // epilogue tile BM x (BN + 1)
  constexpr int STAGES = BN == 128 ? 3 : 4;
  using CF = Cfg<BN, STAGES>;
  static_assert(BM * (BN + 1) * 4 <= STAGES * CF::STAGE_BYTES, "epilogue tile fits the pipeline smem");
  static bool attr = false;
  if (!attr) {
    SLQ_CUDA(cudaFuncSetAttribute(k_tc_multi<BN, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM));
    attr = true;
  }
  dim3 grid((unsigned)ceil_div(a.N, BN), (unsigned)ceil_div(a.M, BM), (unsigned)splits);
  k_tc_multi<BN, STAGES><<<grid, 192, CF::SMEM, L.stream>>>(ops, a, nk, tps, splits, ws);
  SLQ_CUDA(cudaGetLastError());
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

}  // namespace tc

size_t tc_ws_bytes(int M, int N, int K, int terms) {
  using namespace tc;
  const int64_t ldk = (K + 7) / 8 * 8;
  const size_t a_bytes = align256(2 * (size_t)M * ldk), b_bytes = align256(2 * (size_t)N * ldk);
  const int npairs = terms == 1 ? 1 : 6, nk = (K + BK - 1) / BK;
  const int64_t t128 = ceil_div(M, BM) * ceil_div(N, 128);
  const int bn = t128 >= 148 ? 128 : 64;
  const int tiles = (int)(ceil_div(M, BM) * ceil_div(N, bn));
  const int total = npairs * nk;
  int splits = 1;
  if (tiles < 148) splits = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * 148, tiles), total / 4));
  const int tps = (int)ceil_div(total, splits);
  splits = (int)ceil_div(total, tps);
  return terms * (a_bytes + b_bytes) + (splits > 1 ? align256(4 * (size_t)M * N * splits) : 0);
}

void gemm_tc_bf16x3(const Launch& L, const GemmArgs<float>& a, int terms) {
  using namespace tc;
  SLQ_CHECK_ARG(a.batch == 1 && a.M > 0 && a.N > 0 && a.K > 0, "tc gemm: batch 1, non-empty");
  SLQ_CHECK_ARG(terms == 1 || terms == 3, "tc gemm: 1 or 3 bf16 terms");
  const int M = a.M, N = a.N, K = a.K;
  const int64_t ldk = (K + 7) / 8 * 8;  // 16-byte row pitch for TMA
  const size_t a_bytes = align256(2 * (size_t)M * ldk), b_bytes = align256(2 * (size_t)N * ldk);
  // product list (i + j <= 2); one term: the leading product only
  static const int AI[6] = {0, 0, 1, 1, 0, 2}, BI[6] = {0, 1, 0, 1, 2, 0};
  const int npairs = terms == 1 ? 1 : 6, nk = (K + BK - 1) / BK;
  const int64_t t128 = ceil_div(M, BM) * ceil_div(N, 128);
  const int bn = t128 >= 148 ? 128 : 64;
  const int tiles = (int)(ceil_div(M, BM) * ceil_div(N, bn));
  const int total = npairs * nk;
  int splits = 1;
  if (tiles < 148) splits = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * 148, tiles), total / 4));
  const int tps = (int)ceil_div(total, splits);
  splits = (int)ceil_div(total, tps);
  const size_t w_bytes = splits > 1 ? align256(4 * (size_t)M * N * splits) : 0;
  uint8_t* base = (uint8_t*)L.ws->get(terms * (a_bytes + b_bytes) + w_bytes, L.stream);
  __nv_bfloat16* at[3] = {nullptr, nullptr, nullptr};
  __nv_bfloat16* bt[3] = {nullptr, nullptr, nullptr};
  for (int i = 0; i < terms; ++i) {
    at[i] = (__nv_bfloat16*)(base + i * a_bytes);
    bt[i] = (__nv_bfloat16*)(base + terms * a_bytes + i * b_bytes);
  }
  float* ws = splits > 1 ? (float*)(base + terms * (a_bytes + b_bytes)) : nullptr;
  {  // split (and transpose to K-contiguous where needed)
    LaunchScope scope(L.prof, KC_ELEM, L.stream, 0, (4.0 + 2.0 * terms) * ((double)M * K + (double)N * K));
    auto split = [&](const float* X, int64_t R, int64_t C, int64_t ld, bool trans, __nv_bfloat16** o) {
      dim3 g((unsigned)ceil_div(C, 32), (unsigned)ceil_div(R, 32));
      if (terms == 1) {
        if (trans) k_split3<true, 1><<<g, 256, 0, L.stream>>>(X, R, C, ld, o[0], o[1], o[2], ldk);
        else k_split3<false, 1><<<g, 256, 0, L.stream>>>(X, R, C, ld, o[0], o[1], o[2], ldk);
      } else {
        if (trans) k_split3<true, 3><<<g, 256, 0, L.stream>>>(X, R, C, ld, o[0], o[1], o[2], ldk);
        else k_split3<false, 3><<<g, 256, 0, L.stream>>>(X, R, C, ld, o[0], o[1], o[2], ldk);
      }
      SLQ_CUDA(cudaGetLastError());
    };
    if (a.sAk == 1) split(a.A, M, K, a.sAm, false, at);
    else split(a.A, K, M, a.sAk, true, at);  // A stored [K x M] (M contiguous) -> [M x K]
    if (a.sBk == 1) split(a.B, N, K, a.sBn, false, bt);  // B(k, n) at n*sBn + k: stored [N x K]
    else split(a.B, K, N, a.sBk, true, bt);               // stored [K x N] -> [N x K]
    *L.launches += 2;
  }
  MultiOps ops;
  for (int i = 0; i < terms; ++i) {
    ops.a[i] = make_map_bf16(at[i], M, K, ldk, BM);
    ops.b[i] = make_map_bf16(bt[i], N, K, ldk, bn);
  }
  ops.npairs = npairs;
  for (int i = 0; i < npairs; ++i) {
    ops.ai[i] = AI[i];
    ops.bi[i] = BI[i];
  }
  {
    LaunchScope scope(L.prof, KC_GEMM, L.stream, 2.0 * M * N * (double)K * npairs,
                      2.0 * 3 * ((double)M * K + (double)N * K) + 4.0 * M * N);
    if (bn == 128)
      launch_multi<128>(L, ops, a, nk, splits, tps, ws);
    else
      launch_multi<64>(L, ops, a, nk, splits, tps, ws);
    ++*L.launches;
  }
  if (splits > 1) {
    LaunchScope scope(L.prof, KC_GEMM, L.stream, 0, 4.0 * (double)M * N * (splits + 1));
    const int64_t mn = (int64_t)M * N;
    int blocks = (int)std::min<int64_t>(ceil_div(mn, 256), 148 * 8);
    gemm_detail::splitk_reduce<float><<<blocks, 256, 0, L.stream>>>(a, splits, ws);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
}

// ---- general split / multi-product launch (used by the paired evaluation) ----

size_t tc_terms_bytes(int rows, int K) {
  const int64_t ldk = (K + 7) / 8 * 8;
  return 3 * tc::align256(2 * (size_t)rows * ldk);
}

TcTerms tc_split_terms(const Launch& L, const float* X, int rows, int K, int64_t s_row, int64_t s_k, void* dst) {
  using namespace tc;
  SLQ_CHECK_ARG(s_k == 1 || s_row == 1, "tc split: one stride must be 1");
  TcTerms t;
  t.rows = rows;
  t.ldk = (K + 7) / 8 * 8;
  const size_t one = align256(2 * (size_t)rows * t.ldk);
  for (int i = 0; i < 3; ++i) t.t[i] = (uint8_t*)dst + i * one;
  auto* o0 = (__nv_bfloat16*)t.t[0];
  auto* o1 = (__nv_bfloat16*)t.t[1];
  auto* o2 = (__nv_bfloat16*)t.t[2];
  LaunchScope scope(L.prof, KC_ELEM, L.stream, 0, 10.0 * (double)rows * K);
  if (s_k == 1) {  // [rows x K] with row pitch s_row
    dim3 g((unsigned)ceil_div(K, 32), (unsigned)ceil_div(rows, 32));
    k_split3<false><<<g, 256, 0, L.stream>>>(X, rows, K, s_row, o0, o1, o2, t.ldk);
  } else {  // stored [K x rows] with row pitch s_k -> transposed
    dim3 g((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(K, 32));
    k_split3<true><<<g, 256, 0, L.stream>>>(X, K, rows, s_k, o0, o1, o2, t.ldk);
  }
  SLQ_CUDA(cudaGetLastError());
  ++*L.launches;
  return t;
}

TcPlan tc_plan(int M, int N, int K, int nprods) {
  using namespace tc;
  TcPlan p;
  const int64_t t128 = ceil_div(M, BM) * ceil_div(N, 128);
  p.bn = t128 >= 148 ? 128 : 64;
  const int tiles = (int)(ceil_div(M, BM) * ceil_div(N, p.bn));
  const int nk = (K + BK - 1) / BK;
  const int total = nprods * nk;
  int splits = 1;
  if (tiles < 148) splits = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(2 * 148, tiles), total / 4));
  p.tps = (int)ceil_div(total, splits);
  p.splits = (int)ceil_div(total, p.tps);
  p.partial_bytes = p.splits > 1 ? align256(4 * (size_t)M * N * p.splits) : 0;
  return p;
}

void tc_gemm_products(const Launch& L, const TcPlan& plan, int M, int N, int K, const TcTerms* A, int nA,
                      const TcTerms* B, int nB, const TcProd* prods, int nprods, const GemmArgs<float>& epi,
                      void* partial_ws) {
  using namespace tc;
  SLQ_CHECK_ARG(nA * 3 <= kMaxTerms && nB * 3 <= kMaxTerms && nprods <= kMaxPairs, "tc products: too many terms");
  MultiOps ops;
  for (int i = 0; i < nA; ++i)
    for (int t = 0; t < 3; ++t) ops.a[3 * i + t] = make_map_bf16(A[i].t[t], M, K, A[i].ldk, BM);
  for (int i = 0; i < nB; ++i)
    for (int t = 0; t < 3; ++t) ops.b[3 * i + t] = make_map_bf16(B[i].t[t], N, K, B[i].ldk, plan.bn);
  ops.npairs = nprods;
  for (int i = 0; i < nprods; ++i) {
    ops.ai[i] = 3 * prods[i].ia + prods[i].ta;
    ops.bi[i] = 3 * prods[i].ib + prods[i].tb;
  }
  GemmArgs<float> a = epi;
  a.M = M;
  a.N = N;
  a.K = K;
  a.batch = 1;
  const int nk = (K + BK - 1) / BK;
  float* ws = plan.splits > 1 ? (float*)partial_ws : nullptr;
  {
    LaunchScope scope(L.prof, KC_GEMM, L.stream, 2.0 * M * N * (double)K * nprods,
                      2.0 * ((double)M * K * nA * 3 + (double)N * K * nB * 3) + 4.0 * M * N);
    if (plan.bn == 128)
      launch_multi<128>(L, ops, a, nk, plan.splits, plan.tps, ws);
    else
      launch_multi<64>(L, ops, a, nk, plan.splits, plan.tps, ws);
    ++*L.launches;
  }
  if (plan.splits > 1) {
    LaunchScope scope(L.prof, KC_GEMM, L.stream, 0, 4.0 * (double)M * N * (plan.splits + 1));
    const int64_t mn = (int64_t)M * N;
    int blocks = (int)std::min<int64_t>(ceil_div(mn, 256), 148 * 8);
    gemm_detail::splitk_reduce<float><<<blocks, 256, 0, L.stream>>>(a, plan.splits, ws);
    SLQ_CUDA(cudaGetLastError());
    ++*L.launches;
  }
}

namespace tc {

__global__ void k_fill_bf16(__nv_bfloat16* x, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    x[i] = __float2bfloat16((float)((z >> 40) & 0xFFFF) / 65536.0f - 0.5f);
  }
}

// reference: one thread per output, fp32 accumulation of the same bf16 products
__global__ void k_ref_gemm(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int M, int N, int K) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)M * N) return;
  const int m = (int)(i / N), n = (int)(i % N);
  double s = 0;
  for (int k = 0; k < K; ++k) s += (double)__bfloat162float(A[(int64_t)m * K + k]) * __bfloat162float(B[(int64_t)n * K + k]);
  C[i] = (float)s;
}

}  // namespace tc
}  // namespace slq

// Diagnostic (not yet on the pass path): time the tcgen05 bf16 GEMM on one shape and check it
// against a naive reference kernel.  variant: 0 = 128x128x64 4 stages, 1 = 128x256x64 3 stages.
extern "C" slq_status slq_diag_gemm_bf16(int32_t device, int32_t M, int32_t N, int32_t K, int32_t variant,
                                         int32_t iters, double* tflops, double* max_rel_err) {
  using namespace slq;
  __nv_bfloat16 *A = nullptr, *B = nullptr;
  float *C = nullptr, *R = nullptr;
  try {
    SLQ_CUDA(cudaSetDevice(device));
    SLQ_CUDA(cudaMalloc(&A, 2 * (size_t)M * K));
    SLQ_CUDA(cudaMalloc(&B, 2 * (size_t)N * K));
    SLQ_CUDA(cudaMalloc(&C, 4 * (size_t)M * N));
    SLQ_CUDA(cudaMalloc(&R, 4 * (size_t)M * N));
    tc::k_fill_bf16<<<1024, 256>>>(A, (int64_t)M * K, 11);
    tc::k_fill_bf16<<<1024, 256>>>(B, (int64_t)N * K, 12);
    auto run = [&] {
      if (variant == 1)
        tc::launch<256, 3>(0, A, K, B, K, C, N, M, N, K);
      else
        tc::launch<128, 4>(0, A, K, B, K, C, N, M, N, K);
    };
    run();
    SLQ_CUDA(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    SLQ_CUDA(cudaEventCreate(&e0));
    SLQ_CUDA(cudaEventCreate(&e1));
    SLQ_CUDA(cudaEventRecord(e0));
    for (int i = 0; i < iters; ++i) run();
    SLQ_CUDA(cudaEventRecord(e1));
    SLQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    SLQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *tflops = 2.0 * M * N * (double)K * iters / (ms * 1e-3) / 1e12;
    tc::k_ref_gemm<<<(unsigned)ceil_div((int64_t)M * N, 256), 256>>>(A, B, R, M, N, K);
    SLQ_CUDA(cudaDeviceSynchronize());
    std::vector<float> hc((size_t)M * N), hr((size_t)M * N);
    SLQ_CUDA(cudaMemcpy(hc.data(), C, 4 * hc.size(), cudaMemcpyDeviceToHost));
    SLQ_CUDA(cudaMemcpy(hr.data(), R, 4 * hr.size(), cudaMemcpyDeviceToHost));
    double mx = 0, scale = 1e-30;
    for (size_t i = 0; i < hc.size(); ++i) {
      mx = std::max(mx, (double)std::fabs(hc[i] - hr[i]));
      scale = std::max(scale, (double)std::fabs(hr[i]));
    }
    *max_rel_err = mx / scale;
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(R);
    return SLQ_OK;
  } catch (const Error& e) {
    if (A) cudaFree(A);
    if (B) cudaFree(B);
    if (C) cudaFree(C);
    if (R) cudaFree(R);
    return e.status;
  }
}
