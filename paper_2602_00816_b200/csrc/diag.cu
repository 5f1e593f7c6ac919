// Peak probes used to set the roofline denominators that MEASURED_PEAKS.json does not cover
// (the FP64 pipe the fp64 parity passes run on).  Not on the hot path.
#include <cuda_runtime.h>

#include "common.h"

namespace {

// 8 independent DFMA chains per thread, long enough to amortise launch overhead
__global__ void k_dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1e-9, x2 = x0 + 2e-9, x3 = x0 + 3e-9;
  double x4 = x0 + 4e-9, x5 = x0 + 5e-9, x6 = x0 + 6e-9, x7 = x0 + 7e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 8 independent DMMA accumulators per warp
__global__ void k_dmma_peak(double* out, int iters, double a, double b) {
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x * 1e-9 + i;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma884(c[2 * j], c[2 * j + 1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

// one thread that spins on the global nanosecond timer for `ns` (the watchdog test's stall)
__global__ void k_diag_stall(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

}  // namespace

namespace slq {
void diag_stall(cudaStream_t s, int ms) {
  k_diag_stall<<<1, 1, 0, s>>>((uint64_t)ms * 1000000ull);
  SLQ_CUDA(cudaGetLastError());
}
}  // namespace slq

extern "C" slq_status slq_diag_dmma_peak(int32_t device, double* tflops) {
  try {
    SLQ_CUDA(cudaSetDevice(device));
    int sms = 0;
    SLQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* d = nullptr;
    SLQ_CUDA(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t a, b;
    SLQ_CUDA(cudaEventCreate(&a));
    SLQ_CUDA(cudaEventCreate(&b));
    const int blocks = sms * 4, threads = 256, iters = 4096;
    k_dmma_peak<<<blocks, threads>>>(d, 64, 0.5, 1e-3);
    SLQ_CUDA(cudaEventRecord(a));
    k_dmma_peak<<<blocks, threads>>>(d, iters, 0.5, 1e-3);
    SLQ_CUDA(cudaEventRecord(b));
    SLQ_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    SLQ_CUDA(cudaEventElapsedTime(&ms, a, b));
    const double flops = 512.0 * 8 * (double)iters * blocks * (threads / 32);
    *tflops = flops / (ms * 1e-3) / 1e12;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    return SLQ_OK;
  } catch (const slq::Error& e) {
    return e.status;
  }
}

extern "C" slq_status slq_diag_fp64_peak(int32_t device, double* tflops) {
  try {
    SLQ_CUDA(cudaSetDevice(device));
    int sms = 0;
    SLQ_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double* d = nullptr;
    SLQ_CUDA(cudaMalloc(&d, sizeof(double)));
    cudaEvent_t a, b;
    SLQ_CUDA(cudaEventCreate(&a));
    SLQ_CUDA(cudaEventCreate(&b));
    const int blocks = sms * 8, threads = 256, iters = 2048;
    k_dfma_peak<<<blocks, threads>>>(d, 64, 0.999999, 1e-7);  // warm-up
    SLQ_CUDA(cudaEventRecord(a));
    k_dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    SLQ_CUDA(cudaEventRecord(b));
    SLQ_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    SLQ_CUDA(cudaEventElapsedTime(&ms, a, b));
    const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    *tflops = flops / (ms * 1e-3) / 1e12;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    return SLQ_OK;
  } catch (const slq::Error& e) {
    return e.status;
  }
}
