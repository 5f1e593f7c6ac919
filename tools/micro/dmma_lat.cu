// DMMA throughput vs warps per SM and independent accumulators per warp (diagnostic).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
template <int NACC>
__global__ void k(double* out, int iters, double a, double b) {
  double c[2 * NACC];
#pragma unroll
  for (int i = 0; i < 2 * NACC; ++i) c[i] = threadIdx.x * 1e-9 + i;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) dmma884(c[2 * j], c[2 * j + 1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 2 * NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}
template <int NACC>
void run(int warps_per_sm) {
  double* d; cudaMalloc(&d, 8);
  int blocks = 148, threads = 32 * warps_per_sm, iters = 2048 * 8 / NACC;
  k<NACC><<<blocks, threads>>>(d, 16, 0.5, 1e-3);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NACC><<<blocks, threads>>>(d, iters, 0.5, 1e-3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * NACC * iters * (double)blocks * warps_per_sm;
  printf("warps/SM %2d  acc/warp %2d  %.1f TFLOP/s\n", warps_per_sm, NACC, fl / ms / 1e9);
}
int main() {
  for (int w : {1, 2, 4, 8, 16}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); run<16>(w); }
  return 0;
}
