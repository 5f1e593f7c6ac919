// Internal helpers shared by the library's translation units (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/slq.h"

namespace slq {

struct Error : std::runtime_error {
  slq_status status;
  Error(slq_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

#define SLQ_CHECK_ARG(cond, msg)                                                  \
  do {                                                                            \
    if (!(cond)) throw ::slq::Error(SLQ_EINVAL, std::string("invalid: ") + (msg)); \
  } while (0)

#define SLQ_CUDA(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw ::slq::Error(e_ == cudaErrorMemoryAllocation ? SLQ_ENOMEM : SLQ_ECUDA,             \
                         std::string(#expr) + ": " + cudaGetErrorString(e_) + " @" __FILE__ ":" + \
                             std::to_string(__LINE__));                                       \
  } while (0)

// kernel classes for the per-class CUDA-event profiler (slq_profile)
enum KernelClass {
  KC_GEMM = 0,     // dense contractions of the gradient passes
  KC_ATTN,         // softmax / attention elementwise
  KC_NORM,         // layernorm / rmsnorm fwd+bwd and column reductions
  KC_CE,           // cross entropy
  KC_EMBED,        // embedding gather / scatter
  KC_ELEM,         // other elementwise (rope, swiglu, convert)
  KC_PERTURB,      // (a) perturb theta +- eta v
  KC_FD,           // (d) FD difference + Lanczos partials
  KC_REORTH,       // (e) reorthogonalisation GEMV
  KC_VEC,          // other vector ops (probe, normalise, reductions)
  KC_GEMM_I8,      // fp64 GEMMs as tcgen05 INT8 digit products (Ozaki); flops = INT8 ops issued
  KC_OZ_SLICE,     // Ozaki operand scaling + digit slicing (HBM / L2 bound)
  KC_ATTN_I8,      // the causal attention contractions as batched INT8 Ozaki GEMMs (oz_attn.cu)
  KC_COUNT
};
const char* kernel_class_name(int c);

// per-context launch bookkeeping (profiler + launch counter); defined in api.cpp
struct Profiler;
bool prof_enabled(const Profiler* p);
bool prof_serial(const Profiler* p);  // profiler on in serial mode: no concurrency
void prof_begin(Profiler* p, int cls, cudaStream_t s);
void prof_end(Profiler* p, int cls, cudaStream_t s, double flops, double bytes);

struct LaunchScope {
  Profiler* p;
  int cls;
  cudaStream_t s;
  double flops, bytes;
  LaunchScope(Profiler* p_, int c, cudaStream_t s_, double f = 0, double b = 0)
      : p(p_), cls(c), s(s_), flops(f), bytes(b) {
    prof_begin(p, cls, s);
  }
  ~LaunchScope() { prof_end(p, cls, s, flops, bytes); }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace slq
