// The FD-HVP / Lanczos engine behind the C-ABI (one per context).
#pragma once

#include <memory>

#include "comm.h"
#include "kernels.h"
#include "layout.h"
#include "model.h"

namespace slq {

struct LanczosInfo {
  int m_done = 0;
  double beta_next = 0;
  int nonfinite = 0;
};

struct Engine {
  virtual ~Engine() {}
  // v, out: device pointers, P_loc fp32 each
  virtual void hvp(const float* v, float* out, double eps) = 0;
  virtual double grad(float* g) = 0;  // returns the global mean loss
  virtual LanczosInfo lanczos(uint64_t seed, int m, double* alpha, double* beta) = 0;
  // resumable form of lanczos(): start a probe of up to m steps, advance it, read it out
  virtual void start(uint64_t seed, int m) = 0;
  virtual void step(int nsteps) = 0;
  virtual LanczosInfo result(double* alpha, double* beta) = 0;
  virtual void probe(uint64_t seed, float* q) = 0;
  virtual double pass_flops() const = 0;  // algorithmic FLOPs of one fwd+bwd (this rank)
  // CG on (H + damping I) x = b; returns iterations, writes the relative residual
  virtual int cg(const float* b, float* x, double damping, int max_iter, double tol, double* relres) = 0;
  // block-diagonal test over the FSDP units: rel_err[u], cosine[u]
  virtual void blockdiag(uint64_t seed, double* rel_err, double* cosine) = 0;
  LanczosInfo last_info;
  // set by a failing hvp (SLQ_ENUMERIC): local index of the first sequence (MLP: row) with a
  // non-finite loss in the two passes, -1 if the losses were finite (S:114's "offending batch id")
  int nonfinite_seq = -1;
};

// slq_plan_memory: the per-rank device bytes by category (slq.h SLQ_MEM_*)
void plan_memory(const slq_model_desc& d, int world, int n_local, int64_t* out);

std::unique_ptr<Engine> make_engine(const slq_model_desc& d, const LayoutPlan& plan, const HostBatch& b,
                                    const float* theta_host_full, int rank, Comm* comm, const Launch& L);

}  // namespace slq
