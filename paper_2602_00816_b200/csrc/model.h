// Gradient-pass runners: one forward + one backward of the dataset-mean loss over this rank's
// data slice (Alg. 1 lines 5-8 / 10-13), unit by unit through a PassIO that hides the
// FSDP collectives (per-unit all-gather before forward and again before backward; per-unit
// reduce-scatter of the gradient after backward).
#pragma once

#include <memory>
#include <vector>

#include "kernels.h"
#include "layout.h"

namespace slq {

template <class T>
struct PassIO {
  virtual ~PassIO() {}
  // full (padded) parameters of unit u in the pass dtype; valid until params() is called for a
  // unit that maps to the same slot (unit 0 has its own slot, so it may stay live with any other)
  virtual const T* params(int u) = 0;
  // buffer receiving the full gradient of unit u (kernels overwrite real entries; unit 0's
  // buffer persists from the first grads(0) call to grads_done(0))
  virtual T* grads(int u) = 0;
  virtual void grads_done(int u) = 0;
  // true when grads_done() starts a collective on the unit's gradient (FSDP reduce-scatter): the
  // runner must then finish the unit's side-stream gradient work first
  virtual bool collective() const { return false; }
  // hint: unit u's parameters will be requested next (FSDP: start its all-gather now, overlapped
  // with the compute of the current unit)
  virtual void prefetch(int) {}
};

struct HostBatch {
  std::vector<int32_t> tokens;  // [n_seq][seq_len + 1]
  int n_seq = 0, n_seq_global = 0;
  std::vector<float> x;  // MLP
  std::vector<int32_t> y;
  int n_rows = 0, n_rows_global = 0;
};

template <class T>
struct Runner {
  virtual ~Runner() {}
  // writes this rank's sum of per-token losses to *loss_sum_dev (device double)
  virtual void fwd_bwd(PassIO<T>& io, double* loss_sum_dev) = 0;
  virtual double tokens_global() const = 0;
  virtual double flops_per_pass() const = 0;  // algorithmic fwd+bwd FLOPs (this rank)
  // paired evaluation (model_paired.cu): mean = (theta, gbar), diff = (eta v, gtil) in one pass
  virtual bool paired() const { return false; }
  // after a failed pass: local index of the first sequence (MLP: row) whose loss in this runner's
  // last pass is non-finite, -1 if every loss was finite (error attribution)
  virtual int first_nonfinite_seq() { return -1; }
  virtual void fwd_bwd_pair(PassIO<T>& mean, PassIO<T>& diff, double* loss_sum) {
    throw Error(SLQ_EUNSUPPORTED, "paired evaluation not available for this runner");
  }
  // device bytes of the runner's own buffers by memory-plan category (0 activations + data, 1 logits,
  // 2 backward scratch) -- exact for a real runner, the plan for a dry one
  virtual size_t arena_bytes(int) const { return 0; }
  // the largest GEMM / reduction workspace its pass asks for on the data-gradient lane (main) and
  // on the side stream (side); reserved up front by real runners
  virtual void plan_ws(size_t& main, size_t& side) const {}
};

// first group of `per` consecutive rows of dev[n] (device doubles) holding a non-finite value,
// -1 if none (synchronous device -> host copy; error paths only)
int first_nonfinite_group(const double* dev, int n, int per, cudaStream_t s);

// dry: allocate nothing, launch nothing -- only count the bytes (slq_plan_memory)
template <class T>
std::unique_ptr<Runner<T>> make_runner(const slq_model_desc& d, const LayoutPlan& plan, const HostBatch& b,
                                       const Launch& L, bool dry = false);
// paired-evaluation runner (GPT); nullptr if the arch has none yet
std::unique_ptr<Runner<float>> make_paired_runner(const slq_model_desc& d, const LayoutPlan& plan,
                                                  const HostBatch& b, const Launch& L);

}  // namespace slq
