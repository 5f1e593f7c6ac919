/* slq.h -- C-ABI of the B200-native SLQ / FD-HVP library (libslq.so).
 *
 * The one hot path of arXiv 2602.00816 ("Hessian Spectral Analysis at Foundation Model Scale"):
 * stochastic Lanczos quadrature driven by shard-local central finite-difference Hessian-vector
 * products, with theta and every P-vector partitioned FSDP-style.  Citations are PAPER.md line
 * numbers (P:n) with their section / equation / algorithm; S:n are SPEC.md lines.
 *
 * Conventions (all entry points)
 *   - Every call returns slq_status; SLQ_OK == 0.  On error, slq_last_error(ctx) (or
 *     slq_last_error(NULL) for calls without a context) returns a NUL-terminated message that
 *     stays valid until the next call on the same context/thread.
 *   - "collective" calls must be made by every rank of the world, in the same order, with the
 *     same scalar arguments.  With world_size == 1 no communicator is created.
 *   - Shard pointers (v_shard, out_shard, g_shard) hold P_loc = slq_local_len(ctx) fp32 values in
 *     the library's FSDP layout (below).  They may be DEVICE pointers on the context's device
 *     (zero-copy, stream-ordered) or HOST pointers (copied in/out inside the call).  The caller
 *     owns them; the library never retains a caller pointer after the call returns.
 *   - Calls are synchronous on return (the library's stream is synchronised before returning).
 *   - A context is bound to one process/GPU and is not thread-safe.
 *
 * FSDP layout ("perturbations ... applied to each rank's local DTensor shard";
 * SURVEY.md §8(a) A0, §8(e)).  Parameters are in canonical order (layer-major; see DESIGN.md
 * "Canonical parameter order").  They are grouped into FSDP units: MLP = 1 unit; GPT/Llama =
 * [embedding], [block 0] ... [block L-1], [final norm (+ head)].  Unit u has numel_u real
 * parameters, padded to padded_u = roundup(numel_u, 16*world_size); rank r owns the chunk
 * [r*chunk_u, (r+1)*chunk_u) with chunk_u = padded_u / world_size.  The local shard is the
 * concatenation of the rank's chunks of all units, P_loc = sum_u chunk_u.  Padding entries are
 * zero on input and are returned as zero.  No full-length vector is ever gathered
 * (P:112).
 */
#ifndef SLQ_H_
#define SLQ_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct slq_ctx slq_ctx; /* opaque; one per process/GPU */

typedef enum {
  SLQ_OK = 0,
  SLQ_EINVAL = 2,       /* bad descriptor / shape / layout / argument (SPEC exit code 2) */
  SLQ_ENUMERIC = 3,     /* non-finite loss or gradient; see slq_lanczos_info */
  SLQ_ECUDA = 4,        /* CUDA runtime error, or the CUDA kernels are unavailable */
  SLQ_ENCCL = 5,        /* NCCL error (including a peer abort) */
  SLQ_ETIMEOUT = 6,     /* collective watchdog expired */
  SLQ_ENOMEM = 7,       /* device allocation failed */
  SLQ_EUNSUPPORTED = 8  /* valid request this build does not implement */
} slq_status;

enum { SLQ_ARCH_MLP = 0, SLQ_ARCH_GPT = 1, SLQ_ARCH_LLAMA = 2 };
/* arithmetic of the two gradient passes.  FP64: fp64 activations/accumulation on the GPU, GEMMs
 * on the FP64 tensor core (the parity mode of the fp32 models); FP32: fp32
 * passes on SIMT GEMMs (reported only); BF16X3: fp32 activations, every non-batched GEMM on the
 * tcgen05 tensor cores with operands split into three bf16 terms (fp32-faithful; the mode for the
 * bf16 models' gates). */
enum { SLQ_PASS_FP64 = 0, SLQ_PASS_FP32 = 1, SLQ_PASS_BF16X3 = 2, SLQ_PASS_PAIRED = 3, SLQ_PASS_PAIRED_FP32 = 4,
       SLQ_PASS_FP64_OZ = 5, SLQ_PASS_BF16 = 6 };
/* SLQ_PASS_BF16: "BF16 native" (SURVEY.md §8(a) numerics modes; the paper's own bf16 runs,
 * P:602): fp32 activations, every non-batched GEMM on tcgen05 with operands rounded once to bf16
 * (one product, fp32 accumulation).  The throughput mode of the bf16 models; its FD-HVP carries
 * Theorem 1's bf16 round-off floor and does not meet the parity gates. */
/* SLQ_PASS_FP64_OZ: as FP64 (fp64 activations and nonlinearities), but every dense non-batched
 * GEMM with M N K >= oz_min_mnk runs on the tcgen05 INT8 tensor cores as exact digit products
 * (Ozaki scheme: each operand row/column scaled by a power of two and cut into S signed 7-bit
 * digit planes, S = oz_slices; the S(S+1)/2 leading products accumulate exactly in INT32 TMEM;
 * error <~ (S + 2) 2^-7S K max|a| max|b|).  The batched causal attention GEMMs and the smaller
 * dense GEMMs stay on the FP64 DMMA path.  Non-finite operand rows / columns give NaN outputs. */
/* SLQ_PASS_PAIRED: the two gradient evaluations of Eq. (1) carried as (mean, half-difference)
 * pairs through ONE pass, so (g+ - g-) is never formed by subtracting rounded gradients
 * (SURVEY.md §8(f1)); non-batched pair GEMMs on tcgen05 (fp32-faithful three-term bf16 splits),
 * nonlinear steps evaluated at both points in fp64.  SLQ_PASS_PAIRED_FP32: same with fp32 SIMT
 * GEMMs.  GPT and Llama archs, any world size (FSDP: the mean and the half-difference are gathered
 * and reduce-scattered as two streams of per-unit collectives). */
/* Lanczos reorthogonalisation: NONE = three-term recurrence with three
 * rotating vectors and no stored basis; FULL = CGS2 against every stored vector; WINDOW = CGS2
 * against the reorth_window most recent vectors q_{k-r+1} .. q_k (ring buffer of r rows;
 * DESIGN.md reading R17). */
enum { SLQ_REORTH_NONE = 0, SLQ_REORTH_FULL = 1, SLQ_REORTH_WINDOW = 2 };
/* Storage of the Lanczos basis: FP32, or BF16 (each q_{k+1} rounded once,
 * RNE, from fp64 w / beta_{k+1}; every later use reads the stored value; R19).  Scalars
 * are fp64 either way.  BF16 needs reorth FULL or WINDOW. */
enum { SLQ_BASIS_FP32 = 0, SLQ_BASIS_BF16 = 1 };
enum { SLQ_PARAM_FP32 = 0, SLQ_PARAM_BF16 = 1 };

/* Model + numerics description.  Fields unused by an arch are ignored (set them to 0). */
typedef struct {
  int32_t arch;            /* SLQ_ARCH_* */
  int32_t n_layers, d_model, n_heads, n_kv_heads, d_ff, vocab, seq_len; /* GPT / Llama */
  int32_t d_in, d_hidden, n_classes;                                    /* MLP */
  int32_t tie_embeddings;  /* 1: output head reuses the token embedding (GPT-2 style) */
  double rope_theta;       /* Llama RoPE base */
  double norm_eps;         /* LayerNorm / RMSNorm epsilon */
  int32_t param_dtype;     /* SLQ_PARAM_*: storage dtype of theta (bf16 values are held in fp32) */
  int32_t pass_numerics;   /* SLQ_PASS_* */
  int32_t reorth;          /* SLQ_REORTH_*: Lanczos reorthogonalisation */
  int32_t max_steps;       /* largest m slq_lanczos will be asked for (sizes the Krylov basis) */
  double eps_default;      /* FD step used by slq_lanczos (the north-star signature has no eps) */
  int32_t perturb;         /* SLQ_PERTURB_*: how theta +- eta v is formed (reading R9) */
  int32_t reorth_window;   /* r for SLQ_REORTH_WINDOW (2 <= r); ignored otherwise */
  int32_t basis_dtype;     /* SLQ_BASIS_* */
  /* SLQ_PASS_FP64_OZ only: dense GEMMs with M*N*K below oz_min_mnk stay on the FP64 DMMA pipe, the
   * rest run as int8 digit products.  0 = library default (1e9, the measured break-even on B200);
   * 1 puts every dense GEMM on the int8 path.  Per context (no process-global state). */
  double oz_min_mnk;
  int32_t oz_slices;       /* SLQ_PASS_FP64_OZ digit planes S (4..7); 0 = default: 7 for fp32 models (param_dtype
                            * FP32; S < 7 misses their fp32 alpha / beta gate), for bf16 models (their bf16
                            * gates) 5 when eps_default >= 5e-4, else 6 (R27) */
  /* 1: activation checkpointing (BASELINE configs[4]): each transformer block keeps only its input
   * residual stream from the forward and recomputes its forward inside its backward (bit-identical
   * gradients, +1 block forward per block, block activations for 2 blocks instead of n_layers) */
  int32_t act_ckpt;
} slq_model_desc;

/* SLQ_PERTURB_EXACT: theta +- eta*v is evaluated in the pass precision (fp64 passes: an fp64
 *   product and an fp64 sum, divisor 2*eta in fp64), so the perturbed point carries no
 *   storage-rounding error.  Default.
 * SLQ_PERTURB_STORAGE: Alg. 1's in-storage perturbation done out of place:
 *   fmaf(+-fl32(eta), v, theta) rounded once to fp32, divisor 2*fl32(eta).
 * With fp32 passes both modes form fp32 points (STORAGE semantics). */
enum { SLQ_PERTURB_EXACT = 0, SLQ_PERTURB_STORAGE = 1 };

/* This rank's slice of the data (Alg. 1 "dataloader").  The loss is the mean token
 * cross-entropy over the GLOBAL batch (sum of w_b = 1), so every rank passes the global
 * count.  The library copies what it needs; pointers are host memory, not retained. */
typedef struct {
  const float* params_host;  /* FULL canonical-order theta_0, fp32, P values (every rank) */
  const int32_t* tokens;     /* GPT/Llama: [n_seq_local][seq_len + 1] token ids */
  int32_t n_seq_local, n_seq_global;
  const float* x;            /* MLP: [n_rows_local][d_in] inputs */
  const int32_t* y;          /* MLP: [n_rows_local] labels */
  int32_t n_rows_local, n_rows_global;
} slq_batch;

/* Communication backend of a world_size > 1 context.  NCCL: the product path (one process per GPU).
 * LOOPBACK: TEST ONLY -- world_size ranks as contexts of ONE process on one GPU, driven by one
 * host thread each; every collective is host-synchronous (stream sync, host barrier, device
 * copies / a fixed rank-order sum), so no kernel ever waits on another rank's kernel.  It runs
 * the FSDP engine (per-unit all-gather / reduce-scatter, ping-pong buffers, prefetch, scalar
 * all-reduces) at world_size > 1 without a second GPU; CUDA graphs are off in this mode.  The
 * ranks of one group pass the same 128-byte key in nccl_unique_id. */
enum { SLQ_COMM_NCCL = 0, SLQ_COMM_LOOPBACK = 1 };

typedef struct {
  int32_t rank, world_size, device;
  const void* nccl_unique_id; /* 128 bytes from slq_nccl_unique_id() on rank 0, broadcast by the
                                 caller (LOOPBACK: the group key); ignored when world_size == 1 */
  void* cuda_stream;          /* cudaStream_t to run on, or NULL for a library-owned stream.  A
                                 library-owned stream orders every call after the work already
                                 queued on the legacy default stream (where a caller's device
                                 pointers are typically written); with a caller stream, ordering
                                 is the caller's */
  int32_t comm_backend;       /* SLQ_COMM_* (world_size > 1) */
} slq_world;

/* Create a context: validate, plan the FSDP layout ("perturbations ... applied to each
 * rank's local DTensor shard"), create the NCCL communicators (world > 1: one
 * for the scalar all-reduces and one per concurrent gradient pass, split from it), check the
 * device memory plan (slq_plan_memory) against the free memory (SLQ_ENOMEM with the plan in the
 * message when it does not fit), allocate device state, upload this rank's chunks of theta_0 and
 * its data slice (Alg. 1 "dataloader").  Every pointer in desc / batch / world is read
 * during the call only.  Collective. */
slq_status slq_init(const slq_model_desc* desc, const slq_batch* batch, const slq_world* world,
                    slq_ctx** out);
slq_status slq_destroy(slq_ctx* ctx);
const char* slq_last_error(const slq_ctx* ctx);

int64_t slq_local_len(const slq_ctx* ctx);   /* P_loc (padded, this rank) */
int64_t slq_global_len(const slq_ctx* ctx);  /* P (real parameters) */
int32_t slq_num_units(const slq_ctx* ctx);
/* unit u: global canonical offset, real numel, this rank's local offset and chunk length */
slq_status slq_unit_info(const slq_ctx* ctx, int32_t u, int64_t* global_offset, int64_t* numel,
                         int64_t* local_offset, int64_t* chunk);

/* Host-only layout planner (no GPU, no context): the same plan slq_init makes.  unit_table gets
 * 4 int64 per unit {global_offset, numel, local_offset, chunk}; pass NULL to query n_units. */
slq_status slq_plan_layout(const slq_model_desc* desc, int32_t world_size, int64_t* P,
                           int64_t* P_loc, int32_t* n_units, int64_t* unit_table);

/* Host-only device-memory plan (no GPU, no context) of one rank: the bytes slq_init would allocate
 * for desc at world_size ranks with n_local sequences (MLP: rows) on this rank.  bytes[SLQ_MEM_COUNT]
 * gets one entry per category below (SLQ_MEM_TOTAL = their sum).  Activations, logits, backward
 * scratch and FSDP buffers are per gradient-pass executor (two run concurrently unless the paired
 * mode is used); GEMM workspace is the largest Ozaki / split-K scratch of one pass (estimate). */
enum { SLQ_MEM_THETA = 0, SLQ_MEM_POINTS, SLQ_MEM_GRADS, SLQ_MEM_LANCZOS, SLQ_MEM_FSDP, SLQ_MEM_ACTIVATIONS,
       SLQ_MEM_LOGITS, SLQ_MEM_SCRATCH, SLQ_MEM_WORKSPACE, SLQ_MEM_TOTAL, SLQ_MEM_COUNT };
slq_status slq_plan_memory(const slq_model_desc* desc, int32_t world_size, int32_t n_local, int64_t* bytes);

/* 128-byte NCCL unique id for slq_world.nccl_unique_id (call on rank 0 only). */
slq_status slq_nccl_unique_id(void* out128);

/* Hv for a caller direction: out = ||v|| (grad L(theta + eps vhat) - grad L(theta - eps vhat))/(2 eps)
 * (Eq. (1); Alg. 1).  Implemented as a step eta = eps/||v|| along v with
 * theta+- formed out of place (theta is never written, so it is bit-identical afterwards),
 * two gradient passes, out = (g+ - g-)/(2 eta).  How theta+- is formed follows desc.perturb
 * (reading R9): SLQ_PERTURB_EXACT (default) with fp64 passes forms theta +- eta v in
 * fp64 (rounded product, rounded sum) with an fp64 divisor 2 eta; SLQ_PERTURB_STORAGE, and every
 * fp32 pass mode, forms fmaf(+-fl32(eta), v, theta) rounded once to fp32 with divisor
 * 2 fl32(eta).  ||v|| costs the one scalar all-reduce P:197 allows.  v == 0 returns 0.
 * v_shard / out_shard: P_loc fp32 each, device or host, must not alias.  SLQ_ENUMERIC on a
 * non-finite v or gradient (slq_nonfinite_seq names the sequence).  Collective. */
slq_status slq_hvp(slq_ctx* ctx, const float* v_shard, float* out_shard, double eps);

/* One gradient evaluation = the paper's T_grad (one forward + one backward with all
 * FSDP collectives, no optimiser).  g_shard may be NULL (timing); loss may be NULL.  Collective. */
slq_status slq_grad(slq_ctx* ctx, float* g_shard, double* loss);

/* m steps of Lanczos (App. C) on the FD-HVP operator with step
 * eps_default, from the Rademacher probe q_1[i] = s(probe_seed, gid(i))/sqrt(P) (integer
 * splitmix64 hash).  alpha[m] and beta[m-1] (= beta_2..beta_m) are host
 * arrays.  Breakdown (beta_{k+1} <= tol * max|T|) returns SLQ_OK with the unfilled entries NaN;
 * see slq_lanczos_info.  Collective. */
slq_status slq_lanczos(slq_ctx* ctx, uint64_t probe_seed, int32_t m, double* alpha, double* beta);
slq_status slq_lanczos_info(const slq_ctx* ctx, int32_t* m_done, double* beta_next,
                            int32_t* nonfinite);
/* The same recurrence in segments (slq_lanczos == start + step(m) + result, bit for bit): start
 * draws q_1 for probe_seed and fixes m (<= max_steps); step runs n_steps more steps (the total
 * must stay <= m); result copies alpha[m] / beta[m - 1] (host; entries not reached yet are NaN,
 * and so is the last beta of an unfinished probe), ends the probe and sets slq_lanczos_info.
 * Between calls the probe's state (basis rows or the three vectors, recurrence scalars) stays on
 * the device; any other call on the context except slq_lanczos_info / host-only calls ends the
 * probe's validity.  Used to time steps k0 .. k0 + K of a long probe (bench.py) and to monitor
 * Ritz-value convergence.  All three are collective. */
slq_status slq_lanczos_start(slq_ctx* ctx, uint64_t probe_seed, int32_t m);
slq_status slq_lanczos_step(slq_ctx* ctx, int32_t n_steps);
slq_status slq_lanczos_result(slq_ctx* ctx, double* alpha, double* beta);
/* After slq_hvp returned SLQ_ENUMERIC (non-finite gradient, "error carrying the offending
 * batch id"): *seq = local index of the first sequence (MLP: data row) whose loss was non-finite
 * in the theta+ or theta- pass, or -1 when every loss was finite (overflow inside the backward
 * only).  -1 after a successful slq_hvp.  Host-only, no device work. */
slq_status slq_nonfinite_seq(const slq_ctx* ctx, int32_t* seq);
/* Stochastic Lanczos quadrature's probe loop ("T_SLQ ~ s m T_Lanczos iter"):
 * slq_lanczos for each of the n_probes seeds; alpha [n_probes][m], beta [n_probes][m - 1] (host),
 * m_done [n_probes] (may be NULL).  Feed each probe's (alpha, beta) to slq_quadrature and the node
 * sets to slq_density for the probe average.  Collective. */
slq_status slq_slq(slq_ctx* ctx, const uint64_t* seeds, int32_t n_probes, int32_t m, double* alpha, double* beta,
                   int32_t* m_done);

/* Gauss quadrature of T_m (host only, no context, pure): nodes ascending (Ritz values) and
 * weights = squared first components of the normalised eigenvectors (sum 1).
 * beta may be NULL when m == 1.  Implicit-shift QL (Golub-Welsch). */
slq_status slq_quadrature(const double* alpha, const double* beta, int32_t m, double* nodes,
                          double* weights);

/* SLQ probe average (host only, no context, pure): n_probes node/weight sets
 * of m_p = m_counts[p] nodes each, packed back to back in nodes[] / weights[] (sum of m_counts).
 * moments (may be NULL): [jmax + 1] probe-averaged e_1^T T^j e_1 = (1/s) sum_p sum_i w_i theta_i^j;
 * density (may be NULL): Gaussian-smoothed spectral density (1/s) sum_p sum_i w_i N(x_g; theta_i,
 * sigma^2) at the n_grid points grid[] (sigma > 0).  SLQ_EINVAL on bad sizes / sigma. */
slq_status slq_density(const double* nodes, const double* weights, const int32_t* m_counts, int32_t n_probes,
                       int32_t jmax, double* moments, const double* grid, int32_t n_grid, double sigma,
                       double* density);

/* Ghost diagnostic (host only, no context, pure; Theorem 3 "spurious duplicate
 * eigenvalues"; R18): single-linkage clusters of ascending Ritz values `nodes[m]`,
 * neighbours joined when nodes[i+1] - nodes[i] <= tol.  cluster_id[m] (may be NULL) gets each
 * node's cluster index (0-based, ascending); *n_ghost = number of clusters with >= 2 members;
 * *max_split = the largest max - min over those clusters (0 if none).  SLQ_EINVAL if nodes are
 * not ascending / finite or tol < 0. */
slq_status slq_ghost_clusters(const double* nodes, int32_t m, double tol, int32_t* cluster_id, int32_t* n_ghost,
                              double* max_split);

/* Conjugate-gradient inverse-HVP ("repeated HVP calls plus
 * scalar reductions and shard-local vector operations"): solves (H + damping I) x = b with x_0 = 0,
 * each H p one FD-HVP with step eps_default (same normalisation as slq_hvp), until
 * ||r|| <= tol ||b|| or max_iter.  H is indefinite: damping must make H + damping I positive
 * definite (SLQ_ENUMERIC if p^T (H + damping I) p <= 0).  b, x: shards, device or host.  Collective. */
slq_status slq_cg(slq_ctx* ctx, const float* b_shard, float* x_shard, double damping, int32_t max_iter, double tol,
                  int32_t* iters, double* rel_residual);

/* Block-diagonal hypothesis test: v = the Rademacher probe of probe_seed
 * (unit norm), h = H v; for each FSDP unit b (embedding, transformer blocks, final norm + head):
 * h_b = H v^(b) with v zeroed outside b; rel_err[b] = ||h|_b - h_b|_b|| / ||h|_b||,
 * cosine[b] = cos(h|_b, h_b|_b).  rel_err / cosine: host arrays of slq_num_units.  Costs
 * 1 + n_units HVPs.  Collective. */
slq_status slq_blockdiag(slq_ctx* ctx, uint64_t probe_seed, double* rel_err, double* cosine);

/* Writes the Lanczos start vector q_1 (probe) for probe_seed into a caller shard (device or host).
 * Exposed so the probe can be checked bit-exactly against an independent generator. */
slq_status slq_probe(slq_ctx* ctx, uint64_t probe_seed, float* q_shard);

/* Per-kernel-class timing with CUDA events recorded on the launching stream around every launch
 * (off by default; launches run eagerly, not from CUDA graphs, while it is on).  enable = 1:
 * serial mode (both gradient passes and their side work on one stream, so each launch's duration
 * is its own); enable = 2: overlap-aware mode (the normal concurrency is kept; slq_kernel_busy
 * gives each class's busy time = the union of its launch intervals on the device timeline);
 * 0 = off.  classes: see slq_kernel_class_name.  Stats accumulate until reset. */
slq_status slq_profile(slq_ctx* ctx, int32_t enable, int32_t reset);
int32_t slq_num_kernel_classes(void);
const char* slq_kernel_class_name(int32_t cls);
slq_status slq_kernel_stats(const slq_ctx* ctx, int32_t cls, double* total_ms, int64_t* launches,
                            double* flops, double* bytes);
/* busy time (ms) of class cls since the last reset: the length of the union of its launches'
 * [start, end] intervals; cls = -1: of all classes together (device busy time) */
slq_status slq_kernel_busy(const slq_ctx* ctx, int32_t cls, double* busy_ms);
/* NCCL collectives issued since the context was created (collective audit):
 * all-gathers, reduce-scatters, all-reduces.  All zero when world_size == 1. */
slq_status slq_collective_counts(const slq_ctx* ctx, int64_t* allgather, int64_t* reduce_scatter,
                                 int64_t* allreduce);
/* total kernel launches issued by the library since the context was created */
int64_t slq_launch_count(const slq_ctx* ctx);
void* slq_stream(const slq_ctx* ctx);

/* Diagnostic of the collective watchdog: enqueue a kernel that stalls the
 * context's stream for `stall_ms` (0..10000) milliseconds, then wait for the stream the way every
 * collective call does, with `timeout_s` (<= 0: no timeout).  Returns SLQ_ETIMEOUT when the stall
 * outlasts the timeout -- the context's NCCL communicator (if any) is then aborted and every later
 * collective call returns SLQ_ENCCL -- else SLQ_OK.  Collective calls use the timeout from the
 * environment variable SLQ_TIMEOUT_S (default 1800 s, 0 = none) and also return SLQ_ENCCL on an
 * asynchronous NCCL error (e.g. a failed peer), after aborting the communicator. */
slq_status slq_diag_watchdog(slq_ctx* ctx, int32_t stall_ms, double timeout_s);
/* Diagnostic, not on the hot path: measured FP64 FMA throughput of `device` in TFLOP/s (the
 * roofline denominator of the fp64 gradient-pass GEMMs, which MEASURED_PEAKS.json lacks). */
slq_status slq_diag_fp64_peak(int32_t device, double* tflops);
/* Diagnostic: the int8 Ozaki fp64 GEMM (S digit planes) against the DMMA fp64 GEMM on random data
 * (ragged shapes allowed): *max_err = max |C_oz - C_dmma| / (K max_k|A_ik| max_k|B_kj|) over all
 * (i, j); *tflops = fp64-equivalent rate of the Ozaki GEMM (2 M N K / time, slicing included). */
slq_status slq_diag_oz_check(int32_t device, int32_t M, int32_t N, int32_t K, int32_t a_kmajor, int32_t b_kmajor,
                             int32_t S, int32_t iters, double* max_err, double* tflops);
/* Diagnostic: causal multi-head attention forward + backward (nseq sequences of Tn tokens, Hq query
 * heads sharing Hkv key/value heads of width hd) on random data through the FP64 DMMA path and
 * through the FP64_OZ path (all six contractions as batched INT8 Ozaki GEMMs with S digit planes,
 * oz_attn.cu).  err[4] = max |x_oz - x_dmma| / max |x_dmma| for O, dQ, dK, dV; ms[2] = time of one
 * forward + backward of each path averaged over `iters` repetitions (0: not timed).  SLQ_EINVAL when
 * the shape is not eligible for the Ozaki path (Tn % 128, hd % 32, hd <= 128). */
slq_status slq_diag_attn_oz(int32_t device, int32_t nseq, int32_t Tn, int32_t Hq, int32_t Hkv, int32_t hd, int32_t S,
                            int32_t iters, double* err, double* ms);
/* Diagnostic: measured FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput in TFLOP/s. */
slq_status slq_diag_dmma_peak(int32_t device, double* tflops);
/* Diagnostic: time the library's fp64 GEMM on one shape.  A [M x K] (K-contiguous if a_kmajor,
 * else M-contiguous), B [K x N] (stored [N x K] if b_kmajor, else [K x N]); variant = tile
 * configuration (-1: production heuristic), splits = split-K factor (0: auto).  Outputs TFLOP/s
 * over `iters` back-to-back launches and a weighted checksum of C (variants must agree). */
slq_status slq_diag_gemm_f64(int32_t device, int32_t M, int32_t N, int32_t K, int32_t a_kmajor, int32_t b_kmajor,
                             int32_t variant, int32_t splits, int32_t iters, double* tflops, double* checksum);

#ifdef __cplusplus
}
#endif
#endif /* SLQ_H_ */
