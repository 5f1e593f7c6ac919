#!/usr/bin/env python
"""Benchmark of the SLQ / FD-HVP hot path (arXiv 2602.00816) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3|c2|...]
                    [--numerics fp64_oz|fp64|bf16x3|bf16|fp32|paired|paired_fp32]
                    [--reorth config|full|none|window [--window r]] [--basis fp32|bf16]

Default workload: BASELINE.json configs[2] ("c3", the configuration the metric is quoted on at
1/2/4/8 GPUs and the largest single-GPU config): GPT-2-small shape, 12 layers, d 768, 12 heads,
MLP 3072, vocab 50257, tied, 124,439,808 bf16-representable params; 8 x 1024 Zipf(1.1) tokens PER
GPU (weak scaling); eps = 1e-3; Lanczos m = 100 with full CGS2 reorthogonalisation; pass numerics
FP64_OZ (fp64 passes; dense GEMMs >= 1e9 M N K as exact int8 digit products on tcgen05 (Ozaki), the
rest on DMMA) -- the fastest mode that meets the parity gates on c3.  `--config c2` gives the small-
GPT line (global batch 8 x 256 split across ranks: strong scaling).

A "step" is one Lanczos iteration = one FD-HVP (perturb + two gradient passes + FD difference) +
the recurrence + CGS2 reorthogonalisation, i.e. every SURVEY §8(a) row.  The K timed steps are
steps k0 .. k0 + K - 1 of ONE probe of the config's m steps (slq_lanczos_start / _step / _result),
with k0 = max(W, (m - K) / 2): the W (or more) steps before them are the untimed warm-up and the
window is centred on step m / 2, so the growing-basis reorthogonalisation costs what it costs on
average over a whole m-step probe.  metric = HVPs/sec, whole job: for the weak-scaling configs one
unit is an HVP over one GPU's batch (value = N / T_step); for c2 one unit is the HVP over the fixed
global batch.  Each rank's CUDA-event time is max-reduced.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import slq_inputs as si  # noqa: E402

UNIT = "HVP/s"
WEAK = {"c3": 8, "c4": 4, "c5": 2}  # sequences per GPU (BASELINE "batch B/GPU")


def metric_name(cfg_name: str) -> str:
    if cfg_name in WEAK:
        return (f"HVPs/sec (FD-HVP Lanczos steps/s x N; unit = an HVP over one GPU's {WEAK[cfg_name]} x "
                f"seq batch; {cfg_name}, full reorth)")
    return f"HVPs/sec (FD-HVP Lanczos steps/s over the global batch; {cfg_name})"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c3")
    p.add_argument("--numerics", default="fp64_oz", choices=["fp64", "fp64_oz", "fp32", "bf16x3", "bf16", "paired", "paired_fp32"],
                   help="gradient-pass arithmetic: fp64_oz (default) = fp64 passes with the large GEMMs as "
                        "exact int8 digit products on tcgen05 (Ozaki) and the rest on DMMA; fp64 = all DMMA; "
                        "bf16x3 = fp32-faithful tcgen05")
    p.add_argument("--oz-slices", type=int, default=0,
                   help="FP64_OZ digit planes S (0: the library default, 5 for bf16 models, 7 for fp32 models)")
    p.add_argument("--act-ckpt", action="store_true", help="activation checkpointing (BASELINE configs[4])")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--probe-m", type=int, default=0,
                   help="length of the probe holding the timed window (default: the config's m); a short probe "
                        "for profiler runs (ncu), whose numbers are never bench values")
    # "report with reorth on and off where the config asks"; window / bf16 basis (f3)
    p.add_argument("--reorth", default="config", choices=["config", "full", "none", "window"])
    p.add_argument("--window", type=int, default=8)
    p.add_argument("--basis", default="fp32", choices=["fp32", "bf16"])
    a = p.parse_args()
    if a.config not in si.CONFIGS or si.CONFIGS[a.config].arch == si.ARCH_MLP:
        p.error(f"--config {a.config}: bench lines are for the transformer configs "
                f"({', '.join(k for k, c in si.CONFIGS.items() if c.arch != si.ARCH_MLP)}); c1 is a parity case")
    return a


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def split_batch(cfg, rank, world):
    """Weak-scaling configs: rank r holds sequences [r B, (r + 1) B) of the data stream (B per GPU);
    otherwise the config's global batch is split across ranks."""
    if cfg.name in WEAK:
        b = WEAK[cfg.name]
        return si.tokens(cfg, n_seq=b, first_seq=rank * b), b * world
    tok = si.tokens(cfg)
    n = tok.shape[0]
    return tok[si.rank_slice(n, rank, world)], n


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [l.split(",") for l in open(self.f.name).read().strip().splitlines() if l.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) >= 9:
                for nm, val in zip(names, r[5:9]):
                    if "Active" in val and "Not" not in val:
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_traffic(kernel_class: str):
    """Per-launch DRAM bytes of the dominant kernel class from the committed ncu summary."""
    try:
        s = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return s.get(kernel_class)
    except Exception:
        return None


def oracle_sample(cfg):
    """(tokens, scale): the oracle's bounded sample of one HVP unit and the linear-in-tokens factor
    that converts sample HVPs/s into unit HVPs/s.  c2: the full global batch (factor 1: a smaller
    batch is not proportionally cheaper for the numpy oracle, ~4 s per step at 2 of 8 sequences vs
    5.2 s at 8, so a token-scaled sample would understate it); weak-scaling configs: 1 sequence
    truncated to 32 tokens of the per-GPU unit."""
    if cfg.name in WEAK:
        t = 32
        tok = si.tokens(cfg, n_seq=1)[:, :t + 1]
        return tok, t / float(WEAK[cfg.name] * cfg.seq_len)
    return si.tokens(cfg), 1.0


def default_oz_slices(cfg) -> int:
    """the library's default FP64_OZ digit planes (slq.h oz_slices; R27)"""
    return (5 if cfg.eps >= 5e-4 else 6) if cfg.param_bf16 else 7


def host_cpu() -> str:
    try:
        for l in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if l.startswith("Model name:"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(cfg, budget_s=12.0):
    """The oracle, as it stands, timed on this host: exact-mode FD-HVPs on a bounded sample."""
    from oracle import fdhvp, probe
    th = si.init_params(cfg)
    tok, scale = oracle_sample(cfg)
    g = fdhvp.make_grad_fn(cfg, tok)
    q = probe.rademacher_probe(cfg.probe_seed0, th.size)
    n = 0
    t0 = time.perf_counter()
    while True:
        fdhvp.fd_hvp_step(g, th, q, cfg.eps, "exact")
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    what = (f"{n} oracle FD-HVPs (fp64 numpy, 2 gradient passes each) on {tok.shape[0]} x {tok.shape[1] - 1} "
            f"tokens, {dt:.1f} s")
    if scale != 1.0:
        what += f"; scaled to the {cfg.name} unit by linear-in-tokens extrapolation (x {scale:.4g})"
    return {"value": n / dt * scale, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "cpu": host_cpu(),
            "sample": what + "; the recurrence/reorth is <1% and excluded"}


def reorth_of(args, cfg):
    return ("full" if cfg.reorth_full else "none") if args.reorth == "config" else args.reorth


def reorth_label(args, cfg):
    r = reorth_of(args, cfg)
    lab = {"full": "full CGS2 reorth", "none": "no reorth", "window": f"window-{args.window} CGS2 reorth"}[r]
    return lab + (", bf16 basis" if args.basis == "bf16" and r != "none" else "")


def config_dict(args, cfg, world, n_glob):
    """The bench line's `config` (both arms print the same one)."""
    arch = {si.ARCH_GPT: "GPT", si.ARCH_LLAMA: "Llama"}.get(cfg.arch, "MLP")
    return {"workload": f"{args.config}: {arch} {cfg.n_layers}L "
                        f"d{cfg.d_model} {cfg.n_heads}h ff{cfg.d_ff} V{cfg.vocab}, {si.n_params(cfg)} params "
                        f"({'bf16' if cfg.param_bf16 else 'fp32'}), "
                        + (f"{WEAK[cfg.name]}x{cfg.seq_len} Zipf(1.1) tokens per GPU" if cfg.name in WEAK
                           else f"{cfg.n_seq}x{cfg.seq_len} Zipf(1.1) tokens in total")
                        + f", eps={cfg.eps}, Lanczos m={cfg.m} {reorth_label(args, cfg)}",
            "global_batch": n_glob, "seq_len": cfg.seq_len, "parallelism": f"fsdp{world}",
            "pass_numerics": args.numerics, "perturb": "exact",
            "oz_slices": (args.oz_slices or default_oz_slices(cfg)) if args.numerics == "fp64_oz" else None,
            "act_ckpt": bool(args.act_ckpt),
            "l2": "no flush: per-step working set (theta+-, g+- fp64, activations, basis) > 0.5 GB > 126 MB L2"}


def run_reference(args, cfg):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import fdhvp, lanczos as OL, probe
    th = si.init_params(cfg)
    tok, scale = oracle_sample(cfg)
    g = fdhvp.make_grad_fn(cfg, tok)
    op = lambda q: fdhvp.fd_hvp_step(g, th, q, cfg.eps, "exact")
    # the weak-scaling configs' basis (m x P fp64: 99 GB on c3) does not fit a host: the reference
    # step there is the FD-HVP + three-term recurrence without a stored basis
    reorth = "none" if cfg.name in WEAK else reorth_of(args, cfg)
    okw = dict(window=args.window if reorth == "window" else 0, basis=args.basis)
    # (the numpy oracle has no warm-up effects beyond the first call: at most 2 untimed steps)
    OL.lanczos(op, probe.rademacher_probe(cfg.probe_seed0 + 99, th.size), max(min(args.warmup, 2), 1), reorth, **okw)
    t0 = time.perf_counter()
    done = 0
    j = 0
    while done < args.steps:
        m = min(cfg.m, args.steps - done)
        OL.lanczos(op, probe.rademacher_probe(cfg.probe_seed0 + j, th.size), m, reorth, **okw)
        done += m
        j += 1
    dt = time.perf_counter() - t0
    v = args.steps / dt * scale
    what = (f"{args.steps} oracle Lanczos steps ({reorth} reorth) on {tok.shape[0]} x {tok.shape[1] - 1} tokens"
            + ("" if scale == 1.0 else f", scaled to the {cfg.name} unit by linear-in-tokens extrapolation "
                                       f"(x {scale:.4g})"))
    print(json.dumps({
        "impl": "reference", "metric": metric_name(cfg.name), "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * dt / args.steps / scale,
        "higher_is_better": True, "scaling": "weak" if cfg.name in WEAK else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args, cfg, world, WEAK.get(cfg.name, cfg.n_seq) * world if cfg.name in WEAK
                              else cfg.n_seq),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "cpu": host_cpu(),
                         "sample": what},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}), flush=True)


def main():
    args = parse()
    cfg = si.CONFIGS[args.config]
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, cfg)
        return

    import torch
    import torch.distributed as dist
    from paper_2602_00816_b200 import build, slq

    if world > 1:
        dist.init_process_group("gloo", init_method="env://")
    torch.cuda.set_device(local)
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()

    uid = None
    if world > 1:
        obj = [slq.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    tok, n_glob = split_batch(cfg, rank, world)
    K, W = args.steps, max(args.warmup, 0)
    m_probe = max(args.probe_m or cfg.m, K + W)  # one probe holds the warm-up steps and the timed window
    k0 = max(W, (m_probe - K) // 2)
    ctx = slq.SlqContext(cfg, si.init_params(cfg), tok, n_global=n_glob, rank=rank, world_size=world, device=local,
                         unique_id=uid, pass_numerics=args.numerics,
                         reorth=reorth_of(args, cfg), window=args.window if args.reorth == "window" else 0,
                         basis=args.basis, max_steps=m_probe, perturb="exact", oz_slices=args.oz_slices,
                         act_ckpt=args.act_ckpt)
    stream = torch.cuda.ExternalStream(ctx.stream)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, n):
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / n

    # ---- headline: steps k0 .. k0 + K - 1 of one m-step probe, device-resident inputs ----
    ctx.lanczos_start(cfg.probe_seed0, m_probe)
    ctx.lanczos_step(k0)  # warm-up (untimed): the first k0 >= W steps of the probe
    clocks = ClockSampler(local) if rank == 0 else None
    l0 = ctx.launch_count()
    ms_step = timed(lambda: ctx.lanczos_step(K), K)
    launches = ctx.launch_count() - l0
    clk = clocks.stop() if clocks else None
    ctx.lanczos_step(m_probe - k0 - K)
    alpha, beta = ctx.lanczos_result()

    # ---- per-kernel-class profile of the same window in the same execution mode (overlap-aware:
    # both passes concurrent, side streams on; launches eager so each is event-timed) ----
    ctx.lanczos_start(cfg.probe_seed0, m_probe)
    ctx.lanczos_step(k0)
    torch.cuda.synchronize()
    ctx.profile("overlap", reset=True)
    prof_ms = timed(lambda: ctx.lanczos_step(K), K)
    stats = ctx.kernel_stats()
    busy_all = ctx.kernel_busy(-1)
    ctx.profile(False)
    ctx.lanczos_step(m_probe - k0 - K)
    ctx.lanczos_result()
    # ... and once more in the serial mode (one stream, no concurrency): each launch's event-timed
    # duration is its own -- the kernel's efficiency without the time it shares the GPU
    Ks = min(K, 4)
    ctx.lanczos_start(cfg.probe_seed0, m_probe)
    ctx.lanczos_step(k0)
    torch.cuda.synchronize()
    ctx.profile(True, reset=True)
    serial_ms = timed(lambda: ctx.lanczos_step(Ks), Ks)
    stats_serial = ctx.kernel_stats()
    ctx.profile(False)
    ctx.lanczos_step(m_probe - k0 - Ks)
    ctx.lanczos_result()

    # ---- standalone HVP, gradient step (same numerics), end-to-end HVP with host buffers ----
    P_loc = ctx.P_loc
    lay = ctx.layout()
    v_full = si.random_vector(ctx.P, 5)
    v_dev = torch.from_numpy(slq.shard_of(v_full, lay, rank, world)).cuda()
    out_dev = torch.empty_like(v_dev)
    nh = max(3, min(args.steps, 16))
    ctx.hvp(v_dev, out_dev, cfg.eps)
    hvp_ms = timed(lambda: [ctx.hvp(v_dev, out_dev, cfg.eps) for _ in range(nh)], nh)
    ctx.grad(None)
    grad_ms = timed(lambda: [ctx.grad(None) for _ in range(nh)], nh)
    v_host = torch.from_numpy(slq.shard_of(v_full, lay, rank, world)).pin_memory()
    out_host = torch.empty(P_loc, dtype=torch.float32).pin_memory()
    ctx.hvp(v_host, out_host, cfg.eps)
    e2e_ms = timed(lambda: [ctx.hvp(v_host, out_host, cfg.eps) for _ in range(nh)], nh)

    if rank != 0:
        ctx.close()
        if world > 1:
            dist.barrier()
        return

    # ---- roofline of the dominant kernel class: algorithmic work / its own time, from the serial-
    # mode re-run of the window (every kernel alone on the GPU, event-timed per launch: the same
    # serialisation as the committed ncu launch list, whose shares it must match); the overlap-aware
    # busy time of the class in the concurrent run is reported beside it ----
    peaks = measured_peaks()
    dom = max(stats_serial, key=lambda k: stats_serial[k]["ms"])
    st = stats_serial[dom]
    t_dom = st["ms"]  # (work and time both over the Ks serial steps)
    nS = args.oz_slices or default_oz_slices(cfg)
    if dom == "gemm_i8":
        # INT8 tensor-core products of the Ozaki fp64 GEMMs: peak = the measured bf16 SUSTAINED rate
        # (the timed region lasts seconds) x the nominal dense INT8 / BF16 ratio (4.5 / 2.25 POPS)
        bf16 = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0))
        i8_peak = 2.0 * bf16
        achieved = st["flops"] / (t_dom * 1e-3) / 1e12
        nprod = nS * (nS + 1) // 2
        roof = {"bound": "tensor", "achieved": achieved, "peak": i8_peak, "unit": "TOP/s", "frac": achieved / i8_peak,
                "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained" if "bf16_tflops_sustained" in peaks
                                else "fallback 1590 TFLOP/s") + " x 2 (nominal INT8 / BF16 dense ratio)",
                "fp64_equiv_tflops": achieved / nprod,
                "note": f"tcgen05 kind::i8 digit products, {nprod} INT8 GEMMs per fp64 GEMM (S = {nS} digit "
                        f"planes); every INT8 op issued is counted"}
    elif dom == "gemm" and args.numerics not in ("fp64", "fp64_oz"):
        bf16 = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1590.0))
        achieved = st["flops"] / (t_dom * 1e-3) / 1e12
        tc_note = {"bf16x3": "tcgen05 kind::f16 bf16 products (6 per fp32-faithful GEMM, all counted)",
                   "bf16": "tcgen05 kind::f16, one bf16 product per GEMM (native bf16 operands, fp32 accumulation)",
                   "paired": "tcgen05 pair GEMMs (7 + 12 bf16 products per pair GEMM) and SIMT fp32 attention",
                   }.get(args.numerics, "SIMT fp32 (no tensor core)")
        roof = {"bound": "tensor", "achieved": achieved, "peak": bf16, "unit": "TFLOP/s", "frac": achieved / bf16,
                "peak_source": ("MEASURED_PEAKS.json bf16_tflops_sustained" if "bf16_tflops_sustained" in peaks
                                else "fallback 1590 TFLOP/s") + "; " + tc_note}
    elif dom == "gemm":
        pk = slq.fp64_peak_tflops(local)
        fp64_peak = max(pk["dmma"], pk["dfma"])
        achieved = st["flops"] / (t_dom * 1e-3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak,
                "peak_source": f"measured on this GPU: fp64 tensor-core mma.sync m8n8k4 (DMMA) {pk['dmma']:.1f}, "
                               f"DFMA {pk['dfma']:.1f} TFLOP/s (slq_diag_*_peak); MEASURED_PEAKS.json has no fp64 "
                               f"entry and tcgen05 has no fp64 kind"}
    else:
        hbm = peaks.get("hbm_gbs", 6650.0)
        achieved = st["bytes"] / (t_dom * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6650 GB/s"}
    roof["ms_per_step"] = st["ms"] / Ks
    roof["serial_step_ms"] = serial_ms
    roof["share_of_serial_step"] = st["ms"] / Ks / serial_ms
    roof["what"] = ("achieved = the class's algorithmic work / its summed launch durations in a serial-mode re-run "
                    "of the timed window (one stream, each launch event-timed alone)")
    bd = stats[dom]["busy_ms"]
    if bd > 0:
        a_busy = st["flops" if roof["unit"] != "GB/s" else "bytes"] / Ks / (bd / K * 1e-3) / (
            1e12 if roof["unit"] != "GB/s" else 1e9)
        roof["overlap"] = {"busy_ms_per_step": bd / K, "achieved": a_busy, "frac": a_busy / roof["peak"],
                           "what": "the same work / the class's busy time (union of its launch intervals) in the "
                                   "concurrent run: includes the time it shares the GPU with the other pass"}
    roof["kernel"] = dom
    if dom == "gemm_i8" and "attn_i8" in stats_serial and stats_serial["attn_i8"]["ms"] > 0:
        # the same k_oz_gemm kernel on the batched causal attention contractions (oz_attn.cu), a class
        # of its own: N = hd = 64 tiles, k-clipped causal ranges
        sa = stats_serial["attn_i8"]
        a_att = sa["flops"] / (sa["ms"] * 1e-3) / 1e12
        roof["attention_i8"] = {"ms_per_step": sa["ms"] / Ks, "achieved": a_att, "frac": a_att / roof["peak"],
                                "launches_per_step": sa["launches"] / Ks,
                                "what": "batched causal attention GEMMs (S, O, dP, dV, dQ, dK) on the same kernel; "
                                        "algorithmic work = the causal half of each contraction"}
    roof["launches_per_step"] = st["launches"] / Ks
    roof["profiled_ms_per_step"] = prof_ms
    roof["device_busy_ms_per_step"] = busy_all / K
    roof["traffic"] = ncu_traffic(dom)

    units = world if cfg.name in WEAK else 1  # HVP units per step, whole job
    value = 1000.0 / ms_step * units
    out = {
        "metric": metric_name(cfg.name), "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": k0, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if cfg.name in WEAK else "strong",
        "vs_baseline": None, "dtype": {"fp64": "f64", "fp64_oz": "f64", "fp32": "f32", "bf16x3": "bf16x3", "bf16": "bf16", "paired": "paired-bf16x3", "paired_fp32": "paired-f32"}[args.numerics],
        "dtype_note": {"fp64_oz": f"fp64 activations and accumulation; dense GEMMs with M*N*K >= 1e9 and the causal attention contractions as exact int8 "
                                  f"digit products on tcgen05 (Ozaki, S={nS} digit planes of 7 bits per operand, "
                                  f"{nS * (nS + 1) // 2} products; S=5 (6 at eps < 5e-4) for the bf16 models, whose "
                                  f"gates are the bf16 ones, S=7 for the fp32 models), the rest fp64 DMMA"}.get(args.numerics, ""),
        "data": "synthetic",
        "config": config_dict(args, cfg, world, n_glob),
        "s_per_lanczos_step": ms_step / 1000.0,
        "hvp_per_s_standalone": 1000.0 / hvp_ms * units,
        # normalised throughput, tokens of the global batch x Lanczos steps per second
        "tokens_x_hvp_per_s": 1000.0 / ms_step * n_glob * cfg.seq_len,
        "grad_step_ms": grad_ms,
        "hvp_over_grad": hvp_ms / grad_ms,
        "e2e": {"value": 1000.0 / e2e_ms * units, "unit": UNIT, "h2d_bytes_per_step": 4 * P_loc * world,
                "d2h_bytes_per_step": 4 * P_loc * world,
                "what": "slq_hvp with pinned host v and host out (copies inside the call) per step"},
        "gpu_launches": launches,
        "memory_plan_gib": {k: round(v / 2**30, 2) for k, v in slq.plan_memory(ctx.desc, world, tok.shape[0]).items()},
        "kernel_busy_ms_per_step": {k: s["busy_ms"] / K for k, s in stats.items() if s["launches"]},
        "kernel_serial_ms_per_step": {k: s["ms"] / Ks for k, s in stats_serial.items() if s["launches"]},
        "timed_window": {"probe_m": m_probe, "first_step": k0, "steps": K,
                         "what": "steps k0 .. k0+K-1 of one m-step probe (slq_lanczos_step), centred on m/2"},
        "ritz_extremes": [float(x) for x in (lambda n: (n[0], n[-1]))(slq.quadrature(alpha, beta)[0])],
        "roofline": roof,
        "clocks": clk,
    }
    if not args.no_cpu_baseline and world == 1:
        out["cpu_baseline"] = cpu_baseline(cfg)
    print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.barrier()


if __name__ == "__main__":
    main()
