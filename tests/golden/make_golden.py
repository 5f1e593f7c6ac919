"""Writes the stored oracle results of the large parity cases (test infrastructure only).

Every value this script writes comes from `oracle/` (fp64 numpy) on the seeded
inputs of `slq_inputs` -- nothing from the CUDA path.  The large cases (c3 / c4 parity batches,
the c5 twin) cost the oracle 30-70 s per FD-HVP, too slow to recompute inside the GPU test run,
so their Lanczos coefficients and a sampled image of H q_1 are stored here:

  * alpha[m], beta[m-1], beta_{m+1}: `oracle.lanczos.lanczos` (Paige's A(2,7) order;
    CGS2 for reorth "full") on the FD-HVP operator `oracle.fdhvp.fd_hvp_step(..., "exact")`
    (Eq. (1); reading R9) from the Rademacher probe q_1 (R4);
  * H q_1 (the first operator application of that run): its 2-norm, its value at 8192 seeded
    indices plus the first / last 64, and its projections on four Rademacher sign vectors.

usage: python tests/golden/make_golden.py --case c3_parity --m 32 --eps 1e-2 1e-3 1e-4 --reorth full
Output: tests/golden/lanczos_<case>_eps<eps>_m<m>_<reorth>.json (one file per eps).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import slq_inputs as si  # noqa: E402
from oracle import fdhvp, lanczos as OL, probe  # noqa: E402

N_SAMPLE = 8192
PROJ_SEEDS = (9001, 9002, 9003, 9004)


def sample_indices(P: int, seed: int) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 4242])))
    mid = g.choice(np.arange(64, P - 64), size=min(N_SAMPLE, P - 128), replace=False)
    return np.unique(np.concatenate([np.arange(64), mid, np.arange(P - 64, P)])).astype(np.int64)


OUT_DIR = HERE


def golden_path(case: str, eps: float, m: int, reorth: str) -> str:
    return os.path.join(OUT_DIR, f"lanczos_{case}_eps{eps:g}_m{m}_{reorth}.json")


def run(case: str, eps: float, m: int, reorth: str) -> dict:
    cfg = si.get_config(case, eps=eps, m=m)
    t0 = time.time()
    th = si.init_params(cfg)
    tok = si.tokens(cfg)
    P = th.size
    q1 = probe.rademacher_probe(cfg.probe_seed0, P)
    g = fdhvp.make_grad_fn(cfg, tok)
    first = {}
    steps = []  # operator applications so far (a partial file is rewritten after each one)

    def record(alpha, beta, beta_next, m_done, breakdown):
        hq1 = first["hq1"]
        idx = first.setdefault("idx", sample_indices(P, cfg.probe_seed0))
        if "proj" not in first:
            first["proj"] = [float(np.dot(probe.signs(s, P), hq1)) for s in PROJ_SEEDS]
        return {
            "case": case, "eps": eps, "m": m, "reorth": reorth, "perturb": "exact", "P": int(P),
            "n_seq": cfg.n_seq, "seq_len": cfg.seq_len, "probe_seed": cfg.probe_seed0,
            "alpha": [float(x) for x in alpha], "beta": [float(x) for x in beta],
            "beta_next": float(beta_next), "m_done": int(m_done), "breakdown": bool(breakdown),
            "hvp_q1": {"norm": float(np.linalg.norm(hq1)), "idx": [int(i) for i in idx],
                       "val": [float(hq1[i]) for i in idx], "proj_seeds": list(PROJ_SEEDS), "proj": first["proj"]},
            "generator": "tests/golden/make_golden.py (oracle/ only)",
            "oracle_seconds": round(time.time() - t0, 1),
            "host": f"{platform.node()} {os.cpu_count()} cpus",
        }

    def op(q):
        h = fdhvp.fd_hvp_step(g, th, q, eps, "exact")
        if not first:
            first["hq1"] = h
            print(f"  {case} eps={eps:g}: H q1 after {time.time() - t0:.0f} s", flush=True)
        steps.append(1)
        return h

    # checkpoint after every step: a run cut short still leaves the coefficients of the steps it
    # finished (the first k steps of an m-step run are the k-step run), as m = k in the file
    def on_step(alpha, betas):
        k = len(alpha)
        if k < m:
            d = record(alpha, betas[:k - 1], betas[k - 1], k, False)
            d["m"] = k
            d["partial_of"] = m
            with open(golden_path(case, eps, m, reorth) + ".partial", "w") as f:
                json.dump(d, f)

    r = OL.lanczos(op, q1, m, reorth, on_step=on_step)
    out = record(r.alpha, r.beta, r.beta_next, r.m_done, r.breakdown)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    ap.add_argument("--m", type=int, required=True)
    ap.add_argument("--eps", type=float, nargs="+", required=True)
    ap.add_argument("--reorth", default="full", choices=["full", "none"])
    ap.add_argument("--out-dir", default=HERE)
    ap.add_argument("--mem-limit-gb", type=float, default=0.0,
                    help="RLIMIT_AS for this process (a MemoryError instead of the host's OOM killer)")
    a = ap.parse_args()
    global OUT_DIR
    OUT_DIR = a.out_dir
    os.makedirs(OUT_DIR, exist_ok=True)
    if a.mem_limit_gb > 0:
        import resource
        lim = int(a.mem_limit_gb * 2**30)
        resource.setrlimit(resource.RLIMIT_AS, (lim, lim))
    for eps in a.eps:
        d = run(a.case, eps, a.m, a.reorth)
        path = golden_path(a.case, eps, a.m, a.reorth)
        with open(path, "w") as f:
            json.dump(d, f)
        print(f"wrote {path} ({d['oracle_seconds']} s)", flush=True)


if __name__ == "__main__":
    main()
