"""compute-sanitizer target: a small run of every path the product takes (probe, perturb, both
gradient passes on the FP64_OZ hybrid route, FD difference, CGS2, checkpointing, resumable
Lanczos) on gpt_tiny and c2.  Usage: compute-sanitizer --tool memcheck python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SLQ_NO_GRAPHS", "1")  # eager launches: every kernel is checked as launched

import numpy as np
import torch

import slq_inputs as si
from paper_2602_00816_b200 import slq

for name, num, kw in [("gpt_tiny", "fp64_oz", dict(oz_min_mnk=1.0)), ("llama_tiny", "fp64", dict(act_ckpt=True)),
                      ("c2", "fp64_oz", {})]:
    cfg = si.get_config(name, n_layers=3) if name == "llama_tiny" else si.CONFIGS[name]
    th = si.init_params(cfg)
    with slq.SlqContext(cfg, th, si.tokens(cfg), pass_numerics=num, reorth="full", max_steps=4, **kw) as c:
        v = torch.from_numpy(slq.shard_of(si.random_vector(th.size, 5), c.layout(), 0, 1)).cuda()
        out = torch.empty_like(v)
        c.hvp(v, out, cfg.eps)
        c.lanczos_start(cfg.probe_seed0, 4)
        c.lanczos_step(2)
        c.lanczos_step(2)
        a, b = c.lanczos_result()
        print(name, num, "alpha", a, flush=True)
print("sanitize run done")
