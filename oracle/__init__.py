"""CPU oracle for the SLQ / FD-HVP hot path of arXiv 2602.00816 -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import, call, link or execute anything under `oracle/`.  The product path
(`paper_2602_00816_b200`, `include/slq.h`, the CUDA library) never does, and shares no code
with it: the only common module is `slq_inputs`, which holds seeded input generators and no
method arithmetic.

Plain, slow, fp64 numpy (plus one C helper for the single-rounding fp32 FMA perturbation).
Every function cites the PAPER.md passage it follows as `P:<line>` (section / equation /
algorithm), or the SURVEY.md reading it takes where the paper is silent.

Modules
  probe      -- Rademacher probe from the integer splitmix64 hash (SURVEY §8(c2) hash reading)
  models     -- MLP / GPT / Llama loss and hand-derived gradient (the L of Eq. (1))
  fdhvp      -- Eq. (1) central FD-HVP, Alg. 1, Theorem 1 step size
  lanczos    -- §4 Lanczos recurrence with optional CGS2 full reorthogonalisation,
                Jacobi tridiagonal eigensolver -> Gauss nodes/weights, SLQ moments / density

Parity status of each function is listed in DESIGN.md §"Oracle pins"; every function here is
pinned by at least one `-m "not gpu"` test in tests/test_oracle_*.py.
"""
from . import probe, models, fdhvp, lanczos, cg, blockdiag  # noqa: F401
