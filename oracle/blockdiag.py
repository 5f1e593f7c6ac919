"""Block-diagonal hypothesis test (oracle; test infrastructure only).

PAPER.md P:501-517 (§6, Exp I): theta is partitioned into contiguous blocks theta^(b) (transformer
layers); for a probe v with ||v|| = 1, h_full = H v and, per block, h_masked^(b) = H v^(b) with
v^(b) = v zeroed outside block b.  Both are restricted to block b and compared:
    rel_err_b = ||(Hv)^(b) - (H v^(b))^(b)|| / ||(Hv)^(b)||,    cos_b = <(Hv)^(b), (H v^(b))^(b)> / norms
Readings (R18): the paper draws v ~ N(0, I) normalised; the product path uses the
Rademacher probe of the Lanczos runs (any probe works for the test); blocks = the FSDP units
(embedding, each transformer block, final norm + head) in canonical order; H v is the FD-HVP of
Eq. (1) in exact mode.
"""
from __future__ import annotations

from typing import Callable, List, Sequence, Tuple

import numpy as np


def block_test(apply_h: Callable[[np.ndarray], np.ndarray], v: np.ndarray,
               blocks: Sequence[Tuple[int, int]]):
    """blocks: [(start, end)) canonical ranges.  Returns (rel_err[b], cosine[b])."""
    v = np.asarray(v, dtype=np.float64)
    h_full = np.asarray(apply_h(v), dtype=np.float64)
    rel: List[float] = []
    cos: List[float] = []
    for s, e in blocks:
        vb = np.zeros_like(v)
        vb[s:e] = v[s:e]
        hb = np.asarray(apply_h(vb), dtype=np.float64)[s:e]
        hf = h_full[s:e]
        rel.append(float(np.linalg.norm(hf - hb) / np.linalg.norm(hf)))
        cos.append(float(hf @ hb / (np.linalg.norm(hf) * np.linalg.norm(hb))))
    return np.array(rel), np.array(cos)
