"""Conjugate-gradient inverse-HVP on the FD-HVP operator (oracle; test infrastructure only).

PAPER.md P:30 / P:74 ("CG-based inverse-HVP solvers"), P:445 and P:1164-1165 ("A CG-based
inverse-HVP solver similarly reduces to repeated HVP calls plus scalar reductions and shard-local
vector operations").  The paper gives no algorithm beyond that, so this is textbook CG
(Hestenes-Stiefel) on (H + lambda I) x = b with x_0 = 0:
    r = b; p = r; repeat: Ap = H p + lambda p; a = r.r / p.Ap; x += a p; r -= a Ap;
    stop if ||r|| <= tol ||b||; beta = r'.r' / r.r; p = r' + beta p
Reading (R17): damping lambda makes the indefinite Hessian SPD for the solver.
"""
from __future__ import annotations

from typing import Callable, List

import numpy as np


def cg(apply_h: Callable[[np.ndarray], np.ndarray], b: np.ndarray, damping: float, max_iter: int,
       tol: float = 0.0):
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = float(r @ r)
    nb = float(np.sqrt(b @ b))
    hist: List[float] = []
    it = 0
    for it in range(1, max_iter + 1):
        ap = np.asarray(apply_h(p), dtype=np.float64) + damping * p
        a = rr / float(p @ ap)
        x = x + a * p
        r = r - a * ap
        rr_new = float(r @ r)
        hist.append(np.sqrt(rr_new) / nb)
        if np.sqrt(rr_new) <= tol * nb:
            break
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, it, hist
