"""Lanczos recurrence, reorthogonalisation, Gauss quadrature and SLQ (oracle; test infra only).

PAPER.md P:305-316 (§4):
    beta_{k+1} q_{k+1} = H q_k - alpha_k q_k - beta_k q_{k-1},   alpha_k = q_k^T H q_k
    v^T f(H) v ~= e_1^T f(T_m) e_1           (stochastic Lanczos quadrature)
PAPER.md P:1097-1121 (App. C): shard-local mechanics; reorthogonalisation against stored
vectors, one global dot product + one AXPY each.

Readings:
  * App. C's printed order (beta_t = ||w|| before the subtraction) is garbled;
    this follows the §4 recurrence in Paige's A(2,7) order:
        w = H q_k - beta_k q_{k-1};  alpha_k = <w, q_k>;  w -= alpha_k q_k;
        [full: classical Gram-Schmidt against q_1..q_k, done twice (CGS2)]
        beta_{k+1} = ||w||;  stop if beta_{k+1} <= tol * max|T|;  q_{k+1} = w / beta_{k+1}
  * Output alpha[1..m], beta[2..m] (the API's beta[m-1]) and beta_{m+1} as a diagnostic.
  * Quadrature nodes/weights: eigen-decomposition of T_m by cyclic Jacobi rotations (an
    algorithm independent of the library's implicit-shift QL); nodes ascending, weights =
    squared first components of the normalised eigenvectors.
  * Sliding-window reorthogonalisation ("sliding-window reorthogonalisation of size
    r"; "orthogonalised against up to r previously stored Lanczos vectors"): the same
    CGS2 as `full`, restricted to the r most recent vectors q_{k-r+1} .. q_k (DESIGN.md reading
    R17; r >= k reduces to full).
  * Basis storage precision ("only the Lanczos basis vectors are stored in
    either bfloat16 or float32", scalars in higher precision): q_{k+1} = round(w / beta_{k+1})
    to the storage format, and every later use of q_j (the HVP direction, the three-term
    recurrence, alpha, the reorthogonalisation) reads the stored, rounded vector.  bf16 rounding
    is round-to-nearest-even from the fp64 value (`bf16_round`).
  * Ghosts ("loss of orthogonality yields ghost eigenvalues"; Theorem 3's "spurious
    duplicate eigenvalues"): `ghost_clusters` groups the sorted Ritz values whose neighbour gaps
    are <= tol; a cluster with two or more members is a duplicate ("ghost") cluster.  An
    unreduced T_m has distinct eigenvalues, so in exact arithmetic such clusters arise only
    from genuinely clustered eigenvalues of H or from lost orthogonality (R18).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, List, Sequence, Tuple

import numpy as np


@dataclass
class LanczosResult:
    alpha: np.ndarray        # [m_done]
    beta: np.ndarray         # [m_done - 1]  (beta_2 .. beta_{m_done})
    beta_next: float         # beta_{m_done + 1}
    m_done: int
    breakdown: bool
    basis: np.ndarray | None = None   # [m_done, P] when kept


def bf16_round(x) -> np.ndarray:
    """Round fp64 values to the nearest bfloat16 (8 significant bits, exponent range of fp32),
    ties to even; returned as fp64.  Written out from the format's definition: with e the
    binary exponent of |x| (clamped to the fp32 subnormal floor -126), the bf16 spacing near x
    is 2^(e-7); x / spacing is exact (power-of-two scaling) and np.round rounds half to even."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    nz = (x != 0) & np.isfinite(x)
    e = np.floor(np.log2(np.abs(x[nz])))
    # log2 can be off by one ulp near powers of two: fix e so that 2^e <= |x| < 2^(e+1)
    ax = np.abs(x[nz])
    e = np.where(np.ldexp(1.0, e.astype(np.int64)) > ax, e - 1, e)
    e = np.where(np.ldexp(1.0, (e + 1).astype(np.int64)) <= ax, e + 1, e)
    e = np.maximum(e, -126.0)
    spacing = np.ldexp(1.0, (e - 7).astype(np.int64))
    out[nz] = np.round(x[nz] / spacing) * spacing
    out[~np.isfinite(x)] = x[~np.isfinite(x)]
    return out


def store(x: np.ndarray, basis: str) -> np.ndarray:
    """Basis storage rounding: fp64 (none), fp32 (RNE) or bf16 (RNE)."""
    if basis == "fp64":
        return np.asarray(x, dtype=np.float64)
    if basis == "fp32":
        return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)
    if basis == "bf16":
        return bf16_round(x)
    raise ValueError(basis)


def lanczos(apply_h: Callable[[np.ndarray], np.ndarray], q1: np.ndarray, m: int,
            reorth: str = "full", tol: float = 1e-10, keep_basis: bool = False,
            window: int = 0, basis: str = "fp64", on_step=None) -> LanczosResult:
    """m steps of symmetric Lanczos from unit q1, A(2,7) order, fp64 scalars.
    reorth: "none" | "full" | "window" (CGS2 against the `window` most recent vectors);
    basis: storage of the Lanczos vectors, "fp64" | "fp32" | "bf16".
    on_step(alpha, betas): optional progress hook (no arithmetic), called after every step with the
    coefficients so far -- alpha_1..alpha_k and beta_2..beta_{k+1}."""
    if reorth == "window" and window < 1:
        raise ValueError("window reorthogonalisation needs window >= 1")
    q = store(q1, basis).copy()
    P = q.size
    Q = np.empty((m, P)) if (reorth in ("full", "window") or keep_basis) else None
    alpha: List[float] = []
    betas: List[float] = []          # beta_{k+1} for k = 1..m_done
    q_prev = np.zeros(P)
    b = 0.0
    breakdown = False
    for k in range(m):
        w = np.asarray(apply_h(q), dtype=np.float64) - b * q_prev
        a = float(np.dot(w, q))
        w = w - a * q
        if Q is not None:
            Q[k] = q
        if reorth in ("full", "window"):
            Qk = Q[:k + 1] if reorth == "full" else Q[max(0, k + 1 - window):k + 1]
            for _ in range(2):                       # CGS2
                c = Qk @ w
                w = w - Qk.T @ c
        elif reorth != "none":
            raise ValueError(reorth)
        b_next = float(np.sqrt(np.dot(w, w)))
        alpha.append(a)
        betas.append(b_next)
        if on_step is not None:
            on_step(list(alpha), list(betas))
        tmax = max(max(abs(x) for x in alpha), max(betas[:-1], default=0.0))
        if b_next <= tol * tmax:
            breakdown = True
            break
        q_prev, q = q, store(w / b_next, basis)
        b = b_next
    md = len(alpha)
    return LanczosResult(alpha=np.array(alpha), beta=np.array(betas[:md - 1]),
                         beta_next=betas[md - 1], m_done=md, breakdown=breakdown,
                         basis=(Q[:md] if (keep_basis and Q is not None) else None))


def tridiag(alpha: Sequence[float], beta: Sequence[float]) -> np.ndarray:
    a = np.asarray(alpha, dtype=np.float64)
    b = np.asarray(beta, dtype=np.float64)
    return np.diag(a) + np.diag(b, 1) + np.diag(b, -1)


def jacobi_eigh(A: np.ndarray, max_sweeps: int = 60) -> Tuple[np.ndarray, np.ndarray]:
    """Cyclic Jacobi eigen-decomposition of a symmetric matrix: A = V diag(lam) V^T."""
    A = np.array(A, dtype=np.float64)
    n = A.shape[0]
    V = np.eye(n)
    scale = max(np.abs(A).max(), 1e-300)
    for _ in range(max_sweeps):
        off = math.sqrt(float(np.sum(np.triu(A, 1) ** 2)))
        if off <= 1e-17 * scale * n:
            break
        for p in range(n - 1):
            for r in range(p + 1, n):
                apr = A[p, r]
                if abs(apr) <= 1e-300:
                    continue
                th = (A[r, r] - A[p, p]) / (2.0 * apr)
                t = math.copysign(1.0, th) / (abs(th) + math.sqrt(th * th + 1.0))
                c = 1.0 / math.sqrt(t * t + 1.0)
                s = t * c
                # A <- J^T A J with J the (p, r) rotation
                Ap, Ar = A[:, p].copy(), A[:, r].copy()
                A[:, p] = c * Ap - s * Ar
                A[:, r] = s * Ap + c * Ar
                Ap, Ar = A[p, :].copy(), A[r, :].copy()
                A[p, :] = c * Ap - s * Ar
                A[r, :] = s * Ap + c * Ar
                Vp, Vr = V[:, p].copy(), V[:, r].copy()
                V[:, p] = c * Vp - s * Vr
                V[:, r] = s * Vp + c * Vr
    return np.diag(A).copy(), V


def gauss_quadrature(alpha: Sequence[float], beta: Sequence[float]) -> Tuple[np.ndarray, np.ndarray]:
    """Nodes theta_i (ascending) and weights tau_i = (e_1^T s_i)^2 of T_m."""
    lam, V = jacobi_eigh(tridiag(alpha, beta))
    order = np.argsort(lam, kind="stable")
    return lam[order], (V[0, order] ** 2)


def moment(nodes: np.ndarray, weights: np.ndarray, j: int) -> float:
    """e_1^T T^j e_1 = sum_i tau_i theta_i^j (the j-th spectral moment of one probe)."""
    return float(np.sum(weights * nodes ** j))


def slq_moments(node_sets, weight_sets, jmax: int = 2) -> np.ndarray:
    """Probe-averaged moments mu_0..mu_jmax."""
    s = len(node_sets)
    return np.array([sum(moment(n, w, j) for n, w in zip(node_sets, weight_sets)) / s
                     for j in range(jmax + 1)])


def slq_density(grid: np.ndarray, node_sets, weight_sets, sigma: float) -> np.ndarray:
    """Gaussian-smoothed SLQ density (1/s) sum_p sum_i tau_i N(x; theta_i, sigma^2)."""
    out = np.zeros_like(grid, dtype=np.float64)
    for nodes, w in zip(node_sets, weight_sets):
        out += (w[None, :] * np.exp(-0.5 * ((grid[:, None] - nodes[None, :]) / sigma) ** 2)).sum(1)
    return out / (len(node_sets) * sigma * math.sqrt(2 * math.pi))


def ghost_clusters(nodes: Sequence[float], tol: float) -> Tuple[np.ndarray, List[Tuple[int, int, float]]]:
    """Single-linkage clusters of the ascending Ritz values: nodes i and i+1 share a cluster when
    nodes[i+1] - nodes[i] <= tol.  Returns the cluster id of every node and, for every cluster
    with >= 2 members (a duplicate / "ghost" cluster), (first index, size, splitting =
    max - min).  tol = 0 separates distinct values (an unreduced T_m has distinct eigenvalues)."""
    x = np.asarray(nodes, dtype=np.float64)
    ids = np.zeros(x.size, dtype=np.int64)
    for i in range(1, x.size):
        ids[i] = ids[i - 1] + (0 if x[i] - x[i - 1] <= tol else 1)
    ghosts = []
    for c in range(int(ids[-1]) + 1 if x.size else 0):
        idx = np.nonzero(ids == c)[0]
        if idx.size >= 2:
            ghosts.append((int(idx[0]), int(idx.size), float(x[idx[-1]] - x[idx[0]])))
    return ids, ghosts
