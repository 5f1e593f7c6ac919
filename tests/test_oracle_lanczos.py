"""Pins for oracle/lanczos.py: §4 recurrence, SLQ quadrature (CPU only)."""
import math

import numpy as np
import pytest

import slq_inputs as si
from oracle import fdhvp, lanczos as L, probe


def _unit(n, seed):
    x = np.random.default_rng(seed).standard_normal(n)
    return x / np.linalg.norm(x)


def test_diag_full_spectrum():
    """H = diag(1..32), m = 32, full reorth: Ritz values = 1..32."""
    H = np.diag(np.arange(1.0, 33.0))
    r = L.lanczos(lambda q: H @ q, probe.rademacher_probe(1, 32), 32, "full")
    nodes, w = L.gauss_quadrature(r.alpha, r.beta)
    assert r.m_done == 32
    assert np.max(np.abs(nodes - np.arange(1.0, 33.0))) < 1e-10
    # Rademacher probe has equal weight on every eigenvector of a diagonal matrix
    assert np.max(np.abs(w - 1 / 32)) < 1e-10


def test_scaled_identity_breakdown():
    """H = c I: one-dimensional Krylov space -> breakdown at step 1 with alpha_1 = c."""
    c = 2.5
    r = L.lanczos(lambda q: c * q, _unit(40, 1), 10, "full")
    assert r.breakdown and r.m_done == 1
    assert abs(r.alpha[0] - c) < 1e-14
    assert r.beta.size == 0


def test_extremal_convergence_no_reorth():
    """H = diag(1..200), m = 30, no reorth: largest Ritz value converges to 200."""
    H = np.arange(1.0, 201.0)
    r = L.lanczos(lambda q: H * q, _unit(200, 3), 30, "none")
    nodes, _ = L.gauss_quadrature(r.alpha, r.beta)
    assert abs(nodes[-1] - 200.0) < 1e-2
    # residual bound of the largest Ritz pair (exact arithmetic statement, holds here)
    lam, V = np.linalg.eigh(L.tridiag(r.alpha, r.beta))
    assert abs(nodes[-1] - 200.0) <= r.beta_next * abs(V[-1, -1]) + 1e-10


def _rand_sym(n, seed):
    A = np.random.default_rng(seed).standard_normal((n, n))
    return (A + A.T) / 2


def test_interlacing_and_moments():
    """Ritz values of T_m interlace those of T_{m+1}; Gauss quadrature with m nodes
    reproduces q1^T H^j q1 for j <= 2m-1 (S:332 checks j <= 3)."""
    H = _rand_sym(60, 11)
    q1 = _unit(60, 12)
    r = L.lanczos(lambda q: H @ q, q1, 12, "full")
    for m in range(2, 12):
        a = np.sort(np.linalg.eigvalsh(L.tridiag(r.alpha[:m], r.beta[:m - 1])))
        b = np.sort(np.linalg.eigvalsh(L.tridiag(r.alpha[:m + 1], r.beta[:m])))
        assert np.all(b[:-1] <= a + 1e-12) and np.all(a <= b[1:] + 1e-12)
    m = 4
    nodes, w = L.gauss_quadrature(r.alpha[:m], r.beta[:m - 1])
    x = q1.copy()
    for j in range(2 * m):
        ref = q1 @ x
        assert abs(L.moment(nodes, w, j) - ref) <= 1e-9 * max(1.0, np.linalg.norm(H, 2) ** j)
        x = H @ x


def test_quadrature_chebyshev_closed_form():
    """Jacobi matrix of the Chebyshev (1st kind) weight: alpha = 0, beta_1 = 1/sqrt2,
    beta_k = 1/2 -> nodes cos((2i-1)pi/(2m)), weights exactly 1/m."""
    for m in (1, 2, 5, 16, 40):
        beta = np.full(m - 1, 0.5)
        if m > 1:
            beta[0] = 1 / math.sqrt(2)
        nodes, w = L.gauss_quadrature(np.zeros(m), beta)
        ref = np.sort(np.cos((2 * np.arange(1, m + 1) - 1) * math.pi / (2 * m)))
        assert np.max(np.abs(nodes - ref)) < 1e-13
        assert np.max(np.abs(w - 1.0 / m)) < 1e-13


def test_quadrature_legendre_textbook():
    """Legendre: alpha = 0, beta_k = k/sqrt(4k^2-1) -> Gauss-Legendre nodes, weights/2."""
    for m in (3, 10, 33):
        k = np.arange(1, m)
        nodes, w = L.gauss_quadrature(np.zeros(m), k / np.sqrt(4 * k * k - 1.0))
        x, wl = np.polynomial.legendre.leggauss(m)
        assert np.max(np.abs(nodes - x)) < 1e-13
        assert np.max(np.abs(w - wl / 2)) < 1e-13


def test_quadrature_edge_cases():
    """m = 1 -> ({alpha_1}, {1});  T = diag(2, 5) (beta = 0) -> ({2, 5}, {1, 0})."""
    n, w = L.gauss_quadrature([3.25], [])
    assert n.tolist() == [3.25] and w.tolist() == [1.0]
    n, w = L.gauss_quadrature([2.0, 5.0], [0.0])
    assert n.tolist() == [2.0, 5.0] and w.tolist() == [1.0, 0.0]
    n, w = L.gauss_quadrature([5.0, 2.0], [0.0])
    assert n.tolist() == [2.0, 5.0] and w.tolist() == [0.0, 1.0]


def test_weights_sum_and_first_moment():
    """mu_0 = sum tau = 1 and mu_1 = alpha_1 = q1^T H q1 (Hutchinson identity per probe)."""
    H = _rand_sym(50, 21)
    z = probe.signs(5, 50)
    q1 = z / math.sqrt(50)
    r = L.lanczos(lambda q: H @ q, q1, 20, "full")
    nodes, w = L.gauss_quadrature(r.alpha, r.beta)
    assert abs(w.sum() - 1) < 1e-12
    assert abs(L.moment(nodes, w, 1) - r.alpha[0]) < 1e-12
    assert abs(50 * L.moment(nodes, w, 1) - z @ H @ z) < 1e-10 * abs(z @ H @ z) + 1e-12
    # SLQ trace over many probes approaches the exact trace (S:305 example, 5% band)
    ns, ws = [], []
    for s in range(64):
        qs = probe.rademacher_probe(100 + s, 50)
        rr = L.lanczos(lambda q: H @ q, qs, 10, "full")
        a, b = L.gauss_quadrature(rr.alpha, rr.beta)
        ns.append(a)
        ws.append(b)
    mu = L.slq_moments(ns, ws, 2)
    assert abs(mu[0] - 1) < 1e-12
    # Hutchinson: Var(z^T H z) = 2 sum_{i!=j} H_ij^2 for Rademacher z; 4-sigma band
    off = H - np.diag(np.diag(H))
    assert abs(50 * mu[1] - np.trace(H)) < 4 * math.sqrt(2.0) * np.linalg.norm(off, "fro") / 8
    grid = np.linspace(-20, 20, 4001)
    dens = L.slq_density(grid, ns, ws, 0.5)
    assert abs(np.trapezoid(dens, grid) - 1) < 1e-6


def test_jacobi_reconstructs():
    A = _rand_sym(30, 4)
    lam, V = L.jacobi_eigh(A)
    assert np.max(np.abs(V @ np.diag(lam) @ V.T - A)) < 1e-12
    assert np.max(np.abs(V.T @ V - np.eye(30))) < 1e-12


def test_full_reorth_keeps_orthogonality():
    """With CGS2 full reorth the fp64 basis stays orthonormal to ~1e-14 even past
    convergence; without it orthogonality is lost (Paige)."""
    H = np.concatenate([np.linspace(0, 1, 299), [100.0]])
    q1 = _unit(300, 9)
    rf = L.lanczos(lambda q: H * q, q1, 60, "full", keep_basis=True)
    Qf = rf.basis
    assert np.max(np.abs(Qf @ Qf.T - np.eye(rf.m_done))) < 1e-13
    rn = L.lanczos(lambda q: H * q, q1, 60, "none", keep_basis=True)
    Qn = rn.basis
    assert np.max(np.abs(Qn @ Qn.T - np.eye(rn.m_done))) > 1e-6
