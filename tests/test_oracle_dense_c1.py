"""Brute-force dense Hessian of config c1 (BASELINE configs[0] "Oracle cross-check: brute-force
dense Hessian via eigvalsh"; SURVEY §8(c3) 'Dense Hessian (c1)' / 'Extreme Ritz (c1)').

H is built column by column with the oracle's own FD-HVP (Eq. (1), exact mode, fp64 passes)
and checked for symmetry; its extreme eigenvalues (LAPACK eigvalsh, a library routine) must
match the oracle Lanczos' extreme Ritz values within the residual bound.
"""
import numpy as np
import pytest

import slq_inputs as si
from oracle import fdhvp, lanczos as L, probe


@pytest.fixture(scope="module")
def dense_c1():
    d = si.CONFIGS["c1"]
    th = si.init_params(d)
    b = si.mlp_data(d)
    g = fdhvp.make_grad_fn(d, b)
    P = th.size
    H = np.empty((P, P))
    e = np.zeros(P)
    for i in range(P):
        e[i] = 1.0
        # step 1e-4 in fp64: coordinate directions have a larger third-derivative term, so the
        # brute-force matrix uses a smaller step (bias ~1e-10, round-off ~u||g||/eps ~1e-12)
        H[:, i] = fdhvp.fd_hvp_step(g, th, e, 1e-4, "exact")
        e[i] = 0.0
    return d, th, b, g, H


def test_dense_hessian_symmetric(dense_c1):
    d, th, b, g, H = dense_c1
    assert np.linalg.norm(H - H.T) <= 1e-6 * np.linalg.norm(H)


def test_extreme_ritz_match_eigvalsh(dense_c1):
    d, th, b, g, H = dense_c1
    Hs = (H + H.T) / 2
    lam = np.linalg.eigvalsh(Hs)
    nrm = max(abs(lam[0]), abs(lam[-1]))
    q1 = probe.rademacher_probe(d.probe_seed0, th.size)
    for m in (32, 64):
        # (i) exact matvec with the dense matrix: residual bound + round-off
        # (ii) the FD operator at the config eps: + Theorem 1 bias (~eps^2, measured 1.3e-7)
        for op, slack in ((lambda q: Hs @ q, 1e-10),
                          (lambda q: fdhvp.fd_hvp_step(g, th, q, d.eps, "exact"), 1e-6)):
            r = L.lanczos(op, q1, m, "full")
            ritz, S = np.linalg.eigh(L.tridiag(r.alpha, r.beta))
            for idx in (0, -1):
                bound = r.beta_next * abs(S[-1, idx]) + slack * nrm
                assert np.min(np.abs(lam - ritz[idx])) <= bound
            # the largest eigenvalue is an isolated outlier: converged at m = 32
            assert abs(ritz[-1] - lam[-1]) <= slack * nrm
    # parity-mode operator (fp32-rounded perturbed points): extreme value within the
    # perturbation-quantisation error (~4e-4 on c1)
    r = L.lanczos(lambda q: fdhvp.fd_hvp_step(g, th, q.astype(np.float32), d.eps, "param_dtype"),
                  q1, 32, "full")
    ritz = np.linalg.eigvalsh(L.tridiag(r.alpha, r.beta))
    assert abs(ritz[-1] - lam[-1]) <= 2e-3 * nrm


def test_trace_and_moments_identity(dense_c1):
    """P * mu_1 is that probe's Hutchinson sample z^T H z (identity per probe, §8(c3))."""
    d, th, b, g, H = dense_c1
    P = th.size
    z = probe.signs(d.probe_seed0 + 1, P)
    r = L.lanczos(lambda q: H @ q, z / np.sqrt(P), 16, "full")
    nodes, w = L.gauss_quadrature(r.alpha, r.beta)
    assert abs(w.sum() - 1) < 1e-12
    assert abs(P * L.moment(nodes, w, 1) - z @ H @ z) <= 1e-10 * abs(z @ H @ z)
    # second moment: mu_2 = ||H q1||^2 = alpha_1^2 + beta_2^2
    q1 = z / np.sqrt(P)
    assert abs(L.moment(nodes, w, 2) - np.dot(H @ q1, H @ q1)) <= 1e-10 * np.dot(H @ q1, H @ q1)
    assert abs(L.moment(nodes, w, 2) - (r.alpha[0] ** 2 + r.beta[0] ** 2)) <= 1e-12 * L.moment(nodes, w, 2)
