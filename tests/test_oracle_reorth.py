"""Pins for the §8(f3) oracle pieces: sliding-window reorthogonalisation,
bf16 basis storage and ghost clusters.  CPU only."""
import numpy as np
import pytest

import slq_inputs as si
from oracle import fdhvp, lanczos as L, probe

torch = pytest.importorskip("torch")


def test_bf16_round_ties_and_specials():
    """Hand-worked cases of round-to-nearest-even with 8 significant bits."""
    x = np.array([1.0, 1 + 2.0**-8, 1 + 3 * 2.0**-8, 1 + 2.0**-8 + 2.0**-30, -(1 + 3 * 2.0**-8), 0.0, 2.0**-133,
                  1.5 * 2.0**-133, 2.0**-134, 3.0 * 2.0**-135])
    want = np.array([1.0, 1.0, 1 + 2.0**-6, 1 + 2.0**-7, -(1 + 2.0**-6), 0.0, 2.0**-133,
                     2.0 * 2.0**-133, 0.0, 2.0**-133])
    assert np.array_equal(L.bf16_round(x), want)


def test_bf16_round_matches_library_on_fp32_inputs():
    """On fp32-representable inputs, fp64 -> bf16 RNE is the library's fp32 -> bf16 cast."""
    rng = np.random.default_rng(0)
    r = np.concatenate([rng.standard_normal(200000), rng.standard_normal(1000) * 1e-39,
                        rng.standard_normal(1000) * 1e30]).astype(np.float32)
    # fp32 values with every low-16-bit pattern near a tie
    ties = (np.arange(4096, dtype=np.uint32) << 4 | 0x3F808000).view(np.float32)
    r = np.concatenate([r, ties, -ties])
    lib = torch.from_numpy(r).to(torch.bfloat16).float().numpy().astype(np.float64)
    assert np.array_equal(L.bf16_round(r.astype(np.float64)), lib)


def _outlier_matrix(n=400, seed=5):
    rng = np.random.default_rng(seed)
    lam = np.concatenate([rng.uniform(-1, 1, n - 1), [10.0]])
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return (U * lam) @ U.T


def test_window_orthogonality_band():
    """Window r: q_{k+1} is orthogonal (to fp64 round-off) to the r vectors it was
    orthogonalised against, i.e. |q_i . q_j| ~ u for |i - j| <= r; outside the band
    orthogonality is lost after the outlier converges (Paige), as with no reorthogonalisation."""
    H = _outlier_matrix()
    q1 = probe.rademacher_probe(7, H.shape[0])
    for r_ in (2, 4, 8):
        res = L.lanczos(lambda q: H @ q, q1, 60, "window", window=r_, keep_basis=True)
        Q = res.basis
        G = np.abs(Q @ Q.T - np.eye(len(Q)))
        i, j = np.indices(G.shape)
        assert G[np.abs(i - j) <= r_].max() < 1e-13
        assert G[np.abs(i - j) > r_].max() > 1e-2


def test_window_covering_all_steps_is_full():
    H = _outlier_matrix(120, 2)
    q1 = probe.rademacher_probe(3, 120)
    a = L.lanczos(lambda q: H @ q, q1, 40, "window", window=40)
    b = L.lanczos(lambda q: H @ q, q1, 40, "full")
    assert np.array_equal(a.alpha, b.alpha) and np.array_equal(a.beta, b.beta)


def test_bf16_basis_vectors_are_stored_rounded():
    """Every stored Lanczos vector is exactly bf16-representable, and alpha_k is the Rayleigh
    quotient of the STORED vector with the recurrence of P:309-311 (brute force, dense H)."""
    H = _outlier_matrix(64, 4)
    q1 = probe.rademacher_probe(9, 64)
    res = L.lanczos(lambda q: H @ q, q1, 10, "full", basis="bf16", keep_basis=True)
    Q = res.basis
    assert np.array_equal(L.bf16_round(Q), Q)
    # step 1: alpha_1 = q1^T H q1 with q1 = bf16(s / sqrt(P))
    q1s = L.bf16_round(q1)
    assert abs(res.alpha[0] - q1s @ H @ q1s) <= 1e-14 * np.abs(H).max()
    # step 2: w = H q2 - beta_2 q1 (the stored q1, q2); alpha_2 = <w, q2>
    w = H @ Q[1] - res.beta[0] * Q[0]
    assert abs(res.alpha[1] - w @ Q[1]) <= 1e-14 * np.abs(H).max()


def test_ghost_clusters_spec_examples():
    """full reorth, fp64, exact matvec on diag(1..100), m = 60 -> no duplicate clusters;
    no reorth, m = 60 on a matrix with one dominant outlier (gap 10x) -> a duplicate cluster at
    the outlier (Paige); tol = 0 -> no clusters (an unreduced T_m has distinct eigenvalues)."""
    D = np.arange(1.0, 101.0)
    r = L.lanczos(lambda q: D * q, probe.rademacher_probe(1, 100), 60, "full")
    nodes, _ = L.gauss_quadrature(r.alpha, r.beta)
    _, g = L.ghost_clusters(nodes, 1e-6 * np.abs(nodes).max())
    assert g == []

    H = _outlier_matrix()
    q1 = probe.rademacher_probe(7, H.shape[0])
    r = L.lanczos(lambda q: H @ q, q1, 60, "none")
    nodes, _ = L.gauss_quadrature(r.alpha, r.beta)
    _, g = L.ghost_clusters(nodes, 1e-6 * np.abs(nodes).max())
    assert any(abs(nodes[i] - 10.0) < 1e-6 and size >= 2 for i, size, _ in g)
    _, g0 = L.ghost_clusters(nodes, 0.0)
    assert g0 == []
    # bf16 basis, no reorth: the ghost copies are split by the storage noise (Theorem 3's
    # splitting grows with the matvec/storage error): a cluster at the outlier at a
    # tolerance of a few bf16 ulps of ||H||
    r = L.lanczos(lambda q: H @ q, q1, 60, "none", basis="bf16")
    nodes, _ = L.gauss_quadrature(r.alpha, r.beta)
    _, g = L.ghost_clusters(nodes, 2e-3 * np.abs(nodes).max())
    assert any(abs(nodes[i] - 10.0) < 0.1 and size >= 2 for i, size, _ in g)
    # full reorth keeps a single copy of the outlier even with a bf16 basis
    r = L.lanczos(lambda q: H @ q, q1, 60, "full", basis="bf16")
    nodes, _ = L.gauss_quadrature(r.alpha, r.beta)
    assert np.sum(np.abs(nodes - 10.0) < 0.5) == 1


def test_bf16_basis_claim_on_c1():
    """The paper's claim: a bf16 Lanczos basis with full reorthogonalisation keeps
    the spectrum; on c1 (FD-HVP, eps = 1e-3, m = 32) the extreme Ritz values move by <= 1e-3
    relative and the first two moments by <= 1e-2 (the bf16-model gates of the north star)."""
    cfg = si.CONFIGS["c1"]
    th = si.init_params(cfg)
    data = si.mlp_data(cfg)
    g = fdhvp.make_grad_fn(cfg, data)
    q1 = probe.rademacher_probe(cfg.probe_seed0, th.size)
    op = lambda q: fdhvp.fd_hvp_step(g, th, q, cfg.eps, "exact")  # noqa: E731
    a = L.lanczos(op, q1, 32, "full")
    b = L.lanczos(op, q1, 32, "full", basis="bf16")
    na, wa = L.gauss_quadrature(a.alpha, a.beta)
    nb, wb = L.gauss_quadrature(b.alpha, b.beta)
    scale = max(abs(na[0]), abs(na[-1]))
    assert abs(na[-1] - nb[-1]) / scale <= 1e-3 and abs(na[0] - nb[0]) / scale <= 1e-3
    mu1a, mu1b = L.moment(na, wa, 1), L.moment(nb, wb, 1)
    mu2a, mu2b = L.moment(na, wa, 2), L.moment(nb, wb, 2)
    assert abs(mu1a - mu1b) / np.sqrt(mu2a) <= 1e-2 and abs(mu2a - mu2b) / mu2a <= 1e-2
