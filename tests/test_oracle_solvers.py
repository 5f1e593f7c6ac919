"""Pins for the oracle's NEXT-row solvers: CG inverse-HVP (§8(f2)) and the block-diagonal test
(§8(f4)) -- closed forms and brute force on tiny inputs (CPU only)."""
import numpy as np

import slq_inputs as si
from oracle import blockdiag as BD, cg as CG, fdhvp, models


def _spd(n, seed, lo=1.0, hi=20.0):
    q, _ = np.linalg.qr(np.random.default_rng(seed).standard_normal((n, n)))
    return q @ np.diag(np.linspace(lo, hi, n)) @ q.T


def test_cg_quadratic_exact_in_n_steps():
    A = _spd(40, 1)
    b = np.random.default_rng(2).standard_normal(40)
    lam = 0.3
    x, it, hist = CG.cg(lambda p: A @ p, b, lam, 40, tol=1e-14)
    ref = np.linalg.solve(A + lam * np.eye(40), b)
    assert np.linalg.norm(x - ref) <= 1e-9 * np.linalg.norm(ref)
    assert it <= 40 and hist[-1] <= 1e-12


def _dense_fd_hessian(d, th, batch, step=1e-4):
    g = fdhvp.make_grad_fn(d, batch)
    P = th.size
    H = np.empty((P, P))
    e = np.zeros(P)
    for i in range(P):
        e[i] = 1.0
        H[:, i] = fdhvp.fd_hvp_step(g, th, e, step, "exact")
        e[i] = 0.0
    return (H + H.T) / 2


def test_cg_on_fd_operator_matches_dense_solve():
    d = si.CONFIGS["mlp_tiny"]
    th = si.init_params(d)
    b_ = si.mlp_data(d)
    H = _dense_fd_hessian(d, th, b_)
    lam = abs(np.linalg.eigvalsh(H)[0]) + 0.1
    rhs = np.random.default_rng(3).standard_normal(th.size)
    g = fdhvp.make_grad_fn(d, b_)
    x, it, hist = CG.cg(lambda p: fdhvp.hvp(g, th, p, 1e-4, "exact"), rhs, lam, th.size, tol=1e-10)
    ref = np.linalg.solve(H + lam * np.eye(th.size), rhs)
    assert np.linalg.norm(x - ref) <= 1e-5 * np.linalg.norm(ref)


def test_blockdiag_special_cases():
    A1, A2 = _spd(10, 4), _spd(7, 5)
    A = np.zeros((17, 17))
    A[:10, :10], A[10:, 10:] = A1, A2
    v = np.random.default_rng(6).standard_normal(17)
    v /= np.linalg.norm(v)
    rel, cos = BD.block_test(lambda x: A @ x, v, [(0, 10), (10, 17)])
    assert np.all(rel <= 1e-14) and np.all(np.abs(cos - 1) <= 1e-14)
    # dense matrix: brute force with explicit block slices
    B = np.random.default_rng(7).standard_normal((17, 17))
    B = B + B.T
    rel, cos = BD.block_test(lambda x: B @ x, v, [(0, 10), (10, 17)])
    for k, (s, e) in enumerate([(0, 10), (10, 17)]):
        full = (B @ v)[s:e]
        diag = B[s:e, s:e] @ v[s:e]
        assert abs(rel[k] - np.linalg.norm(full - diag) / np.linalg.norm(full)) < 1e-12
        assert abs(cos[k] - full @ diag / np.linalg.norm(full) / np.linalg.norm(diag)) < 1e-12


def test_blockdiag_mlp_layers_vs_dense_hessian():
    d = si.CONFIGS["mlp_tiny"]
    th = si.init_params(d)
    b_ = si.mlp_data(d)
    H = _dense_fd_hessian(d, th, b_)
    n1 = d.d_hidden * d.d_in + d.d_hidden
    blocks = [(0, n1), (n1, th.size)]
    v = np.random.default_rng(8).standard_normal(th.size)
    v /= np.linalg.norm(v)
    g = fdhvp.make_grad_fn(d, b_)
    rel, cos = BD.block_test(lambda x: fdhvp.hvp(g, th, x, 1e-4, "exact"), v, blocks)
    for k, (s, e) in enumerate(blocks):
        full = (H @ v)[s:e]
        diag = H[s:e, s:e] @ v[s:e]
        assert abs(rel[k] - np.linalg.norm(full - diag) / np.linalg.norm(full)) < 1e-5
        assert abs(cos[k] - full @ diag / np.linalg.norm(full) / np.linalg.norm(diag)) < 1e-5
    assert np.all(rel > 1e-3)  # an MLP's Hessian is not block diagonal across layers
