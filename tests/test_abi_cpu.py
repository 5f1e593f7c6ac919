"""C-ABI checks that need no GPU: the library loads, exports every symbol include/slq.h declares,
the host-only calls (layout planner, quadrature) behave, and GPU calls fail loudly without a GPU."""
import math
import os
import re

import numpy as np
import pytest

import slq_inputs as si
from paper_2602_00816_b200 import slq

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2602_00816_b200 import build
    build.build()


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "slq.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(slq_[a-z_0-9]+)\s*\(", txt)))


def test_exports_every_declared_symbol():
    L = slq.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(L, n), n


def test_quadrature_chebyshev_and_legendre():
    for m in (1, 2, 7, 32, 100):
        beta = np.full(m - 1, 0.5)
        if m > 1:
            beta[0] = 1 / math.sqrt(2)
        nodes, w = slq.quadrature(np.zeros(m), beta)
        ref = np.sort(np.cos((2 * np.arange(1, m + 1) - 1) * math.pi / (2 * m)))
        assert np.max(np.abs(nodes - ref)) < 1e-13
        assert np.max(np.abs(w - 1.0 / m)) < 1e-13
    for m in (3, 20, 64):
        k = np.arange(1, m)
        nodes, w = slq.quadrature(np.zeros(m), k / np.sqrt(4 * k * k - 1.0))
        x, wl = np.polynomial.legendre.leggauss(m)
        assert np.max(np.abs(nodes - x)) < 1e-13 and np.max(np.abs(w - wl / 2)) < 1e-13


def test_quadrature_edge_cases_and_errors():
    n, w = slq.quadrature([3.25], [])
    assert n.tolist() == [3.25] and w.tolist() == [1.0]
    n, w = slq.quadrature([5.0, 2.0], [0.0])
    assert n.tolist() == [2.0, 5.0] and w.tolist() == [0.0, 1.0]
    with pytest.raises(slq.SlqError) as e:
        slq.quadrature([1.0, float("nan")], [0.5])
    assert e.value.status == slq.SLQ_EINVAL
    with pytest.raises(slq.SlqError):
        slq.quadrature([], [])


def test_quadrature_matches_oracle_jacobi():
    """Library implicit-shift QL vs the oracle's cyclic Jacobi on random T_m."""
    from oracle import lanczos as OL
    rng = np.random.default_rng(3)
    for m in (5, 16, 64):
        a = rng.standard_normal(m)
        b = np.abs(rng.standard_normal(m - 1)) + 0.01
        n1, w1 = slq.quadrature(a, b)
        n2, w2 = OL.gauss_quadrature(a, b)
        assert np.max(np.abs(n1 - n2)) < 1e-12 * max(1, np.abs(n2).max())
        assert np.max(np.abs(w1 - w2)) < 1e-10
        assert abs(w1.sum() - 1) < 1e-12


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5", "gpt_tiny", "gpt_tiny_tied", "llama_tiny"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_layout(name, world):
    cfg = si.CONFIGS[name]
    lay = slq.plan_layout(slq.make_desc(cfg), world)
    assert lay["P"] == si.n_params(cfg)
    u = lay["units"]
    # units tile the canonical order; chunks are multiples of 16 and cover numel
    assert u[0, 0] == 0 and np.all(u[1:, 0] == u[:-1, 0] + u[:-1, 1])
    assert np.all(u[:, 3] % 16 == 0) and np.all(u[:, 3] * world >= u[:, 1])
    assert np.all(u[:, 3] * world - u[:, 1] < 16 * world)
    assert lay["P_loc"] == u[:, 3].sum() and np.all(u[1:, 2] == u[:-1, 2] + u[:-1, 3])
    n_units = 1 if cfg.arch == si.ARCH_MLP else cfg.n_layers + 2
    assert len(u) == n_units


def test_shard_roundtrip():
    cfg = si.CONFIGS["gpt_tiny"]
    full = np.random.default_rng(0).standard_normal(si.n_params(cfg)).astype(np.float32)
    for world in (1, 2, 5):
        lay = slq.plan_layout(slq.make_desc(cfg), world)
        shards = [slq.shard_of(full, lay, r, world) for r in range(world)]
        assert np.array_equal(slq.unshard(shards, lay), full)
        # padding is zero, so shard-local dot products sum to the global one
        assert abs(sum(float(s.astype(np.float64) @ s) for s in shards) - float(full.astype(np.float64) @ full)) < 1e-6


def test_invalid_descriptor_rejected():
    cfg = si.get_config("gpt_tiny", n_heads=5)  # 64 % 5 != 0
    with pytest.raises(slq.SlqError) as e:
        slq.plan_layout(slq.make_desc(cfg), 1)
    assert e.value.status == slq.SLQ_EINVAL


def test_init_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg = si.CONFIGS["mlp_tiny"]
    with pytest.raises(slq.SlqError) as e:
        slq.SlqContext(cfg, si.init_params(cfg), si.mlp_data(cfg))
    assert e.value.status == slq.SLQ_ECUDA


def test_ghost_clusters_host_matches_oracle():
    """slq_ghost_clusters (host, R18) vs the oracle's definition on random node sets
    with planted duplicates, plus the tol = 0 and error cases."""
    from oracle import lanczos as OL
    rng = np.random.default_rng(3)
    for trial in range(50):
        x = np.sort(np.concatenate([rng.uniform(-5, 5, 30), np.repeat(rng.uniform(-5, 5, 3), 3) +
                                    rng.uniform(-1e-7, 1e-7, 9)]))
        for tol in (0.0, 1e-6, 1e-3, 0.3):
            ids, ng, ms = slq.ghost_clusters(x, tol)
            rid, rg = OL.ghost_clusters(x, tol)
            assert np.array_equal(ids, rid)
            assert ng == len(rg)
            assert ms == (max(s for _, _, s in rg) if rg else 0.0)
    ids, ng, ms = slq.ghost_clusters([1.0, 2.0, 3.0], 0.0)
    assert ids.tolist() == [0, 1, 2] and ng == 0 and ms == 0.0
    ids, ng, ms = slq.ghost_clusters([1.0, 1.0, 3.0], 0.0)
    assert ids.tolist() == [0, 0, 1] and ng == 1 and ms == 0.0
    for bad in (([2.0, 1.0], 0.1), ([1.0, float("nan")], 0.1), ([1.0, 2.0], -1.0)):
        with pytest.raises(slq.SlqError) as e:
            slq.ghost_clusters(*bad)
        assert e.value.status == slq.SLQ_EINVAL


def test_descriptor_validation_window_and_basis():
    """reorth WINDOW needs r >= 2; a bf16 basis needs a stored basis (host layout planner
    validates the descriptor without a GPU)."""
    cfg = si.CONFIGS["gpt_tiny"]
    for kw, ok in ((dict(reorth="window", window=1), False), (dict(reorth="window", window=4), True),
                   (dict(reorth="none", basis="bf16"), False), (dict(reorth="full", basis="bf16"), True),
                   (dict(reorth="window", window=3, basis="bf16"), True)):
        d = slq.make_desc(cfg, **kw)
        if ok:
            slq.plan_layout(d, 1)
        else:
            with pytest.raises(slq.SlqError) as e:
                slq.plan_layout(d, 1)
            assert e.value.status == slq.SLQ_EINVAL


def test_density_host_matches_oracle():
    """slq_density (host): probe-averaged moments and Gaussian-smoothed density vs the oracle's
    slq_moments / slq_density; mu_0 = 1 for weights summing to 1."""
    from oracle import lanczos as OL
    rng = np.random.default_rng(7)
    node_sets, weight_sets = [], []
    for m in (5, 9, 1):
        a = rng.standard_normal(m)
        b = np.abs(rng.standard_normal(m - 1)) + 0.1
        n, w = OL.gauss_quadrature(a, b)
        node_sets.append(n)
        weight_sets.append(w)
    grid = np.linspace(-4, 4, 41)
    mom, dens = slq.density(node_sets, weight_sets, jmax=4, grid=grid, sigma=0.3)
    ref_m = OL.slq_moments(node_sets, weight_sets, jmax=4)
    ref_d = OL.slq_density(grid, node_sets, weight_sets, 0.3)
    assert np.allclose(mom, ref_m, rtol=1e-13, atol=1e-14) and abs(mom[0] - 1) < 1e-13
    assert np.allclose(dens, ref_d, rtol=1e-13, atol=1e-15)
    mom2, d2 = slq.density(node_sets, weight_sets, jmax=1)
    assert d2 is None and np.allclose(mom2, ref_m[:2], rtol=1e-13)
    with pytest.raises(slq.SlqError):
        slq.density(node_sets, weight_sets, jmax=1, grid=grid, sigma=0.0)
