"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle on the same seeded inputs.

Tolerances are the north star's (BASELINE.json): fp32 models -> HVP relative L2 <= 1e-4 and
alpha/beta <= 1e-5 relative for the first 32 Lanczos steps.  The GPU runs its gradient passes in
fp64 for these fp32 models; perturbed points are fp32 on both sides
(single-rounding fmaf), so the two sides differ only by fp64 summation order and the fp32
storage of the Lanczos vectors.
"""
import numpy as np
import pytest

import slq_inputs as si

from . import oracle_cache as OC
from oracle import fdhvp, lanczos as OL, models, probe

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_00816_b200 import build
    build.build()


from paper_2602_00816_b200 import slq  # noqa: E402


def _batch(cfg):
    return si.mlp_data(cfg) if cfg.arch == si.ARCH_MLP else si.tokens(cfg)


def _ctx(cfg, **kw):
    return slq.SlqContext(cfg, si.init_params(cfg), _batch(cfg), **kw)


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def _to_dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


SMALL = ["mlp_tiny", "c1", "gpt_tiny", "gpt_tiny_tied", "llama_tiny"]


@pytest.mark.parametrize("name", SMALL + ["c2"])
def test_probe_bit_exact(name):
    cfg = si.CONFIGS[name]
    with _ctx(cfg) as c:
        lay = c.layout()
        q = torch.empty(c.P_loc, dtype=torch.float32, device="cuda")
        c.probe(cfg.probe_seed0, q)
        ref = slq.shard_of(probe.rademacher_probe(cfg.probe_seed0, c.P).astype(np.float32), lay, 0, 1)
        assert np.array_equal(q.cpu().numpy(), ref)


@pytest.mark.parametrize("name", SMALL)
def test_grad_parity(name):
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    with _ctx(cfg) as c:
        g = torch.empty(c.P_loc, dtype=torch.float32, device="cuda")
        loss = c.grad(g)
        full = slq.unshard([g.cpu().numpy()], c.layout())
    l_ref, g_ref = models.loss_grad(th, cfg, _batch(cfg))
    assert abs(loss - l_ref) <= 1e-12 * abs(l_ref)
    assert _rel(full, g_ref) <= 1e-7  # fp64 passes, fp32 output rounding


ORACLE_MODE = {"exact": "exact", "storage": "param_dtype"}


@pytest.mark.parametrize("mode", ["exact", "storage"])
@pytest.mark.parametrize("name", SMALL + ["c2"])
def test_hvp_parity(name, mode):
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    v = si.random_vector(th.size, 5)
    with _ctx(cfg, perturb=mode) as c:
        lay = c.layout()
        vd = _to_dev(slq.shard_of(v, lay, 0, 1))
        out = torch.empty_like(vd)
        c.hvp(vd, out, cfg.eps)
        hv = slq.unshard([out.cpu().numpy()], lay)
        pad = out.cpu().numpy()
    ref = fdhvp.hvp(fdhvp.make_grad_fn(cfg, _batch(cfg)), th, v, cfg.eps, ORACLE_MODE[mode])
    err = _rel(hv, ref)
    print(f"{name} [{mode}]: HVP rel-L2 vs oracle = {err:.3e}")
    assert err <= 1e-4
    # padding entries are returned as zero
    mask = np.ones(lay["P_loc"], bool)
    for g, numel, loc, chunk in lay["units"]:
        mask[loc:loc + numel] = False
    assert np.all(pad[mask] == 0)


def test_hvp_host_pointers_and_edge_cases():
    cfg = si.CONFIGS["gpt_tiny"]
    th = si.init_params(cfg)
    with _ctx(cfg) as c:
        lay = c.layout()
        v = slq.shard_of(si.random_vector(th.size, 9), lay, 0, 1)
        out_h = np.empty_like(v)
        c.hvp(v, out_h, 1e-3)                        # host in / host out
        vd = _to_dev(v)
        out_d = torch.empty_like(vd)
        c.hvp(vd, out_d, 1e-3)                       # device in / device out
        assert np.array_equal(out_h, out_d.cpu().numpy())
        c.hvp(vd * 3.0, out_d, 1e-3)                 # scaling: eta = eps/||v|| keeps the step
        assert _rel(out_d.cpu().numpy(), 3 * out_h) < 1e-4
        z = torch.zeros_like(vd)
        c.hvp(z, out_d, 1e-3)                        # v = 0 -> 0
        assert torch.count_nonzero(out_d).item() == 0
        g0 = torch.empty_like(vd)
        g1 = torch.empty_like(vd)
        c.grad(g0)
        c.hvp(vd, out_d, 1e-3)
        c.grad(g1)                                   # theta bit-identical after an HVP
        assert torch.equal(g0, g1)
        with pytest.raises(slq.SlqError):
            c.hvp(vd, vd, 1e-3)                      # aliasing rejected
        with pytest.raises(slq.SlqError):
            c.hvp(vd, out_d, 0.0)
        assert c.launch_count() > 0


def _oracle_lanczos(cfg, m, reorth, mode="exact"):
    if mode == "exact":
        return OC.lanczos_exact(cfg.name, m, reorth)
    th = si.init_params(cfg)
    g = fdhvp.make_grad_fn(cfg, _batch(cfg))
    q1 = probe.rademacher_probe(cfg.probe_seed0, th.size)
    if mode == "exact":
        op = lambda q: fdhvp.fd_hvp_step(g, th, q, cfg.eps, "exact")
    else:
        op = lambda q: fdhvp.fd_hvp_step(g, th, q.astype(np.float32), cfg.eps, "param_dtype")
    return OL.lanczos(op, q1, m, reorth)


def _ab_rel(a, ref):
    return np.abs(np.asarray(a) - ref) / np.abs(ref)


@pytest.mark.parametrize("name,m", [("c1", 32), ("mlp_tiny", 8), ("gpt_tiny", 16), ("llama_tiny", 16),
                                    ("gpt_tiny_tied", 12), ("c2", 32)])
def test_lanczos_parity_full_reorth(name, m):
    cfg = si.CONFIGS[name]
    with _ctx(cfg, reorth="full", max_steps=m) as c:
        a, b = c.lanczos(cfg.probe_seed0, m)
        info = c.lanczos_info()
    r = _oracle_lanczos(cfg, m, "full")
    md = min(r.m_done, info["m_done"])
    assert md == r.m_done
    ea = _ab_rel(a[:md], r.alpha[:md])
    eb = _ab_rel(b[:md - 1], r.beta[:md - 1])
    print(f"{name}: max rel alpha {ea.max():.2e}  beta {eb.max() if eb.size else 0:.2e}")
    # alpha can pass near zero; the relative gate is applied against the spectral scale there
    scale = np.abs(r.alpha).max()
    assert np.all(np.abs(a[:md] - r.alpha[:md]) <= 1e-5 * np.maximum(np.abs(r.alpha[:md]), 1e-2 * scale))
    assert np.all(eb <= 1e-5)
    # quadrature of the GPU T_m against the oracle's: nodes and weights
    n1, w1 = slq.quadrature(a[:md], b[:md - 1])
    n2, w2 = OL.gauss_quadrature(r.alpha, r.beta)
    assert abs(n1[0] - n2[0]) <= 1e-5 * scale and abs(n1[-1] - n2[-1]) <= 1e-5 * scale
    assert abs(w1.sum() - 1) < 1e-12


def test_lanczos_storage_mode_early_steps():
    """STORAGE perturbation makes the FD operator depend on the last fp32 bit of q_k (each
    rounding flip of fl32(theta + eps q) moves Hv by ~H e_i ulp/(2 eps)); the GPU's fp32 q_k and
    the oracle's fp64 q_k differ in those bits, so agreement holds for the first steps only
    (reading R9)."""
    cfg = si.CONFIGS["c1"]
    m = 8
    with _ctx(cfg, reorth="full", max_steps=m, perturb="storage") as c:
        a, b = c.lanczos(cfg.probe_seed0, m)
    r = _oracle_lanczos(cfg, m, "full", mode="storage")
    assert np.all(_ab_rel(a[:4], r.alpha[:4]) <= 1e-5)
    assert np.all(_ab_rel(b[:3], r.beta[:3]) <= 1e-5)


def test_lanczos_no_reorth_first_steps():
    """Three-term recurrence without a basis (c5 mode): early steps agree before Paige-type
    loss of orthogonality amplifies fp32-vs-fp64 differences."""
    cfg = si.CONFIGS["gpt_tiny"]
    m = 8
    with _ctx(cfg, reorth="none", max_steps=m) as c:
        a, b = c.lanczos(cfg.probe_seed0, m)
    r = _oracle_lanczos(cfg, m, "none")
    assert np.all(_ab_rel(a[:6], r.alpha[:6]) <= 1e-5)
    assert np.all(_ab_rel(b[:5], r.beta[:5]) <= 1e-5)


def test_fp32_pass_mode_reported():
    """fp32 gradient passes run, and land at Theorem 1's round-off floor (~1e-3), not at 1e-4."""
    cfg = si.CONFIGS["c1"]
    th = si.init_params(cfg)
    v = si.random_vector(th.size, 5)
    with _ctx(cfg, pass_numerics="fp32") as c:
        lay = c.layout()
        vd = _to_dev(slq.shard_of(v, lay, 0, 1))
        out = torch.empty_like(vd)
        c.hvp(vd, out, cfg.eps)
        hv = slq.unshard([out.cpu().numpy()], lay)
    ref = fdhvp.hvp(fdhvp.make_grad_fn(cfg, _batch(cfg)), th, v, cfg.eps, "param_dtype")
    err = _rel(hv, ref)
    print(f"c1 fp32-pass HVP rel-L2 = {err:.3e}")
    assert err < 5e-2


def test_lanczos_breakdown_detected_post_hoc():
    """mlp_tiny has P = 112 parameters and an invariant Krylov subspace of dimension 103 from its
    probe (fp64 oracle: beta_104 ~ 4e-13).  Asked for P + 10 steps, the GPU recurrence (device-
    resident scalars, breakdown detected after the loop) must stop at the invariant subspace:
    m_done within a few steps of the oracle's, unfilled entries NaN, and the Ritz values of the
    computed T an invariant set (extremes agree with the oracle's)."""
    cfg = si.CONFIGS["mlp_tiny"]
    th = si.init_params(cfg)
    P = th.size
    m = P + 10
    with _ctx(cfg, reorth="full", max_steps=m) as c:
        a, b = c.lanczos(cfg.probe_seed0, m)
        info = c.lanczos_info()
    r = _oracle_lanczos(cfg, m, "full")
    md = info["m_done"]
    print(f"mlp_tiny breakdown: GPU m_done {md}, oracle {r.m_done}, beta_next {info['beta_next']:.2e}")
    assert r.breakdown and abs(md - r.m_done) <= 3 and md <= P
    assert np.all(np.isnan(a[md:])) and np.all(np.isnan(b[md - 1:]))
    assert np.all(np.isfinite(a[:md])) and np.all(np.isfinite(b[:md - 1]))
    n1, w1 = slq.quadrature(a[:md], b[:md - 1])
    n2, _ = OL.gauss_quadrature(r.alpha, r.beta)
    scale = max(abs(n2[0]), abs(n2[-1]))
    assert abs(n1[0] - n2[0]) <= 1e-5 * scale and abs(n1[-1] - n2[-1]) <= 1e-5 * scale
    assert abs(w1.sum() - 1) < 1e-12


def test_slq_probe_loop_and_density():
    """slq_slq runs the probe loop of SLQ: every probe equals its own slq_lanczos call
    bit for bit, and the probe-averaged moments of the GPU node sets match the oracle's SLQ on the
    same probes (mu_0 = 1, mu_1 and mu_2 within the fp32 gates)."""
    cfg = si.CONFIGS["gpt_tiny"]
    m, seeds = 8, [cfg.probe_seed0 + j for j in range(3)]
    with _ctx(cfg, reorth="full", max_steps=m) as c:
        A, B, md = c.slq(seeds, m)
        single = [c.lanczos(sd, m) for sd in seeds]
    for p in range(3):
        assert md[p] == m
        assert np.array_equal(A[p], single[p][0]) and np.array_equal(B[p], single[p][1])
    th = si.init_params(cfg)
    g = fdhvp.make_grad_fn(cfg, _batch(cfg))
    ns, ws, rn, rw = [], [], [], []
    for p, sd in enumerate(seeds):
        n, w = slq.quadrature(A[p], B[p])
        ns.append(n); ws.append(w)
        r = OL.lanczos(lambda q: fdhvp.fd_hvp_step(g, th, q, cfg.eps, "exact"), probe.rademacher_probe(sd, th.size),
                       m, "full")
        n2, w2 = OL.gauss_quadrature(r.alpha, r.beta)
        rn.append(n2); rw.append(w2)
    mom, _ = slq.density(ns, ws, jmax=2)
    ref = OL.slq_moments(rn, rw, jmax=2)
    print(f"gpt_tiny SLQ moments {mom} vs {ref}")
    assert abs(mom[0] - 1) < 1e-12
    assert abs(mom[1] - ref[1]) <= 1e-5 * np.sqrt(ref[2]) and abs(mom[2] - ref[2]) <= 1e-5 * ref[2]


def test_error_codes():
    """Documented failure modes (include/slq.h): bad arguments -> SLQ_EINVAL, a non-finite
    direction -> SLQ_ENUMERIC; the context stays usable afterwards."""
    cfg = si.CONFIGS["gpt_tiny"]
    with _ctx(cfg, reorth="full", max_steps=4) as c:
        v = torch.zeros(c.P_loc, dtype=torch.float32, device="cuda")
        out = torch.empty_like(v)
        for bad in (lambda: c.lanczos(cfg.probe_seed0, 0), lambda: c.lanczos(cfg.probe_seed0, 5),
                    lambda: c.hvp(v, out, -1.0), lambda: c.cg(v, v, 0.1, 3)):
            with pytest.raises(slq.SlqError) as e:
                bad()
            assert e.value.status == slq.SLQ_EINVAL
        v[3] = float("nan")
        with pytest.raises(slq.SlqError) as e:
            c.hvp(v, out, 1e-3)
        assert e.value.status == slq.SLQ_ENUMERIC
        assert c.nonfinite_seq() == -1  # rejected before any pass ran
        a, b = c.lanczos(cfg.probe_seed0, 4)  # still usable
        assert np.all(np.isfinite(a)) and np.all(np.isfinite(b))


@pytest.mark.parametrize("row", [0, 5, 255])
def test_nonfinite_gradient_names_the_batch(row):
    """a non-finite gradient is an error "carrying the offending batch id": with one data
    row of c1's MLP batch set to inf, slq_hvp returns SLQ_ENUMERIC and slq_nonfinite_seq names that
    row."""
    cfg = si.CONFIGS["mlp_tiny"] if row < si.CONFIGS["mlp_tiny"].n_rows else si.CONFIGS["c1"]
    x, y = si.mlp_data(cfg)
    x = x.copy()
    x[row, :] = np.inf
    th = si.init_params(cfg)
    with slq.SlqContext(cfg, th, (x, y), max_steps=4) as c:
        v = _to_dev(slq.shard_of(si.random_vector(th.size, 3), c.layout(), 0, 1))
        out = torch.empty_like(v)
        with pytest.raises(slq.SlqError) as e:
            c.hvp(v, out, cfg.eps)
        assert e.value.status == slq.SLQ_ENUMERIC
        assert c.nonfinite_seq() == row
        assert f"local sequence {row}" in str(e.value)
