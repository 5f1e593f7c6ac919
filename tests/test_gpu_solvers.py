"""GPU parity of the NEXT-row solvers on the FD-HVP primitive: CG inverse-HVP (§8(f2)) and the
block-diagonal hypothesis test (§8(f4)), against the oracle on the same seeded inputs."""
import numpy as np
import pytest

import slq_inputs as si
from oracle import blockdiag as BD, cg as CG, fdhvp, lanczos as OL, probe

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


@pytest.mark.parametrize("name", ["c1", "gpt_tiny", "llama_tiny"])
def test_cg_parity(name):
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    g = fdhvp.make_grad_fn(cfg, _batch(cfg))
    op = lambda q: fdhvp.hvp(g, th, q, cfg.eps, "exact")
    r = OL.lanczos(op, probe.rademacher_probe(cfg.probe_seed0, th.size), 12, "full")
    lam = 1.5 * abs(min(np.linalg.eigvalsh(OL.tridiag(r.alpha, r.beta))[0], 0.0)) + 0.05
    rhs = si.random_vector(th.size, 21)
    iters = 8
    x_ref, _, hist = CG.cg(op, rhs, lam, iters)
    with slq.SlqContext(cfg, th, _batch(cfg)) as c:
        lay = c.layout()
        b = torch.from_numpy(slq.shard_of(rhs, lay, 0, 1)).cuda()
        x = torch.empty_like(b)
        it, rr = c.cg(b, x, lam, iters, 0.0)
        xg = slq.unshard([x.cpu().numpy()], lay)
    err = np.linalg.norm(xg - x_ref) / np.linalg.norm(x_ref)
    print(f"{name}: damping {lam:.3f} iters {it} residual {rr:.3e} (oracle {hist[-1]:.3e}) x rel err {err:.2e}")
    assert it == iters
    assert abs(rr - hist[-1]) <= 1e-3 * hist[0] + 1e-3 * hist[-1]
    assert err <= 1e-4


@pytest.mark.parametrize("name", ["gpt_tiny", "llama_tiny", "c1"])
def test_blockdiag_parity(name):
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    with slq.SlqContext(cfg, th, _batch(cfg)) as c:
        units = c.layout()["units"]
        rel, cos = c.blockdiag(cfg.probe_seed0)
    g = fdhvp.make_grad_fn(cfg, _batch(cfg))
    v = probe.rademacher_probe(cfg.probe_seed0, th.size)
    blocks = [(int(u[0]), int(u[0] + u[1])) for u in units]
    rel_ref, cos_ref = BD.block_test(lambda q: fdhvp.hvp(g, th, q, cfg.eps, "exact"), v, blocks)
    print(f"{name}: rel {np.round(rel, 4)} cos {np.round(cos, 4)}")
    assert np.max(np.abs(rel - rel_ref)) <= 1e-5 * max(1.0, np.max(rel_ref))
    assert np.max(np.abs(cos - cos_ref)) <= 1e-5
