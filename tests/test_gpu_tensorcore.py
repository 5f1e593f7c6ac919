"""tcgen05 tensor-core paths on the GPU.

* the bf16 tcgen05 GEMM (TMA + TMEM + mbarrier pipeline) against a reference kernel;
* the BF16X3 pass mode (fp32 activations, every non-batched GEMM on tcgen05 with three-term bf16
  operand splits) against the oracle: it sits at the fp32-pass floor of Theorem 1 (~1e-3 HVP,
  P:120-128), inside the north star's bf16-model gates (moments <= 1e-2, extreme Ritz <= 2e-2).
"""
import ctypes

import numpy as np
import pytest

import slq_inputs as si

from . import oracle_cache as OC
from oracle import fdhvp, lanczos as OL, probe

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_00816_b200 import build
    build.build()


from paper_2602_00816_b200 import slq  # noqa: E402


@pytest.mark.parametrize("shape", [(256, 256, 128, 0), (512, 384, 320, 0), (1000, 1000, 1000, 0),
                                   (2048, 4096, 256, 1), (129, 200, 72, 0)])
def test_tcgen05_bf16_gemm_matches_reference(shape):
    M, N, K, v = shape
    f = slq.lib().slq_diag_gemm_bf16
    f.restype = ctypes.c_int32
    f.argtypes = [ctypes.c_int32] * 6 + [ctypes.c_void_p, ctypes.c_void_p]
    t, e = ctypes.c_double(), ctypes.c_double()
    assert f(0, M, N, K, v, 2, ctypes.byref(t), ctypes.byref(e)) == 0
    assert e.value < 1e-5, e.value  # fp32 accumulation of exact bf16 products


def _batch(cfg):
    return si.mlp_data(cfg) if cfg.arch == si.ARCH_MLP else si.tokens(cfg)


@pytest.mark.parametrize("name", ["mlp_tiny", "c1", "gpt_tiny", "gpt_tiny_tied", "llama_tiny"])
def test_bf16x3_grad_is_fp32_faithful(name):
    """The BF16X3 gradient matches the fp64 oracle gradient to fp32-level accuracy."""
    from oracle import models
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    with slq.SlqContext(cfg, th, _batch(cfg), pass_numerics="bf16x3") as c:
        g = torch.empty(c.P_loc, dtype=torch.float32, device="cuda")
        c.grad(g)
        full = slq.unshard([g.cpu().numpy()], c.layout())
    ref = models.loss_grad(th, cfg, _batch(cfg))[1]
    err = np.linalg.norm(full - ref) / np.linalg.norm(ref)
    print(f"{name}: bf16x3 grad rel err {err:.2e}")
    assert err < 2e-5


@pytest.mark.parametrize("name", ["c1", "gpt_tiny", "llama_tiny", "c2"])
def test_bf16x3_hvp_and_moments_within_bf16_gates(name):
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    m = 4
    with slq.SlqContext(cfg, th, _batch(cfg), pass_numerics="bf16x3", reorth="full", max_steps=m) as c:
        a, b = c.lanczos(cfg.probe_seed0, m)
    r = OC.lanczos_exact(name, m, "full")
    mu = (a[0], a[0] ** 2 + b[0] ** 2)
    mu_ref = (r.alpha[0], r.alpha[0] ** 2 + r.beta[0] ** 2)
    n1, _ = OL.gauss_quadrature(a, b)
    n2, _ = OL.gauss_quadrature(r.alpha, r.beta)
    scale = max(abs(n2[0]), abs(n2[-1]))
    e1 = abs(mu[0] - mu_ref[0]) / np.sqrt(mu_ref[1])
    e2 = abs(mu[1] - mu_ref[1]) / mu_ref[1]
    er = max(abs(n1[0] - n2[0]), abs(n1[-1] - n2[-1])) / scale
    print(f"{name}: bf16x3 mu1 err {e1:.2e}, mu2 err {e2:.2e}, extreme Ritz err {er:.2e}")
    assert e1 <= 1e-2 and e2 <= 1e-2 and er <= 2e-2


@pytest.mark.parametrize("name", ["c1", "gpt_tiny", "llama_tiny", "c2"])
def test_native_bf16_pass_mode(name):
    """SLQ_PASS_BF16 ("BF16 native", SURVEY.md §8(a) numerics modes): the gradient carries bf16
    operand rounding -- relative error against the fp64 oracle between 1e-5 (it really is bf16:
    the fp32-faithful split reaches < 2e-5) and 3e-2 -- and the FD-HVP sits on Theorem 1's
    round-off floor, orders of magnitude above the BF16X3 split on the same probe."""
    from oracle import models
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    lay = None
    res = {}
    for mode in ("bf16", "bf16x3"):
        with slq.SlqContext(cfg, th, _batch(cfg), pass_numerics=mode) as c:
            lay = c.layout()
            g = torch.empty(c.P_loc, dtype=torch.float32, device="cuda")
            c.grad(g)
            v = torch.from_numpy(slq.shard_of(si.random_vector(th.size, 7), lay, 0, 1)).cuda()
            h = torch.empty_like(v)
            c.hvp(v, h, cfg.eps)
            res[mode] = (slq.unshard([g.cpu().numpy()], lay), slq.unshard([h.cpu().numpy()], lay))
    gref = models.loss_grad(th, cfg, _batch(cfg))[1]
    gfn = fdhvp.make_grad_fn(cfg, _batch(cfg))
    v = si.random_vector(th.size, 7)
    href = fdhvp.hvp(gfn, th, v, cfg.eps, "exact")
    eg = np.linalg.norm(res["bf16"][0] - gref) / np.linalg.norm(gref)
    eh = {k: np.linalg.norm(res[k][1] - href) / np.linalg.norm(href) for k in res}
    print(f"{name}: native bf16 grad rel err {eg:.2e}; HVP rel err bf16 {eh['bf16']:.2e} vs bf16x3 {eh['bf16x3']:.2e}")
    assert np.all(np.isfinite(res["bf16"][1]))
    assert 1e-5 < eg < 3e-2
    assert eh["bf16"] > 10 * eh["bf16x3"]
