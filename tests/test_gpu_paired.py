"""Paired (mean, half-difference) evaluation of Eq. (1) on the GPU.

GPT and Llama.  One pass carries both gradient evaluations as pairs, so g+ - g- is never formed from rounded
gradients; with fp32-faithful arithmetic (tcgen05 three-term splits, or fp32 SIMT) it must meet
the FP32 gates of the north star against the fp64 oracle (exact perturbed points): HVP relative
L2 <= 1e-4 and alpha/beta <= 1e-5 over the first 32 Lanczos steps.
"""
import numpy as np
import pytest

import slq_inputs as si
from oracle import fdhvp, lanczos as OL, models, probe

from . import oracle_cache as OC

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_00816_b200 import build
    build.build()


from paper_2602_00816_b200 import slq  # noqa: E402

MODES = ["paired", "paired_fp32"]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", ["gpt_tiny", "gpt_tiny_tied", "llama_tiny", "c2"])
def test_paired_grad_and_hvp(name, mode):
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    tok = si.tokens(cfg)
    v = si.random_vector(th.size, 5)
    with slq.SlqContext(cfg, th, tok, pass_numerics=mode) as c:
        lay = c.layout()
        g = torch.empty(c.P_loc, dtype=torch.float32, device="cuda")
        loss = c.grad(g)
        gfull = slq.unshard([g.cpu().numpy()], lay)
        vd = torch.from_numpy(slq.shard_of(v, lay, 0, 1)).cuda()
        out = torch.empty_like(vd)
        c.hvp(vd, out, cfg.eps)
        hv = slq.unshard([out.cpu().numpy()], lay)
    l_ref, g_ref = OC.loss_grad(name)
    ref = OC.hvp_exact(name, 5)
    eg = np.linalg.norm(gfull - g_ref) / np.linalg.norm(g_ref)
    eh = np.linalg.norm(hv - ref) / np.linalg.norm(ref)
    print(f"{name} [{mode}]: loss {abs(loss - l_ref) / abs(l_ref):.1e} grad {eg:.2e} HVP {eh:.2e}")
    assert abs(loss - l_ref) <= 1e-6 * abs(l_ref)
    assert eg <= 2e-5
    assert eh <= 1e-4


PAIRED_TC_XFAIL = pytest.mark.xfail(
    strict=False, raises=AssertionError,
    reason="SLQ_PASS_PAIRED (tcgen05 three-term bf16 splits, fp32 TMEM accumulation) misses the north star's "
           "fp32 alpha/beta gate: B200, c2 m=32: alpha 8.8e-4 (reading R14), beta 2.1e-5 -- its HVP (1.3e-5) "
           "meets the 1e-4 HVP gate and the bf16-model gates (c3: extreme Ritz 2.2e-4, mu2 4.5e-4), not "
           "alpha/beta <= 1e-5")
PAIRED_FP32_C2_XFAIL = pytest.mark.xfail(
    strict=False, raises=AssertionError,
    reason="SLQ_PASS_PAIRED_FP32 (fp32 SIMT pair GEMMs) on c2 at m=32: B200 round 2 measured alpha 4.2e-5 "
           "(reading R14; 4.0e-6 of the spectral scale), beta 3.4e-7 -- the fp32 alpha gate (1e-5) is missed at "
           "the alpha_k that pass near zero; gpt_tiny and llama_tiny meet it")


def _mode_param(mode, name):
    if mode == "paired":
        return pytest.param(mode, name, marks=PAIRED_TC_XFAIL)
    if name == "c2":
        return pytest.param(mode, name, marks=PAIRED_FP32_C2_XFAIL)
    return pytest.param(mode, name)


@pytest.mark.parametrize("mode,name", [_mode_param(mo, na) for mo in MODES for na in ("gpt_tiny", "llama_tiny", "c2")])
def test_paired_lanczos_fp32_gates(name, mode):
    """The north star's fp32 gates as every fp32-model mode is held to them: alpha per reading R14
    and beta <= 1e-5 relative over the first 32 steps."""
    m = 32 if name == "c2" else 16
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    tok = si.tokens(cfg)
    with slq.SlqContext(cfg, th, tok, pass_numerics=mode, reorth="full", max_steps=m) as c:
        a, b = c.lanczos(cfg.probe_seed0, m)
    r = OC.lanczos_exact(name, m, "full")
    scale = np.abs(r.alpha).max()
    ea = np.abs(a - r.alpha) / np.maximum(np.abs(r.alpha), 1e-2 * scale)  # reading R14
    es = np.abs(a - r.alpha) / scale                                       # relative to the spectral scale
    eb = np.abs(b - r.beta) / np.abs(r.beta)
    print(f"{name} [{mode}]: max rel alpha {ea.max():.2e} (vs spectral scale {es.max():.2e}) beta {eb.max():.2e}")
    assert ea.max() <= 1e-5 and eb.max() <= 1e-5
