"""The int8 Ozaki fp64 GEMM on tcgen05 (SLQ_PASS_FP64_OZ; oz_gemm.cu) against the DMMA fp64 GEMM,
and the FP64_OZ pass mode against the fp64 oracle at the north star's fp32 gates (HVP rel-L2 <= 1e-4,
alpha/beta <= 1e-5 over the first 32 Lanczos steps).  Two routes, each a per-context descriptor
field (slq_model_desc.oz_min_mnk): "int8" = every dense GEMM on the int8 path (oz_min_mnk = 1), and
"hybrid" = the production default the bench times (GEMMs below 1e9 M N K on DMMA)."""
import numpy as np
import pytest

import slq_inputs as si
from oracle import fdhvp, lanczos as OL, models, probe

from . import oracle_cache as OC

ROUTES = {"int8": 1.0, "hybrid": 0.0}

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_00816_b200 import build
    build.build()


from paper_2602_00816_b200 import slq  # noqa: E402


@pytest.mark.parametrize("M,N,K,ak,bk", [(128, 64, 64, 1, 1), (300, 70, 100, 1, 1), (2048, 768, 256, 1, 1),
                                         (2048, 256, 1024, 1, 0), (768, 256, 2048, 0, 0), (37, 203, 64, 0, 1),
                                         (1, 5, 3, 1, 1), (129, 65, 4000, 1, 1), (64, 4096, 20000, 1, 1),
                                         (100, 50, 8192, 0, 0), (130, 70, 8200, 0, 0), (33, 17, 900, 0, 1)])
@pytest.mark.parametrize("S", [4, 5, 6, 7])
def test_oz_gemm_error_bound(M, N, K, ak, bk, S):
    """Truncated digits only: |C_oz - C| <= (S + 2) 2^-7S K 2^(e_i + f_j) (oz_gemm.cu header) and
    2^e_i < 2 max|A_i.|, so <= 4 (S + 2) 2^-7S K max|A_i.| max|B_.j|; covers ragged tiles, every
    operand layout, split-K and the K cap that keeps INT32 exact; the cols-path operands (ak / bk = 0)
    go through the fused cluster slicing up to K = 8192 (8 CTAs x 1024 k) and the two-pass slicing above."""
    err, tf = slq.oz_check(M, N, K, bool(ak), bool(bk), S, iters=1)
    bound = 4 * (S + 2) * 2.0 ** (-7 * S)
    print(f"oz S={S} {M}x{N}x{K} ak={ak} bk={bk}: err {err:.2e} (bound {bound:.1e}), {tf:.1f} TFLOP/s")
    assert err <= bound


def _batch(cfg):
    return si.mlp_data(cfg) if cfg.arch == si.ARCH_MLP else si.tokens(cfg)


@pytest.mark.parametrize("route", ["int8", "hybrid"])
@pytest.mark.parametrize("name", ["mlp_tiny", "c1", "gpt_tiny", "gpt_tiny_tied", "llama_tiny", "c2"])
def test_fp64_oz_grad_and_hvp(name, route):
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    v = si.random_vector(th.size, 5)
    with slq.SlqContext(cfg, th, _batch(cfg), pass_numerics="fp64_oz", oz_min_mnk=ROUTES[route]) as c:
        lay = c.layout()
        g = torch.empty(c.P_loc, dtype=torch.float32, device="cuda")
        loss = c.grad(g)
        vd = torch.from_numpy(slq.shard_of(v, lay, 0, 1)).cuda()
        out = torch.empty_like(vd)
        c.hvp(vd, out, cfg.eps)
        hv = slq.unshard([out.cpu().numpy()], lay)
        gf = slq.unshard([g.cpu().numpy()], lay)
    l_ref, g_ref = OC.loss_grad(name)
    ref = OC.hvp_exact(name, 5)
    eg = np.linalg.norm(gf - g_ref) / np.linalg.norm(g_ref)
    eh = np.linalg.norm(hv - ref) / np.linalg.norm(ref)
    print(f"{name} [fp64_oz {route}]: loss {abs(loss - l_ref) / abs(l_ref):.1e} grad {eg:.2e} HVP {eh:.2e}")
    assert abs(loss - l_ref) <= 1e-9 * abs(l_ref)
    assert eg <= 1e-7 and eh <= 1e-4


@pytest.mark.parametrize("name,m,route", [("gpt_tiny", 16, "int8"), ("llama_tiny", 16, "int8"), ("c1", 32, "int8"),
                                          ("c2", 32, "int8"), ("c2", 32, "hybrid")])
def test_fp64_oz_lanczos_fp32_gates(name, m, route):
    cfg = si.CONFIGS[name]
    th = si.init_params(cfg)
    with slq.SlqContext(cfg, th, _batch(cfg), pass_numerics="fp64_oz", reorth="full", max_steps=m,
                        oz_min_mnk=ROUTES[route]) as c:
        a, b = c.lanczos(cfg.probe_seed0, m)
    r = OC.lanczos_exact(name, m, "full")
    scale = np.abs(r.alpha).max()
    ea = np.abs(a - r.alpha) / np.maximum(np.abs(r.alpha), 1e-2 * scale)  # reading R14
    eb = np.abs(b - r.beta) / np.abs(r.beta)
    print(f"{name} [fp64_oz {route}]: max rel alpha {ea.max():.2e} beta {eb.max():.2e}")
    assert ea.max() <= 1e-5 and eb.max() <= 1e-5


def test_fp64_oz_nonfinite_propagates():
    """A NaN weight (theta_0) on the int8 path: the operand slicing marks that column of the qkv
    GEMM's B operand and the epilogue writes NaN (finite garbage before), so the loss is
    non-finite and the HVP fails with SLQ_ENUMERIC naming a sequence."""
    cfg = si.CONFIGS["c2"]
    th = si.init_params(cfg).copy()
    lay0 = slq.plan_layout(slq.make_desc(cfg, "fp64_oz"), 1)
    g0 = int(lay0["units"][1][0])  # first transformer block: ln1.g, ln1.b, then attn.qkv.w
    th[g0 + 2 * cfg.d_model + 7] = np.nan
    with slq.SlqContext(cfg, th, _batch(cfg), pass_numerics="fp64_oz", oz_min_mnk=1.0) as c:
        v = torch.from_numpy(slq.shard_of(si.random_vector(th.size, 5), c.layout(), 0, 1)).cuda()
        out = torch.empty_like(v)
        with pytest.raises(slq.SlqError) as e:
            c.hvp(v, out, cfg.eps)
        assert e.value.status == slq.SLQ_ENUMERIC
        seq = c.nonfinite_seq()
        print("nonfinite sequence", seq, e.value)
        assert seq == 0  # the NaN column reaches every token's logits
