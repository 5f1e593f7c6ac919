"""Activation checkpointing (slq_model_desc.act_ckpt; BASELINE configs[4] "with activation
checkpointing"): every block keeps its input residual stream only and recomputes its forward
inside its backward.  The recomputation runs the same kernels on the same inputs, so gradients,
HVPs and Lanczos coefficients must be BIT-IDENTICAL to the run without it.  Also: the device
memory actually taken by a context matches slq_plan_memory."""
import functools

import numpy as np
import pytest

import slq_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_00816_b200 import build
    build.build()


from paper_2602_00816_b200 import slq  # noqa: E402


@functools.lru_cache(maxsize=1)
def _inputs(cfg):
    return si.init_params(cfg), si.tokens(cfg)


@functools.lru_cache(maxsize=1)
def _direction(P):
    return si.random_vector(P, 5)


def _run(cfg, numerics, ckpt, m):
    th, tok = _inputs(cfg)
    with slq.SlqContext(cfg, th, tok, pass_numerics=numerics, reorth="full" if cfg.reorth_full else "none",
                        max_steps=m, act_ckpt=ckpt) as c:
        lay = c.layout()
        v = torch.from_numpy(slq.shard_of(_direction(th.size), lay, 0, 1)).cuda()
        g = torch.empty_like(v)
        loss = c.grad(g)
        out = torch.empty_like(v)
        c.hvp(v, out, cfg.eps)
        a, b = c.lanczos(cfg.probe_seed0, m)
    return loss, g.cpu().numpy(), out.cpu().numpy(), a, b


# the two top blocks keep their forward activations (nothing to recompute), so every case has
# >= 3 blocks; odd and even depths exercise both activation sets
@pytest.mark.parametrize("name,layers,numerics", [("gpt_tiny", 5, "fp64"), ("gpt_tiny_tied", 4, "fp64"),
                                                  ("llama_tiny", 5, "fp64"), ("c2", 4, "fp64_oz"),
                                                  ("llama_tiny", 3, "bf16x3"), ("c4_parity", 4, "fp64_oz"),
                                                  ("c5_twin", 3, "fp64_oz")])
def test_checkpointing_bit_identical(name, layers, numerics):
    cfg = si.get_config(name, n_layers=layers)
    m = {"c4_parity": 3, "c5_twin": 2}.get(name, 6)
    r0 = _run(cfg, numerics, False, m)
    r1 = _run(cfg, numerics, True, m)
    print(f"{name} [{numerics}]: loss {r0[0]:.12f} alpha {r0[3]}")
    assert r0[0] == r1[0]
    for x, y in zip(r0[1:], r1[1:]):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name,numerics,ckpt", [("c2", "fp64_oz", False), ("c3", "fp64_oz", True),
                                                ("c4_parity", "fp64", True)])
def test_memory_plan_matches_allocation(name, numerics, ckpt):
    """Device bytes a context holds after init and one HVP (workspaces are reserved up front at their
    planned size) against slq_plan_memory; the host-call staging buffers are not allocated here."""
    cfg = si.get_config(name, n_layers=4) if name == "c4_parity" else si.CONFIGS[name]
    th, tok = _inputs(cfg)
    desc = slq.make_desc(cfg, numerics, max_steps=cfg.m, act_ckpt=ckpt)
    P_loc = slq.plan_layout(desc, 1)["P_loc"]
    v = torch.zeros(P_loc, dtype=torch.float32, device="cuda")
    v[0] = 1.0
    out = torch.empty_like(v)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()  # (torch's cached blocks would hide allocations from mem_get_info)
    free0, _ = torch.cuda.mem_get_info()
    with slq.SlqContext(cfg, th, tok, pass_numerics=numerics, max_steps=cfg.m, act_ckpt=ckpt) as c:
        torch.cuda.synchronize()
        free1, _ = torch.cuda.mem_get_info()
        c.hvp(v, out, cfg.eps)
        free2, _ = torch.cuda.mem_get_info()
        p = slq.plan_memory(c.desc, 1, cfg.n_seq)
    used_init = free0 - free1
    used_hvp = free0 - free2
    planned = p["total"] - 2 * 4 * P_loc  # minus the staging of host-pointer calls (not used here)
    print(f"{name} ckpt={ckpt}: planned {planned / 2**30:.3f} GiB, after init {used_init / 2**30:.3f}, "
          f"after hvp {used_hvp / 2**30:.3f} GiB; plan {({k: round(x / 2**30, 3) for k, x in p.items()})}")
    assert abs(used_init - planned) <= 0.02 * planned + (256 << 20)
    assert used_hvp - used_init <= 0.03 * planned + (512 << 20)  # graphs, NCCL/cuBLAS-free: small
