"""Host-only device-memory plan (slq_plan_memory; no GPU): the categories add up, activation
checkpointing (BASELINE configs[4]) keeps two blocks' activations instead of n_layers, and the c5
plan (Llama-3-8B shape, 2 x 2048 tokens per GPU, FSDP over 8 ranks, FP64_OZ, no stored basis) fits
a B200 only with checkpointing."""
import pytest

import slq_inputs as si
from paper_2602_00816_b200 import slq


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2602_00816_b200 import build
    build.build()


def plan(name, R, n_local, numerics="fp64_oz", ckpt=False, reorth=None):
    return slq.plan_memory(slq.make_desc(si.CONFIGS[name], numerics, reorth=reorth, act_ckpt=ckpt), R, n_local)


def test_categories_sum_to_total():
    for name, R, n in [("c1", 1, 256), ("c2", 1, 8), ("c2", 2, 4), ("c3", 1, 8), ("c4", 8, 4)]:
        p = plan(name, R, n)
        assert p["total"] == sum(v for k, v in p.items() if k != "total"), (name, p)
        assert all(v >= 0 for v in p.values())


def test_c5_fits_only_with_checkpointing():
    on = plan("c5", 8, 2, ckpt=True)
    off = plan("c5", 8, 2, ckpt=False)
    print({k: round(v / 1e9, 2) for k, v in on.items()})
    assert on["total"] <= 170e9  # VERDICT r1 "done when": <= 170 GB per GPU at R = 8 in FP64_OZ
    assert off["total"] > 180e9  # no checkpointing: does not fit 180 GB of HBM3e
    # activations: 32 layer sets -> 2 sets (the rest is per-layer residual streams and data)
    assert on["activations"] < off["activations"] / 8
    for k in ("theta", "points", "grads", "lanczos", "fsdp", "logits", "scratch", "workspace"):
        assert on[k] == off[k], k


def test_sharding_divides_the_vectors():
    p1, p8 = plan("c4", 1, 4, reorth="none", ckpt=True), plan("c4", 8, 4, reorth="none", ckpt=True)
    assert 7.5 < p1["theta"] / p8["theta"] < 8.5
    assert p1["fsdp"] == 0 and p8["fsdp"] > 0
    assert p1["activations"] == p8["activations"]  # per-GPU batch fixed


def test_basis_storage():
    full = plan("c3", 1, 8, reorth="full")
    none = plan("c3", 1, 8, reorth="none")
    P_loc = slq.plan_layout(slq.make_desc(si.CONFIGS["c3"], "fp64_oz"), 1)["P_loc"]
    # (m + 1) fp32 rows instead of three rotating vectors
    assert abs((full["lanczos"] - none["lanczos"]) - 4 * P_loc * (si.CONFIGS["c3"].m + 1 - 3)) < 1e8
