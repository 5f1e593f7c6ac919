"""Pins for oracle/probe.py and oracle/models.py (CPU only)."""
import json
import math
import os

import numpy as np
import pytest

import slq_inputs as si
from oracle import models, probe

from . import torch_ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_published_value():
    g = json.load(open(os.path.join(GOLD, "probe_splitmix64.json")))
    for k, v in g["splitmix64"].items():
        assert probe.splitmix64_int(int(k)) == int(v, 16)
        assert int(probe.splitmix64(np.array([int(k)], dtype=np.uint64))[0]) == int(v, 16)


def test_probe_sign_vectors():
    g = json.load(open(os.path.join(GOLD, "probe_splitmix64.json")))
    for seed, s in g["signs"].items():
        got = "".join("+" if x > 0 else "-" for x in probe.signs(int(seed), 32))
        assert got == s


def test_probe_offset_and_norm():
    # signs at an offset are the same hash evaluated at the global index
    full = probe.signs(7, 1000)
    assert np.array_equal(full[300:400], probe.signs(7, 100, first=300))
    q = probe.rademacher_probe(3, 9610)
    assert abs(np.linalg.norm(q) - 1.0) < 1e-14
    assert np.allclose(np.abs(q), 1 / math.sqrt(9610))
    # roughly balanced (a plausible wrong bit would give all +1)
    assert abs(probe.signs(5, 100000).mean()) < 0.02


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5", "gpt_tiny", "gpt_tiny_tied", "llama_tiny"])
def test_param_counts(name):
    # BASELINE.json config text: 9,610 / ~5M / ~124M / 1B / 8B (SURVEY §8(c2) #12 exact counts)
    expect = {"c1": 9610, "c2": 5322240, "c3": 124439808, "c4": 1104218112, "c5": 8030261248}
    d = si.CONFIGS[name]
    assert models.num_params(d) == si.n_params(d)
    if name in expect:
        assert models.num_params(d) == expect[name]


def _perturbed_theta(d, seed=5, scale=0.05):
    th = si.init_params(d).astype(np.float64)
    return th + np.random.default_rng(seed).standard_normal(th.size) * scale


def _batch(d):
    return si.mlp_data(d) if d.arch == si.ARCH_MLP else si.tokens(d)


@pytest.mark.parametrize("name", ["mlp_tiny", "c1", "gpt_tiny", "gpt_tiny_tied", "llama_tiny"])
def test_gradient_matches_autograd(name):
    """Hand-derived backprop == torch autograd of an independently written forward."""
    d = si.CONFIGS[name]
    th = _perturbed_theta(d)
    b = _batch(d)
    loss, g = models.loss_grad(th, d, b)
    import torch
    tl = float(torch_ref.loss(torch.tensor(th), d, b))
    gr = torch_ref.grad(th, d, b)
    assert abs(loss - tl) <= 1e-12 * abs(tl)
    assert np.linalg.norm(g - gr) <= 1e-11 * np.linalg.norm(gr)


@pytest.mark.parametrize("name", ["mlp_tiny", "gpt_tiny", "llama_tiny"])
def test_gradient_directional_fd(name):
    """<grad L, v> against a Richardson-extrapolated function-value difference (brute force)."""
    d = si.CONFIGS[name]
    th = _perturbed_theta(d, seed=9)
    b = _batch(d)
    v = np.random.default_rng(2).standard_normal(th.size)
    v /= np.linalg.norm(v)
    g = models.loss_grad(th, d, b)[1]

    def cd(h):
        return (models.loss_only(th + h * v, d, b) - models.loss_only(th - h * v, d, b)) / (2 * h)

    rich = (4 * cd(5e-4) - cd(1e-3)) / 3
    assert abs(g @ v - rich) <= 1e-8 * max(1.0, abs(rich))


@pytest.mark.parametrize("name", ["gpt_tiny", "llama_tiny", "mlp_tiny"])
def test_zero_weights_uniform_loss(name):
    """All weights zero (gains 1) => logits 0 => loss = log(#classes) exactly."""
    d = si.CONFIGS[name]
    th = np.zeros(models.num_params(d))
    if d.arch != si.ARCH_MLP:
        off = 0
        for nm, shape in models.layout(d):
            n = int(np.prod(shape))
            if nm.endswith(".g") or nm.endswith("norm"):
                th[off:off + n] = 1.0
            off += n
    ncls = d.n_classes if d.arch == si.ARCH_MLP else d.vocab
    loss = models.loss_only(th, d, _batch(d))
    assert abs(loss - math.log(ncls)) < 1e-12


@pytest.mark.parametrize("name", ["gpt_tiny", "llama_tiny"])
def test_causality(name):
    """Changing the LAST target token changes only the last position's loss term: the
    gradient w.r.t. everything except via that logit is unchanged in the other positions.
    Checked as: changing the final input-only token (never an input) leaves L(theta) of a
    truncated batch identical."""
    d = si.CONFIGS[name]
    th = _perturbed_theta(d, seed=3)
    tok = si.tokens(d)
    t2 = tok.copy()
    t2[:, -1] = (t2[:, -1] + 1) % d.vocab
    # the last token is a target only: losses differ, but the first T-1 positions agree.
    import dataclasses
    dshort = dataclasses.replace(d)
    l1 = models.loss_only(th, dshort, tok[:, :-1])
    l2 = models.loss_only(th, dshort, t2[:, :-1])
    assert l1 == l2
    assert models.loss_only(th, d, tok) != models.loss_only(th, d, t2)
