"""Per-session memo of oracle results that several GPU parity tests compare against (test
infrastructure only).  The same oracle run -- e.g. c2's 32-step fully reorthogonalised Lanczos on
the exact FD-HVP operator, ~1 min of fp64 numpy -- is the reference of the FP64, FP64_OZ (both
routes), paired and bf16-basis tests; computing it once keeps the GPU suite inside its time budget.
Values are exactly what the direct oracle calls return (same inputs, same functions)."""
import functools

import numpy as np

import slq_inputs as si
from oracle import fdhvp, lanczos as OL, models, probe


def batch(cfg):
    return si.mlp_data(cfg) if cfg.arch == si.ARCH_MLP else si.tokens(cfg)


@functools.lru_cache(maxsize=None)
def theta(name):
    return si.init_params(si.CONFIGS[name])


@functools.lru_cache(maxsize=None)
def grad_fn(name):
    cfg = si.CONFIGS[name]
    return fdhvp.make_grad_fn(cfg, batch(cfg))


def lanczos_exact(name, m, reorth="full", window=0, basis="fp64"):
    """oracle Lanczos from the config's probe on the exact-perturbation FD-HVP operator"""
    return _lanczos_exact(name, int(m), reorth, int(window), basis)  # one cache key per run


@functools.lru_cache(maxsize=None)
def _lanczos_exact(name, m, reorth, window, basis):
    cfg = si.CONFIGS[name]
    th = theta(name)
    g = grad_fn(name)
    return OL.lanczos(lambda q: fdhvp.fd_hvp_step(g, th, q, cfg.eps, "exact"),
                      probe.rademacher_probe(cfg.probe_seed0, th.size), m, reorth, window=window, basis=basis)


@functools.lru_cache(maxsize=None)
def hvp_exact(name, vseed):
    """oracle FD-HVP (exact perturbation) of si.random_vector(P, vseed) at the config's eps"""
    cfg = si.CONFIGS[name]
    th = theta(name)
    return fdhvp.hvp(grad_fn(name), th, si.random_vector(th.size, vseed), cfg.eps, "exact")


@functools.lru_cache(maxsize=None)
def loss_grad(name):
    cfg = si.CONFIGS[name]
    return models.loss_grad(theta(name), cfg, batch(cfg))
