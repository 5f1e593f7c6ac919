"""Central finite-difference HVP, Eq. (1) and Alg. 1 (oracle; test infrastructure only).

PAPER.md P:101-106, Eq. (1):   Hv ~= (grad L(theta + eps v) - grad L(theta - eps v)) / (2 eps)
PAPER.md P:163-185, Alg. 1: perturb shards (+eps v), accumulate weighted gradients, perturb
(-2 eps v), accumulate negated gradients, restore (+eps v), collect in FP32, scale by
1/(2 eps sum_b w_b).  With sum_b w_b = 1 the accumulated difference is g+ - g- where g is the
gradient of the dataset-mean loss.

Perturbation modes:
  * "param_dtype" (parity mode): the perturbed points are fp32 values with a single rounding,
        theta+- = fmaf(+-eta_f, v_f32, theta_f32),   eta_f = fl32(eta),
    and the divisor is 2*eta_f.  This is Alg. 1's "perturb the stored parameters" done out of
    place (theta is never written, "restore" is then exact by construction).
  * "exact" (diagnostic): theta +- eta v in fp64, divisor 2*eta.
`hvp` normalises a non-unit direction with the one scalar norm P:197 allows: it steps by
eta = eps/||v|| along v, which equals ||v|| * (g(theta+eps vhat) - g(theta-eps vhat))/(2 eps).
"""
from __future__ import annotations

import ctypes
from typing import Callable, Tuple

import numpy as np

from . import models
from .build import lib

GradFn = Callable[[np.ndarray], np.ndarray]


def make_grad_fn(d, batch, dt=np.float64) -> GradFn:
    """theta (any float array, canonical order) -> dataset-mean gradient in fp64."""
    return lambda theta: models.loss_grad(theta, d, batch, dt)[1]


def perturb_param_dtype(theta32: np.ndarray, v32: np.ndarray, eta: float) -> Tuple[np.ndarray, np.ndarray, float]:
    """(fl32(theta + eta_f v), fl32(theta - eta_f v), eta_f) with single-rounding fmaf (C helper)."""
    th = np.ascontiguousarray(theta32, dtype=np.float32)
    vv = np.ascontiguousarray(v32, dtype=np.float32)
    assert th.shape == vv.shape
    eta_f = np.float32(eta)
    plus = np.empty_like(th)
    minus = np.empty_like(th)
    lib().oracle_perturb_f32(th.ctypes.data, vv.ctypes.data, ctypes.c_float(eta_f),
                             plus.ctypes.data, minus.ctypes.data, th.size)
    return plus, minus, float(eta_f)


def fd_hvp_step(grad_fn: GradFn, theta: np.ndarray, v: np.ndarray, eta: float,
                mode: str = "param_dtype") -> np.ndarray:
    """Eq. (1) along direction v with step eta: (g(theta+eta v) - g(theta-eta v)) / (2 eta)."""
    if mode == "param_dtype":
        plus, minus, eta_f = perturb_param_dtype(theta, v, eta)
        gp = grad_fn(plus)
        gm = grad_fn(minus)
        return (gp - gm) / (2.0 * eta_f)
    if mode == "exact":
        th = np.asarray(theta, dtype=np.float64)
        vv = np.asarray(v, dtype=np.float64)
        gp = grad_fn(th + eta * vv)
        gm = grad_fn(th - eta * vv)
        return (gp - gm) / (2.0 * eta)
    raise ValueError(mode)


def hvp(grad_fn: GradFn, theta: np.ndarray, v: np.ndarray, eps: float,
        mode: str = "param_dtype") -> np.ndarray:
    """||v|| * FD-HVP along vhat = v/||v|| with step eps (P:197 scalar norm)."""
    nv = float(np.sqrt(np.sum(np.asarray(v, dtype=np.float64) ** 2)))
    if nv == 0.0:
        return np.zeros(np.asarray(v).shape, dtype=np.float64)
    return fd_hvp_step(grad_fn, theta, v, eps / nv, mode)


def alg1_inplace_fp32(grad_fn: GradFn, theta32: np.ndarray, v32: np.ndarray, eps: float):
    """Alg. 1 as printed (P:169/175/180): in-place +eps, -2eps, +eps AXPYs in fp32 storage.

    Diagnostic only: returns (Hv, theta after restore).  In fp32 the restore is not exact in
    general, which is why the product path perturbs out of place.
    """
    e = np.float32(eps)
    v = np.asarray(v32, dtype=np.float32)
    th = np.array(theta32, dtype=np.float32)
    th = (th + e * v).astype(np.float32)
    acc = grad_fn(th)
    th = (th - np.float32(2.0) * e * v).astype(np.float32)
    acc = acc - grad_fn(th)
    th = (th + e * v).astype(np.float32)
    return acc / (2.0 * float(e)), th


def optimal_epsilon(eps_mach: float, grad_norm: float = 1.0, d3_grad_norm: float = 1.0) -> float:
    """Theorem 1: eps* ~ (eps_mach ||grad L|| / ||grad D_v^3 L||)^(1/3)."""
    return (eps_mach * grad_norm / d3_grad_norm) ** (1.0 / 3.0)


def theorem1_bound(eps: float, eps_mach: float, grad_norm: float, d3_grad_norm: float) -> float:
    """Theorem 1 leading terms: eps^2/6 ||grad D^3 L|| + eps_mach ||grad L|| / eps."""
    return eps * eps / 6.0 * d3_grad_norm + eps_mach * grad_norm / eps
