"""Independent torch-CPU forward definitions used ONLY to pin the oracle's hand-derived
gradients (autograd is an independent implementation of the chain rule) and to get exact
Hessian-vector products by double backprop.  Built from torch library ops
(F.layer_norm, torch.softmax, F.gelu(tanh), F.silu, F.cross_entropy), not from the
oracle's code.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

import slq_inputs as si


def _sdpa_causal(q, k, v):
    # explicit causal attention (torch's fused SDPA has no double backward on CPU)
    T = q.shape[-2]
    s = (q @ k.transpose(-1, -2)) / (q.shape[-1] ** 0.5)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool), diagonal=1)
    return torch.softmax(s.masked_fill(mask, float("-inf")), dim=-1) @ v


def _views(theta: torch.Tensor, d):
    out, off = {}, 0
    for name, shape, _ in si.param_table(d):
        n = int(np.prod(shape))
        out[name] = theta[off:off + n].view(*shape)
        off += n
    return out


def loss(theta: torch.Tensor, d, batch) -> torch.Tensor:
    P = _views(theta, d)
    if d.arch == si.ARCH_MLP:
        x, y = batch
        x = torch.as_tensor(x, dtype=theta.dtype)
        h = torch.tanh(F.linear(x, P["fc1.w"], P["fc1.b"]))
        return F.cross_entropy(F.linear(h, P["fc2.w"], P["fc2.b"]), torch.as_tensor(y).long())
    tok = torch.as_tensor(batch).long()
    B, T = tok.shape[0], tok.shape[1] - 1
    inp, tgt = tok[:, :T], tok[:, 1:]
    D, H = d.d_model, d.n_heads
    hd = D // H
    if d.arch == si.ARCH_GPT:
        x = P["wte"][inp] + P["wpe"][:T][None]
        for l in range(d.n_layers):
            p = f"h{l}."
            h = F.layer_norm(x, (D,), P[p + "ln1.g"], P[p + "ln1.b"], eps=d.norm_eps)
            qkv = F.linear(h, P[p + "attn.qkv.w"], P[p + "attn.qkv.b"])
            q, k, v = qkv.split(D, dim=-1)
            q, k, v = (t.view(B, T, H, hd).transpose(1, 2) for t in (q, k, v))
            o = _sdpa_causal(q, k, v)
            o = o.transpose(1, 2).reshape(B, T, D)
            x = x + F.linear(o, P[p + "attn.proj.w"], P[p + "attn.proj.b"])
            h = F.layer_norm(x, (D,), P[p + "ln2.g"], P[p + "ln2.b"], eps=d.norm_eps)
            h = F.gelu(F.linear(h, P[p + "mlp.fc.w"], P[p + "mlp.fc.b"]), approximate="tanh")
            x = x + F.linear(h, P[p + "mlp.proj.w"], P[p + "mlp.proj.b"])
        x = F.layer_norm(x, (D,), P["lnf.g"], P["lnf.b"], eps=d.norm_eps)
        w = P["wte"] if d.tie_embeddings else P["head.w"]
        return F.cross_entropy(F.linear(x, w).reshape(B * T, -1), tgt.reshape(-1))
    # Llama
    KV = d.n_kv_heads
    half = hd // 2
    inv = d.rope_theta ** (-(2.0 * torch.arange(half, dtype=theta.dtype)) / hd)
    ang = torch.arange(T, dtype=theta.dtype)[:, None] * inv[None]
    cos, sin = torch.cos(ang), torch.sin(ang)

    def rope(t):
        t1, t2 = t[..., :half], t[..., half:]
        return torch.cat([t1 * cos - t2 * sin, t2 * cos + t1 * sin], dim=-1)

    def rms(x, g):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + d.norm_eps) * g

    x = P["tok"][inp]
    for l in range(d.n_layers):
        p = f"h{l}."
        h = rms(x, P[p + "attn_norm.g"])
        q = rope(F.linear(h, P[p + "wq"]).view(B, T, H, hd).transpose(1, 2))
        k = rope(F.linear(h, P[p + "wk"]).view(B, T, KV, hd).transpose(1, 2))
        v = F.linear(h, P[p + "wv"]).view(B, T, KV, hd).transpose(1, 2)
        k = k.repeat_interleave(H // KV, dim=1)
        v = v.repeat_interleave(H // KV, dim=1)
        o = _sdpa_causal(q, k, v).transpose(1, 2).reshape(B, T, D)
        x = x + F.linear(o, P[p + "wo"])
        h = rms(x, P[p + "mlp_norm.g"])
        x = x + F.linear(F.silu(F.linear(h, P[p + "w_gate"])) * F.linear(h, P[p + "w_up"]), P[p + "w_down"])
    x = rms(x, P["norm.g"])
    w = P["tok"] if d.tie_embeddings else P["head.w"]
    return F.cross_entropy(F.linear(x, w).reshape(B * T, -1), tgt.reshape(-1))


def grad(theta_np: np.ndarray, d, batch) -> np.ndarray:
    th = torch.tensor(np.asarray(theta_np, dtype=np.float64), requires_grad=True)
    (g,) = torch.autograd.grad(loss(th, d, batch), th)
    return g.numpy()


def exact_hvp(theta_np: np.ndarray, d, batch, v_np: np.ndarray) -> np.ndarray:
    """H v by double backprop (fp64)."""
    th = torch.tensor(np.asarray(theta_np, dtype=np.float64), requires_grad=True)
    v = torch.tensor(np.asarray(v_np, dtype=np.float64))
    (g,) = torch.autograd.grad(loss(th, d, batch), th, create_graph=True)
    (hv,) = torch.autograd.grad(g @ v, th)
    return hv.numpy()
