"""Loss L(theta) and its gradient for the three model families (oracle; test infrastructure only).

The paper's FD-HVP (Eq. (1)) needs only the dataset-averaged gradient
grad L(theta); Alg. 1 accumulates per-batch gradients with weights w_b and scales by
sum_b w_b.  Reading: L is the mean token-level cross
entropy over ALL sequences and positions of the global batch (sum w_b = 1); for the MLP it is
the mean softmax cross entropy over the rows.

Everything here is the plain definition written out with numpy: forward pass, then the
chain rule layer by layer in reverse (hand-derived backprop).  Arithmetic is in the dtype of
`dt` (fp64 by default; fp32 is used only for the Theorem 1 round-off pin).

Model conventions (readings):
  MLP   : logits = W2 tanh(W1 x + b1) + b2
  GPT   : pre-LayerNorm blocks, learned positions, causal MHA (scale 1/sqrt(hd)),
          GELU (tanh approximation), biases, final LayerNorm, head (or tied wte); LN eps 1e-5
  Llama : pre-RMSNorm blocks, RoPE (half-split rotation, freq theta^(-2i/hd)), GQA
          (kv head = q head // (n_heads/n_kv_heads)), SwiGLU (silu(x Wg^T) * x Wu^T) Wd^T,
          no biases, final RMSNorm, untied head; RMSNorm eps 1e-5
The canonical parameter order below is this module's own table (layer-major).
"""
from __future__ import annotations

import math
from typing import Dict, List, Tuple

import numpy as np

ARCH_MLP, ARCH_GPT, ARCH_LLAMA = 0, 1, 2


# ------------------------------------------------------------------------------------------
# parameter table (oracle's own copy of the canonical order)
# ------------------------------------------------------------------------------------------

def layout(d) -> List[Tuple[str, Tuple[int, ...]]]:
    if d.arch == ARCH_MLP:
        return [("fc1.w", (d.d_hidden, d.d_in)), ("fc1.b", (d.d_hidden,)),
                ("fc2.w", (d.n_classes, d.d_hidden)), ("fc2.b", (d.n_classes,))]
    D, F, V = d.d_model, d.d_ff, d.vocab
    out: List[Tuple[str, Tuple[int, ...]]] = []
    if d.arch == ARCH_GPT:
        out += [("wte", (V, D)), ("wpe", (d.seq_len, D))]
        for l in range(d.n_layers):
            p = f"h{l}."
            out += [(p + "ln1.g", (D,)), (p + "ln1.b", (D,)),
                    (p + "qkv.w", (3 * D, D)), (p + "qkv.b", (3 * D,)),
                    (p + "proj.w", (D, D)), (p + "proj.b", (D,)),
                    (p + "ln2.g", (D,)), (p + "ln2.b", (D,)),
                    (p + "fc.w", (F, D)), (p + "fc.b", (F,)),
                    (p + "mproj.w", (D, F)), (p + "mproj.b", (D,))]
        out += [("lnf.g", (D,)), ("lnf.b", (D,))]
        if not d.tie_embeddings:
            out += [("head.w", (V, D))]
        return out
    if d.arch == ARCH_LLAMA:
        hd = d.d_model // d.n_heads
        out += [("tok", (V, D))]
        for l in range(d.n_layers):
            p = f"h{l}."
            out += [(p + "attn_norm", (D,)), (p + "wq", (d.n_heads * hd, D)),
                    (p + "wk", (d.n_kv_heads * hd, D)), (p + "wv", (d.n_kv_heads * hd, D)),
                    (p + "wo", (D, d.n_heads * hd)), (p + "mlp_norm", (D,)),
                    (p + "wg", (F, D)), (p + "wu", (F, D)), (p + "wd", (D, F))]
        out += [("norm", (D,))]
        if not d.tie_embeddings:
            out += [("head.w", (V, D))]
        return out
    raise ValueError(d.arch)


def num_params(d) -> int:
    return int(sum(int(np.prod(s)) for _, s in layout(d)))


def unpack(theta: np.ndarray, d, dt) -> Dict[str, np.ndarray]:
    P, off = {}, 0
    for name, shape in layout(d):
        n = int(np.prod(shape))
        P[name] = np.asarray(theta[off:off + n], dtype=dt).reshape(shape)
        off += n
    assert off == theta.size, (off, theta.size)
    return P


def pack(G: Dict[str, np.ndarray], d) -> np.ndarray:
    return np.concatenate([G[name].reshape(-1).astype(np.float64) for name, _ in layout(d)])


# ------------------------------------------------------------------------------------------
# layer primitives: forward returns (out, cache); backward maps d(out) -> d(inputs)
# ------------------------------------------------------------------------------------------

def cross_entropy(logits: np.ndarray, target: np.ndarray):
    """mean_i [ logsumexp(logits_i) - logits_i[target_i] ] and d/dlogits."""
    n = logits.shape[0]
    mx = logits.max(axis=1, keepdims=True)
    ex = np.exp(logits - mx)
    se = ex.sum(axis=1, keepdims=True)
    lse = (mx + np.log(se))[:, 0]
    loss = float(np.mean(lse - logits[np.arange(n), target]))
    dlogits = ex / se
    dlogits[np.arange(n), target] -= 1.0
    dlogits /= n
    return loss, dlogits


def layernorm_fwd(x, g, b, eps):
    mu = x.mean(axis=1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = xc * rstd
    return xhat * g + b, (xhat, rstd, g)


def layernorm_bwd(dy, cache):
    xhat, rstd, g = cache
    dg = (dy * xhat).sum(axis=0)
    db = dy.sum(axis=0)
    dxhat = dy * g
    dx = rstd * (dxhat - dxhat.mean(axis=1, keepdims=True)
                 - xhat * (dxhat * xhat).mean(axis=1, keepdims=True))
    return dx, dg, db


def rmsnorm_fwd(x, g, eps):
    r = 1.0 / np.sqrt((x * x).mean(axis=1, keepdims=True) + eps)
    return x * r * g, (x, r, g)


def rmsnorm_bwd(dy, cache):
    x, r, g = cache
    dg = (dy * x * r).sum(axis=0)
    dxhat = dy * g
    dx = r * dxhat - x * (r ** 3) * (dxhat * x).mean(axis=1, keepdims=True)
    return dx, dg


_GELU_C = math.sqrt(2.0 / math.pi)


def gelu_tanh(u):
    t = np.tanh(_GELU_C * (u + 0.044715 * u ** 3))
    return 0.5 * u * (1.0 + t), t


def gelu_tanh_grad(u, t):
    return 0.5 * (1.0 + t) + 0.5 * u * (1.0 - t * t) * _GELU_C * (1.0 + 3 * 0.044715 * u * u)


def silu(a):
    s = 1.0 / (1.0 + np.exp(-a))
    return a * s, s


def causal_attention_fwd(q, k, v):
    """q [B,H,T,hd], k,v [B,H,T,hd] (already expanded for GQA); softmax(q k^T / sqrt(hd)) v,
    causal (key j visible to query i iff j <= i)."""
    B, H, T, hd = q.shape
    scale = 1.0 / math.sqrt(hd)
    mask = np.triu(np.ones((T, T), dtype=bool), k=1)
    o = np.empty_like(q)
    for b in range(B):
        s = np.matmul(q[b], np.swapaxes(k[b], -1, -2)) * scale
        s[:, mask] = -np.inf
        s = s - s.max(axis=-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=-1, keepdims=True)
        o[b] = np.matmul(p, v[b])
    return o


def causal_attention_bwd(do, q, k, v):
    """Gradients of causal_attention_fwd (probabilities recomputed)."""
    B, H, T, hd = q.shape
    scale = 1.0 / math.sqrt(hd)
    mask = np.triu(np.ones((T, T), dtype=bool), k=1)
    dq, dk, dv = np.empty_like(q), np.empty_like(k), np.empty_like(v)
    for b in range(B):
        s = np.matmul(q[b], np.swapaxes(k[b], -1, -2)) * scale
        s[:, mask] = -np.inf
        s = s - s.max(axis=-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=-1, keepdims=True)
        dv[b] = np.matmul(np.swapaxes(p, -1, -2), do[b])
        dp = np.matmul(do[b], np.swapaxes(v[b], -1, -2))
        ds = p * (dp - (dp * p).sum(axis=-1, keepdims=True))
        dq[b] = np.matmul(ds, k[b]) * scale
        dk[b] = np.matmul(np.swapaxes(ds, -1, -2), q[b]) * scale
    return dq, dk, dv


def rope_tables(T, hd, theta, dt):
    half = hd // 2
    inv = theta ** (-(2.0 * np.arange(half)) / hd)
    ang = np.arange(T)[:, None] * inv[None, :]           # [T, half]
    return np.cos(ang).astype(dt), np.sin(ang).astype(dt)


def rope_fwd(x, cos, sin):
    """x [B,H,T,hd]; rotate pairs (i, i+hd/2) by angle pos*theta^(-2i/hd)."""
    half = x.shape[-1] // 2
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], axis=-1)


def rope_bwd(dy, cos, sin):
    half = dy.shape[-1] // 2
    d1, d2 = dy[..., :half], dy[..., half:]
    return np.concatenate([d1 * cos + d2 * sin, d2 * cos - d1 * sin], axis=-1)


# ------------------------------------------------------------------------------------------
# models
# ------------------------------------------------------------------------------------------

def mlp_loss_grad(theta, d, x, y, dt=np.float64):
    P = unpack(theta, d, dt)
    X = np.asarray(x, dtype=dt)
    z1 = X @ P["fc1.w"].T + P["fc1.b"]
    h = np.tanh(z1)
    z2 = h @ P["fc2.w"].T + P["fc2.b"]
    loss, dz2 = cross_entropy(z2, y)
    G = {"fc2.w": dz2.T @ h, "fc2.b": dz2.sum(axis=0)}
    dh = dz2 @ P["fc2.w"]
    dz1 = dh * (1.0 - h * h)
    G["fc1.w"] = dz1.T @ X
    G["fc1.b"] = dz1.sum(axis=0)
    return loss, pack(G, d)


def _split_heads(x, B, T, H, hd):
    return x.reshape(B, T, H, hd).transpose(0, 2, 1, 3)


def _merge_heads(x):
    B, H, T, hd = x.shape
    return x.transpose(0, 2, 1, 3).reshape(B * T, H * hd)


def gpt_loss_grad(theta, d, tok, dt=np.float64):
    P = unpack(theta, d, dt)
    B, T = tok.shape[0], tok.shape[1] - 1
    D, H = d.d_model, d.n_heads
    hd = D // H
    N = B * T
    inp, tgt = tok[:, :T], tok[:, 1:].reshape(-1)
    eps = d.norm_eps
    x = (P["wte"][inp] + P["wpe"][None, :T]).reshape(N, D)
    caches = []
    for l in range(d.n_layers):
        p = f"h{l}."
        h1, c1 = layernorm_fwd(x, P[p + "ln1.g"], P[p + "ln1.b"], eps)
        qkv = h1 @ P[p + "qkv.w"].T + P[p + "qkv.b"]
        q = _split_heads(qkv[:, :D], B, T, H, hd)
        k = _split_heads(qkv[:, D:2 * D], B, T, H, hd)
        v = _split_heads(qkv[:, 2 * D:], B, T, H, hd)
        o = _merge_heads(causal_attention_fwd(q, k, v))
        x1 = x + o @ P[p + "proj.w"].T + P[p + "proj.b"]
        h2, c2 = layernorm_fwd(x1, P[p + "ln2.g"], P[p + "ln2.b"], eps)
        u = h2 @ P[p + "fc.w"].T + P[p + "fc.b"]
        gu, t = gelu_tanh(u)
        x = x1 + gu @ P[p + "mproj.w"].T + P[p + "mproj.b"]
        caches.append((c1, h1, q, k, v, o, c2, h2, u, t, gu))
    xf, cf = layernorm_fwd(x, P["lnf.g"], P["lnf.b"], eps)
    w_head = P["wte"] if d.tie_embeddings else P["head.w"]
    logits = xf @ w_head.T
    loss, dlogits = cross_entropy(logits, tgt)

    G: Dict[str, np.ndarray] = {}
    dw_head = dlogits.T @ xf
    dxf = dlogits @ w_head
    dx, G["lnf.g"], G["lnf.b"] = layernorm_bwd(dxf, cf)
    for l in reversed(range(d.n_layers)):
        p = f"h{l}."
        c1, h1, q, k, v, o, c2, h2, u, t, gu = caches[l]
        G[p + "mproj.w"] = dx.T @ gu
        G[p + "mproj.b"] = dx.sum(axis=0)
        du = (dx @ P[p + "mproj.w"]) * gelu_tanh_grad(u, t)
        G[p + "fc.w"] = du.T @ h2
        G[p + "fc.b"] = du.sum(axis=0)
        dh2, G[p + "ln2.g"], G[p + "ln2.b"] = layernorm_bwd(du @ P[p + "fc.w"], c2)
        dx1 = dx + dh2
        G[p + "proj.w"] = dx1.T @ o
        G[p + "proj.b"] = dx1.sum(axis=0)
        do = _split_heads(dx1 @ P[p + "proj.w"], B, T, H, hd)
        dq, dk, dv = causal_attention_bwd(do, q, k, v)
        dqkv = np.concatenate([_merge_heads(dq), _merge_heads(dk), _merge_heads(dv)], axis=1)
        G[p + "qkv.w"] = dqkv.T @ h1
        G[p + "qkv.b"] = dqkv.sum(axis=0)
        dh1, G[p + "ln1.g"], G[p + "ln1.b"] = layernorm_bwd(dqkv @ P[p + "qkv.w"], c1)
        dx = dx1 + dh1
    dx0 = dx.reshape(B, T, D)
    dwte = np.zeros_like(P["wte"])
    np.add.at(dwte, inp.reshape(-1), dx.reshape(N, D))
    if d.tie_embeddings:
        dwte = dwte + dw_head
    else:
        G["head.w"] = dw_head
    G["wte"] = dwte
    dwpe = np.zeros_like(P["wpe"])
    dwpe[:T] = dx0.sum(axis=0)
    G["wpe"] = dwpe
    return loss, pack(G, d)


def llama_loss_grad(theta, d, tok, dt=np.float64):
    P = unpack(theta, d, dt)
    B, T = tok.shape[0], tok.shape[1] - 1
    D, H, KV = d.d_model, d.n_heads, d.n_kv_heads
    hd = D // H
    rep = H // KV
    N = B * T
    inp, tgt = tok[:, :T], tok[:, 1:].reshape(-1)
    eps = d.norm_eps
    cos, sin = rope_tables(T, hd, d.rope_theta, dt)
    x = P["tok"][inp].reshape(N, D)
    caches = []
    for l in range(d.n_layers):
        p = f"h{l}."
        h1, c1 = rmsnorm_fwd(x, P[p + "attn_norm"], eps)
        q = rope_fwd(_split_heads(h1 @ P[p + "wq"].T, B, T, H, hd), cos, sin)
        k = rope_fwd(_split_heads(h1 @ P[p + "wk"].T, B, T, KV, hd), cos, sin)
        v = _split_heads(h1 @ P[p + "wv"].T, B, T, KV, hd)
        ke, ve = np.repeat(k, rep, axis=1), np.repeat(v, rep, axis=1)   # q head h uses kv head h//rep
        o = _merge_heads(causal_attention_fwd(q, ke, ve))
        x1 = x + o @ P[p + "wo"].T
        h2, c2 = rmsnorm_fwd(x1, P[p + "mlp_norm"], eps)
        a = h2 @ P[p + "wg"].T
        bu = h2 @ P[p + "wu"].T
        sa, sg = silu(a)
        f = sa * bu
        x = x1 + f @ P[p + "wd"].T
        caches.append((c1, h1, q, ke, ve, o, c2, h2, a, bu, sa, sg, f))
    xf, cf = rmsnorm_fwd(x, P["norm"], eps)
    w_head = P["tok"] if d.tie_embeddings else P["head.w"]
    logits = xf @ w_head.T
    loss, dlogits = cross_entropy(logits, tgt)

    G: Dict[str, np.ndarray] = {}
    dw_head = dlogits.T @ xf
    dx, G["norm"] = rmsnorm_bwd(dlogits @ w_head, cf)
    for l in reversed(range(d.n_layers)):
        p = f"h{l}."
        c1, h1, q, ke, ve, o, c2, h2, a, bu, sa, sg, f = caches[l]
        G[p + "wd"] = dx.T @ f
        df = dx @ P[p + "wd"]
        da = df * bu * sg * (1.0 + a * (1.0 - sg))
        db = df * sa
        G[p + "wg"] = da.T @ h2
        G[p + "wu"] = db.T @ h2
        dh2, G[p + "mlp_norm"] = rmsnorm_bwd(da @ P[p + "wg"] + db @ P[p + "wu"], c2)
        dx1 = dx + dh2
        G[p + "wo"] = dx1.T @ o
        do = _split_heads(dx1 @ P[p + "wo"], B, T, H, hd)
        dq, dke, dve = causal_attention_bwd(do, q, ke, ve)
        dk = dke.reshape(B, KV, rep, T, hd).sum(axis=2)
        dv = dve.reshape(B, KV, rep, T, hd).sum(axis=2)
        dq_lin = _merge_heads(rope_bwd(dq, cos, sin))
        dk_lin = _merge_heads(rope_bwd(dk, cos, sin))
        dv_lin = _merge_heads(dv)
        G[p + "wq"] = dq_lin.T @ h1
        G[p + "wk"] = dk_lin.T @ h1
        G[p + "wv"] = dv_lin.T @ h1
        dh1 = dq_lin @ P[p + "wq"] + dk_lin @ P[p + "wk"] + dv_lin @ P[p + "wv"]
        dh1, G[p + "attn_norm"] = rmsnorm_bwd(dh1, c1)
        dx = dx1 + dh1
    dtok = np.zeros_like(P["tok"])
    np.add.at(dtok, inp.reshape(-1), dx)
    if d.tie_embeddings:
        dtok = dtok + dw_head
    else:
        G["head.w"] = dw_head
    G["tok"] = dtok
    return loss, pack(G, d)


def loss_grad(theta, d, batch, dt=np.float64):
    """Dispatch: batch is (x, y) for the MLP, the token array [n_seq][T+1] otherwise."""
    if d.arch == ARCH_MLP:
        x, y = batch
        return mlp_loss_grad(theta, d, x, y, dt)
    if d.arch == ARCH_GPT:
        return gpt_loss_grad(theta, d, batch, dt)
    if d.arch == ARCH_LLAMA:
        return llama_loss_grad(theta, d, batch, dt)
    raise ValueError(d.arch)


def loss_only(theta, d, batch, dt=np.float64) -> float:
    return loss_grad(theta, d, batch, dt)[0]
