"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module is the ONLY code both sides use.  It holds configuration data
(model dimensions, seeds, SLQ settings) and seeded generators for the initial
parameters theta_0 and the data batch.  It contains none of the method's
arithmetic: no loss, no gradient, no perturbation, no Lanczos, no probe.

Input recipe (SURVEY.md §8(c2) readings #11-#15, §8(d2)):
  * MLP (config c1): Xavier-uniform weights U(+-sqrt(6/(fan_in+fan_out))), zero
    biases; X ~ N(0,1) rounded to fp32; labels y ~ U{0..n_classes-1}.
  * GPT / Llama (c2-c5): every matrix and embedding ~ N(0, 0.02^2), biases 0,
    norm gains 1.  bf16 models round the init to bf16 (RNE); the fp32 master then
    holds exactly those values.
  * Tokens: Zipf(1.1) over the vocabulary (stand-in for wikitext-2 / the Pile,
    which the paper uses at P:464, P:481, P:602 and which are not available here).
    Sequence j is a pure function of (data_seed, j), so a larger global batch
    extends a smaller one.  Each sequence has seq_len+1 tokens: inputs tok[0:T],
    targets tok[1:T+1].

The canonical parameter order is layer-major, listed by `param_table`.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Tuple

import numpy as np

ARCH_MLP, ARCH_GPT, ARCH_LLAMA = 0, 1, 2


@dataclasses.dataclass(frozen=True)
class ModelDesc:
    """Model + data + SLQ settings of one workload (mirrors slq_model_desc in include/slq.h)."""
    name: str
    arch: int
    n_layers: int = 0
    d_model: int = 0
    n_heads: int = 0
    n_kv_heads: int = 0
    d_ff: int = 0
    vocab: int = 0
    seq_len: int = 0
    d_in: int = 0          # MLP only
    d_hidden: int = 0      # MLP only
    n_classes: int = 0     # MLP only
    tie_embeddings: bool = False
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    param_bf16: bool = False  # bf16-representable init (c3-c5)
    # data (global batch)
    n_seq: int = 0          # GPT/Llama: sequences in the global batch
    n_rows: int = 0         # MLP: rows in the batch
    # SLQ settings
    eps: float = 1e-3
    m: int = 32
    probes: int = 2
    reorth_full: bool = True
    # seeds
    init_seed: int = 0
    data_seed: int = 0
    probe_seed0: int = 0

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads if self.n_heads else 0


CONFIGS: Dict[str, ModelDesc] = {
    # configs[0] of BASELINE.json: tiny MLP, CPU-oracle scale
    "c1": ModelDesc(name="c1", arch=ARCH_MLP, d_in=64, d_hidden=128, n_classes=10,
                    n_rows=256, eps=1e-3, m=32, probes=2, reorth_full=True,
                    init_seed=1001, data_seed=2001, probe_seed0=3100),
    # configs[1]: small decoder-only transformer (fp32 model) -- the N=1 bench workload
    "c2": ModelDesc(name="c2", arch=ARCH_GPT, n_layers=4, d_model=256, n_heads=4,
                    n_kv_heads=4, d_ff=1024, vocab=4096, seq_len=256, n_seq=8,
                    eps=1e-3, m=64, probes=4, reorth_full=True,
                    init_seed=1002, data_seed=2002, probe_seed0=3200),
    # configs[2]: GPT-2-small shape (tied embeddings), bf16 weights, 8 seq per GPU
    "c3": ModelDesc(name="c3", arch=ARCH_GPT, n_layers=12, d_model=768, n_heads=12,
                    n_kv_heads=12, d_ff=3072, vocab=50257, seq_len=1024, n_seq=8,
                    tie_embeddings=True, param_bf16=True, eps=1e-3, m=100, probes=4,
                    reorth_full=True, init_seed=1003, data_seed=2003, probe_seed0=3300),
    # configs[3]: Llama-style 1B
    "c4": ModelDesc(name="c4", arch=ARCH_LLAMA, n_layers=16, d_model=2048, n_heads=32,
                    n_kv_heads=8, d_ff=8192, vocab=32000, seq_len=2048, n_seq=32,
                    rope_theta=10000.0, param_bf16=True, eps=1e-3, m=100, probes=4,
                    reorth_full=True, init_seed=1004, data_seed=2004, probe_seed0=3400),
    # configs[4]: Llama-3-8B shape
    "c5": ModelDesc(name="c5", arch=ARCH_LLAMA, n_layers=32, d_model=4096, n_heads=32,
                    n_kv_heads=8, d_ff=14336, vocab=128256, seq_len=2048, n_seq=16,
                    rope_theta=500000.0, param_bf16=True, eps=1e-3, m=64, probes=2,
                    reorth_full=False, init_seed=1005, data_seed=2005, probe_seed0=3500),
    # ---- small parity cases (same layer types, sizes the oracle finishes in seconds;
    #      ragged sizes so the kernels see partial tiles) ----
    "gpt_tiny": ModelDesc(name="gpt_tiny", arch=ARCH_GPT, n_layers=2, d_model=64, n_heads=2,
                          n_kv_heads=2, d_ff=160, vocab=203, seq_len=37, n_seq=3,
                          eps=1e-3, m=16, probes=1, init_seed=11, data_seed=12, probe_seed0=13),
    "gpt_tiny_tied": ModelDesc(name="gpt_tiny_tied", arch=ARCH_GPT, n_layers=1, d_model=48,
                               n_heads=3, n_kv_heads=3, d_ff=96, vocab=131, seq_len=29, n_seq=2,
                               tie_embeddings=True, eps=1e-3, m=12, probes=1,
                               init_seed=21, data_seed=22, probe_seed0=23),
    "llama_tiny": ModelDesc(name="llama_tiny", arch=ARCH_LLAMA, n_layers=2, d_model=64,
                            n_heads=4, n_kv_heads=2, d_ff=96, vocab=211, seq_len=33, n_seq=3,
                            rope_theta=10000.0, eps=1e-3, m=16, probes=1,
                            init_seed=31, data_seed=32, probe_seed0=33),
    # ---- parity batches of the large configs (same layer shapes) ----
    # c3 at R=1 with 2 of its 8 sequences
    "c3_parity": ModelDesc(name="c3_parity", arch=ARCH_GPT, n_layers=12, d_model=768, n_heads=12,
                           n_kv_heads=12, d_ff=3072, vocab=50257, seq_len=1024, n_seq=2,
                           tie_embeddings=True, param_bf16=True, eps=1e-3, m=3, probes=1,
                           reorth_full=True, init_seed=1003, data_seed=2003, probe_seed0=3300),
    # c4 (Llama 1B): 2 sequences of 256 tokens (SURVEY: 8 x 256 at R=8)
    "c4_parity": ModelDesc(name="c4_parity", arch=ARCH_LLAMA, n_layers=16, d_model=2048, n_heads=32,
                           n_kv_heads=8, d_ff=8192, vocab=32000, seq_len=256, n_seq=2,
                           rope_theta=10000.0, param_bf16=True, eps=1e-3, m=2, probes=1,
                           reorth_full=True, init_seed=1004, data_seed=2004, probe_seed0=3400),
    # c5 twin: every layer shape of Llama-3-8B, 2 blocks, 1 x 512 tokens, no stored basis
    "c5_twin": ModelDesc(name="c5_twin", arch=ARCH_LLAMA, n_layers=2, d_model=4096, n_heads=32,
                         n_kv_heads=8, d_ff=14336, vocab=128256, seq_len=512, n_seq=1,
                         rope_theta=500000.0, param_bf16=True, eps=1e-3, m=2, probes=1,
                         reorth_full=False, init_seed=1005, data_seed=2005, probe_seed0=3500),
    # c2 at twice the batch (diagnostic: what one pass costs at 2 x the rows)
    "c2x2": ModelDesc(name="c2x2", arch=ARCH_GPT, n_layers=4, d_model=256, n_heads=4, n_kv_heads=4,
                      d_ff=1024, vocab=4096, seq_len=256, n_seq=16, eps=1e-3, m=64, probes=4,
                      reorth_full=True, init_seed=1002, data_seed=2002, probe_seed0=3200),
    # GEMM-shape evidence only (not a c5 step): every Llama-3-8B layer shape at c5's per-GPU batch
    # (2 x 2048 tokens) on 2 of the 32 blocks
    "c5_gemm": ModelDesc(name="c5_gemm", arch=ARCH_LLAMA, n_layers=2, d_model=4096, n_heads=32,
                         n_kv_heads=8, d_ff=14336, vocab=128256, seq_len=2048, n_seq=2,
                         rope_theta=500000.0, param_bf16=True, eps=1e-3, m=8, probes=1,
                         reorth_full=False, init_seed=1005, data_seed=2005, probe_seed0=3500),
    "mlp_tiny": ModelDesc(name="mlp_tiny", arch=ARCH_MLP, d_in=7, d_hidden=9, n_classes=4,
                          n_rows=13, eps=1e-3, m=8, probes=1, init_seed=41, data_seed=42,
                          probe_seed0=43),
}


def get_config(name: str, **overrides) -> ModelDesc:
    return dataclasses.replace(CONFIGS[name], **overrides)


# --------------------------------------------------------------------------------------
# canonical parameter table (names, shapes, init kind); layer-major.
# --------------------------------------------------------------------------------------

def param_table(d: ModelDesc) -> List[Tuple[str, Tuple[int, ...], str]]:
    """(name, shape, kind) in canonical order; kind in {matrix, bias, gain, embed}."""
    t: List[Tuple[str, Tuple[int, ...], str]] = []
    if d.arch == ARCH_MLP:
        t += [("fc1.w", (d.d_hidden, d.d_in), "xavier"), ("fc1.b", (d.d_hidden,), "bias"),
              ("fc2.w", (d.n_classes, d.d_hidden), "xavier"), ("fc2.b", (d.n_classes,), "bias")]
        return t
    D, F, V = d.d_model, d.d_ff, d.vocab
    if d.arch == ARCH_GPT:
        t += [("wte", (V, D), "embed"), ("wpe", (d.seq_len, D), "embed")]
        for l in range(d.n_layers):
            p = f"h{l}."
            t += [(p + "ln1.g", (D,), "gain"), (p + "ln1.b", (D,), "bias"),
                  (p + "attn.qkv.w", (3 * D, D), "matrix"), (p + "attn.qkv.b", (3 * D,), "bias"),
                  (p + "attn.proj.w", (D, D), "matrix"), (p + "attn.proj.b", (D,), "bias"),
                  (p + "ln2.g", (D,), "gain"), (p + "ln2.b", (D,), "bias"),
                  (p + "mlp.fc.w", (F, D), "matrix"), (p + "mlp.fc.b", (F,), "bias"),
                  (p + "mlp.proj.w", (D, F), "matrix"), (p + "mlp.proj.b", (D,), "bias")]
        t += [("lnf.g", (D,), "gain"), ("lnf.b", (D,), "bias")]
        if not d.tie_embeddings:
            t += [("head.w", (V, D), "matrix")]
        return t
    if d.arch == ARCH_LLAMA:
        hd = d.head_dim
        t += [("tok", (V, D), "embed")]
        for l in range(d.n_layers):
            p = f"h{l}."
            t += [(p + "attn_norm.g", (D,), "gain"),
                  (p + "wq", (d.n_heads * hd, D), "matrix"),
                  (p + "wk", (d.n_kv_heads * hd, D), "matrix"),
                  (p + "wv", (d.n_kv_heads * hd, D), "matrix"),
                  (p + "wo", (D, d.n_heads * hd), "matrix"),
                  (p + "mlp_norm.g", (D,), "gain"),
                  (p + "w_gate", (F, D), "matrix"), (p + "w_up", (F, D), "matrix"),
                  (p + "w_down", (D, F), "matrix")]
        t += [("norm.g", (D,), "gain")]
        if not d.tie_embeddings:
            t += [("head.w", (V, D), "matrix")]
        return t
    raise ValueError(f"unknown arch {d.arch}")


def n_params(d: ModelDesc) -> int:
    return int(sum(int(np.prod(s)) for _, s, _ in param_table(d)))


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(list(key))))


def _round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (ties to even); returns fp32 holding bf16 values."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def init_params(d: ModelDesc) -> np.ndarray:
    """theta_0 as a flat fp32 vector in canonical order (host memory)."""
    parts = []
    for idx, (name, shape, kind) in enumerate(param_table(d)):
        n = int(np.prod(shape))
        g = _rng(d.init_seed, idx)
        if kind == "xavier":
            fan_out, fan_in = shape
            a = math.sqrt(6.0 / (fan_in + fan_out))
            x = g.uniform(-a, a, size=n)
        elif kind in ("matrix", "embed"):
            x = g.standard_normal(n) * 0.02
        elif kind == "bias":
            x = np.zeros(n)
        elif kind == "gain":
            x = np.ones(n)
        else:
            raise ValueError(kind)
        parts.append(x.astype(np.float32))
    theta = np.concatenate(parts) if parts else np.zeros(0, np.float32)
    if d.param_bf16:
        theta = _round_bf16(theta)
    return theta


def zipf_cdf(vocab: int, s: float = 1.1) -> np.ndarray:
    k = np.arange(1, vocab + 1, dtype=np.float64)
    p = k ** (-s)
    c = np.cumsum(p)
    return c / c[-1]


def tokens(d: ModelDesc, n_seq: int | None = None, first_seq: int = 0) -> np.ndarray:
    """Zipf(1.1) token ids, int32 [n_seq][seq_len+1]; sequence j depends only on (data_seed, j)."""
    n_seq = d.n_seq if n_seq is None else n_seq
    cdf = zipf_cdf(d.vocab)
    out = np.empty((n_seq, d.seq_len + 1), dtype=np.int32)
    for j in range(n_seq):
        u = _rng(d.data_seed, first_seq + j).random(d.seq_len + 1)
        out[j] = np.minimum(np.searchsorted(cdf, u, side="right"), d.vocab - 1)
    return out


def mlp_data(d: ModelDesc) -> Tuple[np.ndarray, np.ndarray]:
    """X fp32 [n_rows][d_in] ~ N(0,1), y int32 [n_rows] ~ U{0..n_classes-1}."""
    g = _rng(d.data_seed, 0)
    x = g.standard_normal((d.n_rows, d.d_in)).astype(np.float32)
    y = _rng(d.data_seed, 1).integers(0, d.n_classes, size=d.n_rows).astype(np.int32)
    return x, y


def split_counts(n: int, world: int) -> List[int]:
    """Rows / sequences per rank: the first n % world ranks get one extra (data-parallel slice)."""
    return [n // world + (1 if r < n % world else 0) for r in range(world)]


def rank_slice(n: int, rank: int, world: int) -> slice:
    c = split_counts(n, world)
    s = sum(c[:rank])
    return slice(s, s + c[rank])


def random_vector(n: int, seed: int) -> np.ndarray:
    """A generic seeded fp32 direction (for hvp tests with a non-unit v)."""
    return _rng(seed, 77).standard_normal(n).astype(np.float32)
