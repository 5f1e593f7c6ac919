"""ctypes binding of libslq.so (include/slq.h).  Marshalling only."""
from __future__ import annotations

import ctypes
import os
import sys
from typing import List, Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslq.so")

SLQ_OK, SLQ_EINVAL, SLQ_ENUMERIC, SLQ_ECUDA, SLQ_ENCCL, SLQ_ETIMEOUT, SLQ_ENOMEM, SLQ_EUNSUPPORTED = 0, 2, 3, 4, 5, 6, 7, 8
PASS = {"fp64": 0, "fp32": 1, "bf16x3": 2, "paired": 3, "paired_fp32": 4, "fp64_oz": 5, "bf16": 6}
REORTH = {"none": 0, "full": 1, "window": 2}
BASIS = {"fp32": 0, "bf16": 1}
PERTURB = {"exact": 0, "storage": 1}


class SlqError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"slq status {status}: {msg}")
        self.status = status


class ModelDescC(ctypes.Structure):
    _fields_ = [("arch", ctypes.c_int32), ("n_layers", ctypes.c_int32), ("d_model", ctypes.c_int32),
                ("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32), ("d_ff", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("seq_len", ctypes.c_int32), ("d_in", ctypes.c_int32),
                ("d_hidden", ctypes.c_int32), ("n_classes", ctypes.c_int32),
                ("tie_embeddings", ctypes.c_int32), ("rope_theta", ctypes.c_double),
                ("norm_eps", ctypes.c_double), ("param_dtype", ctypes.c_int32),
                ("pass_numerics", ctypes.c_int32), ("reorth", ctypes.c_int32),
                ("max_steps", ctypes.c_int32), ("eps_default", ctypes.c_double),
                ("perturb", ctypes.c_int32), ("reorth_window", ctypes.c_int32),
                ("basis_dtype", ctypes.c_int32), ("oz_min_mnk", ctypes.c_double),
                ("oz_slices", ctypes.c_int32), ("act_ckpt", ctypes.c_int32)]


class BatchC(ctypes.Structure):
    _fields_ = [("params_host", ctypes.c_void_p), ("tokens", ctypes.c_void_p),
                ("n_seq_local", ctypes.c_int32), ("n_seq_global", ctypes.c_int32),
                ("x", ctypes.c_void_p), ("y", ctypes.c_void_p),
                ("n_rows_local", ctypes.c_int32), ("n_rows_global", ctypes.c_int32)]


class WorldC(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world_size", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("cuda_stream", ctypes.c_void_p),
                ("comm_backend", ctypes.c_int32)]


COMM = {"nccl": 0, "loopback": 1}
MEM_NAMES = ["theta", "points", "grads", "lanczos", "fsdp", "activations", "logits", "scratch", "workspace",
             "total"]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libslq.so; raises if it has not been built (no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SlqError(SLQ_ECUDA, f"{LIB_PATH} missing: build it with `python -m paper_2602_00816_b200.build`")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, D, U64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
    sig = {
        "slq_init": (I32, [ctypes.POINTER(ModelDescC), ctypes.POINTER(BatchC), ctypes.POINTER(WorldC), ctypes.POINTER(P)]),
        "slq_destroy": (I32, [P]),
        "slq_last_error": (ctypes.c_char_p, [P]),
        "slq_local_len": (I64, [P]),
        "slq_global_len": (I64, [P]),
        "slq_num_units": (I32, [P]),
        "slq_unit_info": (I32, [P, I32, P, P, P, P]),
        "slq_plan_layout": (I32, [ctypes.POINTER(ModelDescC), I32, P, P, P, P]),
        "slq_nccl_unique_id": (I32, [P]),
        "slq_hvp": (I32, [P, P, P, D]),
        "slq_grad": (I32, [P, P, P]),
        "slq_lanczos": (I32, [P, U64, I32, P, P]),
        "slq_lanczos_info": (I32, [P, P, P, P]),
        "slq_slq": (I32, [P, P, I32, I32, P, P, P]),
        "slq_quadrature": (I32, [P, P, I32, P, P]),
        "slq_ghost_clusters": (I32, [P, I32, D, P, P, P]),
        "slq_density": (I32, [P, P, P, I32, I32, P, P, I32, D, P]),
        "slq_probe": (I32, [P, U64, P]),
        "slq_profile": (I32, [P, I32, I32]),
        "slq_num_kernel_classes": (I32, []),
        "slq_kernel_class_name": (ctypes.c_char_p, [I32]),
        "slq_kernel_stats": (I32, [P, I32, P, P, P, P]),
        "slq_collective_counts": (I32, [P, P, P, P]),
        "slq_launch_count": (I64, [P]),
        "slq_stream": (P, [P]),
        "slq_diag_fp64_peak": (I32, [I32, P]),
        "slq_diag_dmma_peak": (I32, [I32, P]),
        "slq_diag_gemm_f64": (I32, [I32, I32, I32, I32, I32, I32, I32, I32, I32, P, P]),
        "slq_diag_oz_check": (I32, [I32, I32, I32, I32, I32, I32, I32, I32, P, P]),
        "slq_diag_attn_oz": (I32, [I32, I32, I32, I32, I32, I32, I32, I32, P, P]),
        "slq_diag_watchdog": (I32, [P, I32, D]),
        "slq_nonfinite_seq": (I32, [P, P]),
        "slq_cg": (I32, [P, P, P, D, I32, D, P, P]),
        "slq_blockdiag": (I32, [P, U64, P, P]),
        "slq_plan_memory": (I32, [ctypes.POINTER(ModelDescC), I32, I32, P]),
        "slq_lanczos_start": (I32, [P, U64, I32]),
        "slq_kernel_busy": (I32, [P, I32, P]),
        "slq_lanczos_step": (I32, [P, I32]),
        "slq_lanczos_result": (I32, [P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(st: int, ctx=None) -> None:
    if st != SLQ_OK:
        msg = lib().slq_last_error(ctx)
        raise SlqError(st, msg.decode() if msg else "")


def make_desc(cfg, pass_numerics: str = "fp64", reorth: Optional[str] = None, max_steps: Optional[int] = None,
              eps: Optional[float] = None, perturb: str = "exact", window: int = 0,
              basis: str = "fp32", oz_min_mnk: float = 0.0, oz_slices: int = 0, act_ckpt: bool = False) -> ModelDescC:
    """slq_model_desc from a slq_inputs.ModelDesc-like object."""
    d = ModelDescC()
    d.arch = cfg.arch
    for f in ("n_layers", "d_model", "n_heads", "n_kv_heads", "d_ff", "vocab", "seq_len", "d_in", "d_hidden",
              "n_classes"):
        setattr(d, f, int(getattr(cfg, f)))
    d.tie_embeddings = int(bool(cfg.tie_embeddings))
    d.rope_theta = float(cfg.rope_theta)
    d.norm_eps = float(cfg.norm_eps)
    d.param_dtype = 1 if getattr(cfg, "param_bf16", False) else 0
    d.pass_numerics = PASS[pass_numerics]
    d.reorth = REORTH[reorth if reorth is not None else ("full" if cfg.reorth_full else "none")]
    d.max_steps = int(max_steps if max_steps is not None else cfg.m)
    d.eps_default = float(eps if eps is not None else cfg.eps)
    d.perturb = PERTURB[perturb]
    d.reorth_window = int(window)
    d.basis_dtype = BASIS[basis]
    d.oz_min_mnk = float(oz_min_mnk)
    d.oz_slices = int(oz_slices)
    d.act_ckpt = int(bool(act_ckpt))
    return d


def plan_memory(desc: ModelDescC, world_size: int, n_local: int) -> dict:
    """Per-rank device-memory plan in bytes by category (slq_plan_memory; host only)."""
    out = np.zeros(len(MEM_NAMES), dtype=np.int64)
    _check(lib().slq_plan_memory(ctypes.byref(desc), int(world_size), int(n_local), out.ctypes.data))
    return dict(zip(MEM_NAMES, (int(x) for x in out)))


def plan_layout(desc: ModelDescC, world_size: int) -> dict:
    L = lib()
    P, Pl, nu = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
    _check(L.slq_plan_layout(ctypes.byref(desc), world_size, ctypes.byref(P), ctypes.byref(Pl), ctypes.byref(nu), None))
    tab = np.zeros((nu.value, 4), dtype=np.int64)
    _check(L.slq_plan_layout(ctypes.byref(desc), world_size, None, None, None, tab.ctypes.data))
    return {"P": P.value, "P_loc": Pl.value, "units": tab}


def shard_of(full: np.ndarray, layout: dict, rank: int, world_size: int) -> np.ndarray:
    """This rank's local shard (padding zero) of a full canonical-order vector (host marshalling)."""
    out = np.zeros(layout["P_loc"], dtype=full.dtype)
    for g, numel, loc, chunk in layout["units"]:
        s = rank * chunk
        e = min(numel, s + chunk)
        if e > s:
            out[loc:loc + (e - s)] = full[g + s:g + e]
    return out


def unshard(shards, layout: dict) -> np.ndarray:
    """Inverse of shard_of over all ranks' shards."""
    full = np.zeros(layout["P"], dtype=shards[0].dtype)
    for r, sh in enumerate(shards):
        for g, numel, loc, chunk in layout["units"]:
            s = r * chunk
            e = min(numel, s + chunk)
            if e > s:
                full[g + s:g + e] = sh[loc:loc + (e - s)]
    return full


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().slq_nccl_unique_id(buf))
    return buf.raw


def fp64_peak_tflops(device: int = 0) -> dict:
    """Measured FP64 peaks: DFMA (SIMT pipe) and DMMA (fp64 tensor core), TFLOP/s (best of 3)."""
    out = {}
    for key, fn in (("dfma", lib().slq_diag_fp64_peak), ("dmma", lib().slq_diag_dmma_peak)):
        best = 0.0
        for _ in range(3):
            t = ctypes.c_double()
            _check(fn(device, ctypes.byref(t)))
            best = max(best, t.value)
        out[key] = best
    return out


def oz_check(M: int, N: int, K: int, a_kmajor: bool = True, b_kmajor: bool = True, S: int = 6, iters: int = 5,
             device: int = 0) -> Tuple[float, float]:
    """(max normalised error vs the DMMA fp64 GEMM, fp64-equivalent TFLOP/s) of the Ozaki GEMM."""
    e, t = ctypes.c_double(), ctypes.c_double()
    _check(lib().slq_diag_oz_check(device, M, N, K, int(a_kmajor), int(b_kmajor), S, iters, ctypes.byref(e),
                                   ctypes.byref(t)))
    return e.value, t.value


def attn_oz_check(nseq: int, Tn: int, Hq: int, Hkv: int, hd: int, S: int = 5, iters: int = 0,
                  device: int = 0) -> Tuple[List[float], Tuple[float, float]]:
    """Causal attention fwd + bwd on random data, FP64_OZ path (batched INT8 Ozaki GEMMs) vs the
    FP64 DMMA path: ([max-norm relative error of O, dQ, dK, dV], (ms DMMA, ms Ozaki))."""
    e = (ctypes.c_double * 4)()
    t = (ctypes.c_double * 2)()
    _check(lib().slq_diag_attn_oz(device, nseq, Tn, Hq, Hkv, hd, S, iters, e, t))
    return list(e), (t[0], t[1])


def kernel_class_names():
    L = lib()
    return [L.slq_kernel_class_name(i).decode() for i in range(L.slq_num_kernel_classes())]


def quadrature(alpha, beta) -> Tuple[np.ndarray, np.ndarray]:
    a = np.ascontiguousarray(alpha, dtype=np.float64)
    b = np.ascontiguousarray(beta, dtype=np.float64)
    m = a.size
    nodes, w = np.empty(m), np.empty(m)
    _check(lib().slq_quadrature(a.ctypes.data, b.ctypes.data if b.size else None, m, nodes.ctypes.data,
                                w.ctypes.data))
    return nodes, w


def density(node_sets, weight_sets, jmax: int = 2, grid=None, sigma: float = 0.0):
    """Probe-averaged moments [jmax + 1] and (if grid is given) the smoothed density -- slq_density."""
    mc = np.array([len(n) for n in node_sets], dtype=np.int32)
    nodes = np.ascontiguousarray(np.concatenate(node_sets), dtype=np.float64)
    w = np.ascontiguousarray(np.concatenate(weight_sets), dtype=np.float64)
    mom = np.empty(jmax + 1)
    g = None if grid is None else np.ascontiguousarray(grid, dtype=np.float64)
    dens = None if g is None else np.empty(g.size)
    _check(lib().slq_density(nodes.ctypes.data, w.ctypes.data, mc.ctypes.data, mc.size, jmax, mom.ctypes.data,
                             g.ctypes.data if g is not None else None, 0 if g is None else g.size, float(sigma),
                             dens.ctypes.data if dens is not None else None))
    return mom, dens


def ghost_clusters(nodes, tol: float) -> Tuple[np.ndarray, int, float]:
    """(cluster id per node, number of duplicate clusters, largest splitting) -- slq_ghost_clusters."""
    x = np.ascontiguousarray(nodes, dtype=np.float64)
    ids = np.empty(x.size, dtype=np.int32)
    ng, ms = ctypes.c_int32(), ctypes.c_double()
    _check(lib().slq_ghost_clusters(x.ctypes.data, x.size, float(tol), ids.ctypes.data, ctypes.byref(ng),
                                    ctypes.byref(ms)))
    return ids, ng.value, ms.value


def _torch_fence() -> None:
    """The library orders its calls after the legacy default stream (slq.h, slq_world.cuda_stream);
    if torch is writing shards on another current stream, wait for that stream first."""
    t = sys.modules.get("torch")
    if t is None or not t.cuda.is_available() or not t.cuda.is_initialized():
        return
    s = t.cuda.current_stream()
    if s.cuda_stream != 0:
        s.synchronize()


def _ptr(x) -> int:
    """Raw pointer of a torch tensor (device or host) or numpy array."""
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data
    assert x.is_contiguous()
    return x.data_ptr()


class SlqContext:
    """One process / GPU.  theta0: full canonical fp32 vector (host); batch: this rank's slice."""

    def __init__(self, cfg, theta0: np.ndarray, batch, *, n_global: Optional[int] = None, rank: int = 0,
                 world_size: int = 1, device: int = 0, stream: Optional[int] = None, unique_id: Optional[bytes] = None,
                 pass_numerics: str = "fp64", reorth: Optional[str] = None, max_steps: Optional[int] = None,
                 eps: Optional[float] = None, perturb: str = "exact", window: int = 0, basis: str = "fp32",
                 oz_min_mnk: float = 0.0, oz_slices: int = 0, act_ckpt: bool = False, comm: str = "nccl"):
        L = lib()
        self._keep = []
        self.desc = make_desc(cfg, pass_numerics, reorth, max_steps, eps, perturb, window, basis, oz_min_mnk,
                              oz_slices, act_ckpt)
        th = np.ascontiguousarray(theta0, dtype=np.float32)
        b = BatchC()
        b.params_host = th.ctypes.data
        self._keep.append(th)
        if cfg.arch == 0:
            x, y = batch
            x = np.ascontiguousarray(x, dtype=np.float32)
            y = np.ascontiguousarray(y, dtype=np.int32)
            self._keep += [x, y]
            b.x, b.y = x.ctypes.data, y.ctypes.data
            b.n_rows_local = x.shape[0]
            b.n_rows_global = n_global if n_global is not None else x.shape[0]
        else:
            tok = np.ascontiguousarray(batch, dtype=np.int32)
            self._keep.append(tok)
            b.tokens = tok.ctypes.data
            b.n_seq_local = tok.shape[0]
            b.n_seq_global = n_global if n_global is not None else tok.shape[0]
        w = WorldC()
        w.rank, w.world_size, w.device = rank, world_size, device
        uid = None
        if world_size > 1:
            assert unique_id is not None and len(unique_id) == 128
            uid = ctypes.create_string_buffer(unique_id, 128)
            w.nccl_unique_id = ctypes.cast(uid, ctypes.c_void_p)
        w.cuda_stream = stream
        w.comm_backend = COMM[comm]
        h = ctypes.c_void_p()
        _check(L.slq_init(ctypes.byref(self.desc), ctypes.byref(b), ctypes.byref(w), ctypes.byref(h)))
        self._h = h
        self._keep = None
        self.rank, self.world_size = rank, world_size
        self.P_loc = L.slq_local_len(h)
        self.P = L.slq_global_len(h)

    # -- lifetime
    def close(self):
        if getattr(self, "_h", None):
            lib().slq_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- layout
    def layout(self) -> dict:
        L = lib()
        nu = L.slq_num_units(self._h)
        tab = np.zeros((nu, 4), dtype=np.int64)
        for u in range(nu):
            vals = [ctypes.c_int64() for _ in range(4)]
            _check(L.slq_unit_info(self._h, u, *[ctypes.byref(v) for v in vals]), self._h)
            tab[u] = [v.value for v in vals]
        return {"P": self.P, "P_loc": self.P_loc, "units": tab}

    @property
    def stream(self) -> int:
        return lib().slq_stream(self._h)

    # -- the path
    def hvp(self, v, out, eps: float) -> None:
        _torch_fence()
        _check(lib().slq_hvp(self._h, _ptr(v), _ptr(out), float(eps)), self._h)

    def grad(self, g=None) -> float:
        loss = ctypes.c_double()
        _torch_fence()
        _check(lib().slq_grad(self._h, _ptr(g) if g is not None else None, ctypes.byref(loss)), self._h)
        return loss.value

    def lanczos(self, seed: int, m: int) -> Tuple[np.ndarray, np.ndarray]:
        a = np.empty(m)
        b = np.empty(max(m - 1, 1))
        _check(lib().slq_lanczos(self._h, ctypes.c_uint64(seed), m, a.ctypes.data, b.ctypes.data), self._h)
        return a, b[:m - 1]

    def lanczos_start(self, seed: int, m: int) -> None:
        self._m = m
        _check(lib().slq_lanczos_start(self._h, ctypes.c_uint64(seed), m), self._h)

    def lanczos_step(self, n: int) -> None:
        _check(lib().slq_lanczos_step(self._h, n), self._h)

    def lanczos_result(self) -> Tuple[np.ndarray, np.ndarray]:
        m = self._m
        a = np.empty(m)
        b = np.empty(max(m - 1, 1))
        _check(lib().slq_lanczos_result(self._h, a.ctypes.data, b.ctypes.data), self._h)
        return a, b[:m - 1]

    def slq(self, seeds, m: int):
        """All probes' (alpha [s][m], beta [s][m-1], m_done [s]) -- slq_slq."""
        sd = np.ascontiguousarray(seeds, dtype=np.uint64)
        a = np.empty((sd.size, m))
        b = np.empty((sd.size, max(m - 1, 1)))
        md = np.empty(sd.size, dtype=np.int32)
        _check(lib().slq_slq(self._h, sd.ctypes.data, sd.size, m, a.ctypes.data, b.ctypes.data, md.ctypes.data),
               self._h)
        return a, b[:, :m - 1], md

    def lanczos_info(self) -> dict:
        md, bn, nf = ctypes.c_int32(), ctypes.c_double(), ctypes.c_int32()
        _check(lib().slq_lanczos_info(self._h, ctypes.byref(md), ctypes.byref(bn), ctypes.byref(nf)), self._h)
        return {"m_done": md.value, "beta_next": bn.value, "nonfinite": nf.value}

    def cg(self, b, x, damping: float, max_iter: int, tol: float = 0.0):
        it, rr = ctypes.c_int32(), ctypes.c_double()
        _torch_fence()
        _check(lib().slq_cg(self._h, _ptr(b), _ptr(x), float(damping), int(max_iter), float(tol), ctypes.byref(it),
                            ctypes.byref(rr)), self._h)
        return it.value, rr.value

    def blockdiag(self, seed: int):
        nu = lib().slq_num_units(self._h)
        rel, cos = np.empty(nu), np.empty(nu)
        _check(lib().slq_blockdiag(self._h, ctypes.c_uint64(seed), rel.ctypes.data, cos.ctypes.data), self._h)
        return rel, cos

    def probe(self, seed: int, q) -> None:
        _torch_fence()
        _check(lib().slq_probe(self._h, ctypes.c_uint64(seed), _ptr(q)), self._h)

    # -- measurement
    def profile(self, enable, reset: bool = False) -> None:
        """enable: False / True (= 1, serial) / "overlap" (= 2, concurrency kept, busy times)."""
        mode = 2 if enable == "overlap" else int(bool(enable))
        _check(lib().slq_profile(self._h, mode, int(reset)), self._h)

    def kernel_busy(self, cls: int = -1) -> float:
        b = ctypes.c_double()
        _check(lib().slq_kernel_busy(self._h, int(cls), ctypes.byref(b)), self._h)
        return b.value

    def kernel_stats(self) -> dict:
        L = lib()
        out = {}
        for i, name in enumerate(kernel_class_names()):
            ms, n, fl, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
            _check(L.slq_kernel_stats(self._h, i, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl), ctypes.byref(by)),
                   self._h)
            out[name] = {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value,
                         "busy_ms": self.kernel_busy(i)}
        return out

    def collective_counts(self) -> dict:
        ag, rs, ar = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(lib().slq_collective_counts(self._h, ctypes.byref(ag), ctypes.byref(rs), ctypes.byref(ar)), self._h)
        return {"allgather": ag.value, "reduce_scatter": rs.value, "allreduce": ar.value}

    def nonfinite_seq(self) -> int:
        """Local sequence (MLP: row) whose loss was non-finite in the last failing hvp, else -1."""
        q = ctypes.c_int32()
        _check(lib().slq_nonfinite_seq(self._h, ctypes.byref(q)), self._h)
        return q.value

    def diag_watchdog(self, stall_ms: int, timeout_s: float) -> int:
        """Stall the context's stream for stall_ms, wait through the collective watchdog with
        timeout_s; returns the status code (SLQ_ETIMEOUT when the stall outlasts the timeout)."""
        return int(lib().slq_diag_watchdog(self._h, int(stall_ms), float(timeout_s)))

    def launch_count(self) -> int:
        return lib().slq_launch_count(self._h)
