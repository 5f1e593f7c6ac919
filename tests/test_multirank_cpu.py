"""World-size-2 (gloo, CPU) tests of the sharded path's host logic (§8(e)).

Each rank owns the chunk of every FSDP unit that `slq_plan_layout` assigns it and a slice of the
sequences.  The exchange steps of the GPU path are reproduced with gloo collectives around the
oracle's per-rank gradients:
  * ZeRO-3 all-gather of the perturbed unit shards  -> every rank sees the full perturbed theta;
  * per-unit reduce-scatter(sum) of the 1/N_global-scaled per-rank gradients -> the shard of
    grad L of the GLOBAL batch;
  * fp64 all-reduce of shard-local partial dot products -> the global Lanczos scalars.
The assembled sharded FD-HVP must equal the single-process oracle HVP, and the partial-dot
all-reduce must equal the global dot (R-equivalence).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import slq_inputs as si


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import fdhvp, models
        from paper_2602_00816_b200 import slq

        cfg = si.CONFIGS[name]
        th = si.init_params(cfg)
        P = th.size
        lay = slq.plan_layout(slq.make_desc(cfg), world)
        tok = si.tokens(cfg)
        n = tok.shape[0]
        mine = tok[si.rank_slice(n, rank, world)]
        v = si.random_vector(P, 3).astype(np.float64)
        eps = cfg.eps

        # shard-local state
        th_sh = slq.shard_of(th.astype(np.float64), lay, rank, world)
        v_sh = slq.shard_of(v, lay, rank, world)
        # (1) ||v||^2 from shard-local partials + all-reduce (the one scalar AR of P:197)
        ss = torch.tensor([float(v_sh @ v_sh)], dtype=torch.float64)
        dist.all_reduce(ss)
        nv = float(np.sqrt(ss.item()))
        eta = eps / nv
        out = {}
        for sign in (+1, -1):
            pert_sh = th_sh + sign * eta * v_sh           # out-of-place shard perturbation
            # (2) ZeRO-3 all-gather of every unit's chunks -> full perturbed theta
            gathered = [torch.zeros_like(torch.from_numpy(pert_sh)) for _ in range(world)]
            dist.all_gather(gathered, torch.from_numpy(pert_sh))
            full = slq.unshard([g.numpy() for g in gathered], lay)
            # per-rank gradient of this rank's slice, scaled to the global-batch mean (R1)
            g_loc = models.loss_grad(full, cfg, mine)[1] * (mine.shape[0] / n)
            # (3) reduce-scatter(sum) per unit == all-reduce then keep own chunk
            g_full = torch.from_numpy(g_loc.copy())
            dist.all_reduce(g_full)
            out[sign] = slq.shard_of(g_full.numpy(), lay, rank, world)
        hv_sh = (out[+1] - out[-1]) / (2 * eta)
        # (4) Lanczos scalars from partials
        a_part = torch.tensor([float(hv_sh @ v_sh), float(hv_sh @ hv_sh)], dtype=torch.float64)
        dist.all_reduce(a_part)
        shards = [torch.zeros(lay["P_loc"], dtype=torch.float64) for _ in range(world)]
        dist.all_gather(shards, torch.from_numpy(hv_sh))
        if rank == 0:
            hv = slq.unshard([s.numpy() for s in shards], lay)
            ref = fdhvp.hvp(fdhvp.make_grad_fn(cfg, tok), th.astype(np.float64), v, eps, "exact")
            q.put(("ok", float(np.linalg.norm(hv - ref) / np.linalg.norm(ref)),
                   float(abs(a_part[0].item() - hv @ v) / abs(hv @ v)),
                   float(abs(a_part[1].item() - hv @ hv) / (hv @ hv))))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced through the queue
        import traceback
        q.put(("err", traceback.format_exc()))


@pytest.mark.parametrize("name", ["gpt_tiny", "llama_tiny"])
def test_sharded_fd_hvp_matches_oracle_world2(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert res[0] == "ok", res[1]
    _, hv_err, dot_err, nrm_err = res
    assert hv_err < 1e-10
    assert dot_err < 1e-12 and nrm_err < 1e-12


def test_layout_chunks_are_rank_disjoint_and_complete():
    """Every real parameter is owned by exactly one rank; padding only at unit tails."""
    from paper_2602_00816_b200 import slq
    for name in ("gpt_tiny", "llama_tiny", "c2"):
        cfg = si.CONFIGS[name]
        P = si.n_params(cfg)
        for world in (2, 4, 8):
            lay = slq.plan_layout(slq.make_desc(cfg), world)
            ids = np.arange(P, dtype=np.int64) + 1
            shards = [slq.shard_of(ids, lay, r, world) for r in range(world)]
            allv = np.concatenate(shards)
            allv = allv[allv > 0]
            assert np.array_equal(np.sort(allv), ids)
