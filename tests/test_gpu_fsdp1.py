"""The FSDP code path (per-unit NCCL all-gather before each unit's forward / backward, per-unit
reduce-scatter of its gradient, NCCL scalar all-reduces; §8(e)) on ONE GPU through a
one-rank NCCL communicator (SLQ_FORCE_NCCL=1).  With one rank every collective is a copy, so the
results must be bit-identical to the local path -- this exercises the multi-GPU host logic,
buffer management, padding, side-stream ordering and NCCL-inside-CUDA-graph capture on the real
library, which the gloo CPU tests cannot."""
import os

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


def _run(cfg, force, numerics="fp64", m=8):
    os.environ["SLQ_FORCE_NCCL"] = "1" if force else "0"
    try:
        th = si.init_params(cfg)
        batch = si.mlp_data(cfg) if cfg.arch == si.ARCH_MLP else si.tokens(cfg)
        with slq.SlqContext(cfg, th, batch, pass_numerics=numerics, reorth="full", max_steps=m) as c:
            lay = c.layout()
            v = torch.from_numpy(slq.shard_of(si.random_vector(th.size, 5), lay, 0, 1)).cuda()
            g = torch.empty_like(v)
            loss = c.grad(g)
            out = torch.empty_like(v)
            c.hvp(v, out, cfg.eps)
            c.hvp(v, out, cfg.eps)  # second call replays the captured graphs
            a, b = c.lanczos(cfg.probe_seed0, m)
            cc = c.collective_counts()
        return loss, g.cpu().numpy(), out.cpu().numpy(), a, b, cc
    finally:
        os.environ["SLQ_FORCE_NCCL"] = "0"


@pytest.mark.parametrize("name,numerics", [("gpt_tiny", "fp64"), ("gpt_tiny_tied", "fp64"), ("llama_tiny", "fp64"),
                                           ("mlp_tiny", "fp64"), ("c2", "fp64_oz"), ("llama_tiny", "bf16x3")])
def test_fsdp_path_one_rank_bit_identical(name, numerics):
    cfg = si.CONFIGS[name]
    l0, g0, h0, a0, b0, c0 = _run(cfg, False, numerics)
    l1, g1, h1, a1, b1, c1 = _run(cfg, True, numerics)
    print(f"{name} [{numerics}]: collectives {c1}")
    assert c0 == {"allgather": 0, "reduce_scatter": 0, "allreduce": 0}
    assert c1["allgather"] > 0 and c1["reduce_scatter"] > 0 and c1["allreduce"] > 0
    assert l0 == l1
    assert np.array_equal(g0, g1)
    assert np.array_equal(h0, h1)
    assert np.array_equal(a0, a1) and np.array_equal(b0, b1)
