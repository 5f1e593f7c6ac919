"""The collective watchdog ("watchdog, then ncclCommAbort, then SLQ_ENCCL or
SLQ_ETIMEOUT on survivors") on one GPU.  A stall kernel stands in for a hung
collective: the wait must give up after the timeout with SLQ_ETIMEOUT, abort the context's NCCL
communicator (one-rank communicator, SLQ_FORCE_NCCL=1), and every later collective call must fail
with SLQ_ENCCL instead of hanging.  (A real peer failure needs two GPUs; the asynchronous-error
branch of the same wait loop is not exercised here.)"""
import os
import time

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


def _ctx(force):
    os.environ["SLQ_FORCE_NCCL"] = "1" if force else "0"
    try:
        cfg = si.CONFIGS["gpt_tiny"]
        th = si.init_params(cfg)
        return cfg, th, slq.SlqContext(cfg, th, si.tokens(cfg), max_steps=4)
    finally:
        os.environ["SLQ_FORCE_NCCL"] = "0"


def _hvp(c, cfg, th):
    lay = c.layout()
    v = torch.from_numpy(slq.shard_of(si.random_vector(th.size, 5), lay, 0, 1)).cuda()
    out = torch.empty_like(v)
    c.hvp(v, out, cfg.eps)
    return out.cpu().numpy()


def test_watchdog_without_communicator():
    cfg, th, c = _ctx(False)
    with c:
        ref = _hvp(c, cfg, th)
        assert c.diag_watchdog(10, 5.0) == slq.SLQ_OK
        t0 = time.time()
        assert c.diag_watchdog(1500, 0.2) == slq.SLQ_ETIMEOUT
        assert time.time() - t0 < 1.2  # gave up at the timeout, not at the end of the stall
        time.sleep(1.6)  # the stall kernel ends; with no communicator the context stays usable
        assert np.array_equal(_hvp(c, cfg, th), ref)
        assert c.diag_watchdog(0, 0.0) == slq.SLQ_OK


def test_watchdog_aborts_the_communicator():
    cfg, th, c = _ctx(True)
    with c:
        ref = _hvp(c, cfg, th)
        assert c.diag_watchdog(10, 5.0) == slq.SLQ_OK
        assert c.diag_watchdog(1500, 0.2) == slq.SLQ_ETIMEOUT
        time.sleep(1.6)
        with pytest.raises(slq.SlqError) as e:
            _hvp(c, cfg, th)
        assert e.value.status == slq.SLQ_ENCCL and "aborted" in str(e.value)
        with pytest.raises(slq.SlqError) as e:
            c.lanczos(cfg.probe_seed0, 4)
        assert e.value.status == slq.SLQ_ENCCL
    # a new context (new communicator) works again
    cfg, th, c2 = _ctx(True)
    with c2:
        assert np.array_equal(_hvp(c2, cfg, th), ref)


def test_watchdog_argument_check():
    cfg, th, c = _ctx(False)
    with c:
        assert c.diag_watchdog(-1, 1.0) == slq.SLQ_EINVAL
        assert c.diag_watchdog(20000, 1.0) == slq.SLQ_EINVAL
