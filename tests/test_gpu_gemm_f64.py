"""fp64 DMMA GEMM plans on the GPU: split-K (single and batched) and the tile variants compute the
same product as the unsplit plan, to fp64 summation-order rounding (the kernel-level pieces behind
the FP64 pass mode of DESIGN.md §5; the end-to-end parity is in test_gpu_parity.py)."""
import ctypes
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_00816_b200 import build
    build.build()


from paper_2602_00816_b200 import slq  # noqa: E402


def _run(M, N, K, ak, bk, variant, splits, batch=1):
    os.environ["SLQ_DIAG_BATCH"] = str(batch)
    try:
        t, c = ctypes.c_double(), ctypes.c_double()
        st = slq.lib().slq_diag_gemm_f64(0, M, N, K, ak, bk, variant, splits, 1, ctypes.byref(t), ctypes.byref(c))
        assert st == 0
        return c.value
    finally:
        del os.environ["SLQ_DIAG_BATCH"]


# (M, N, K, a_kmajor, b_kmajor): the weight-gradient shapes of c2 / c3 (dY^T . X, K = tokens)
@pytest.mark.parametrize("shape", [(256, 1024, 2048, 0, 0), (768, 256, 2048, 0, 0), (1000, 300, 2500, 0, 0),
                                   (256, 256, 4096, 1, 0)])
@pytest.mark.parametrize("batch", [1, 3])
def test_split_k_matches_unsplit(shape, batch):
    M, N, K, ak, bk = shape
    ref = _run(M, N, K, ak, bk, 0, 1, batch)
    for v, s in ((0, 4), (11, 8), (7, 3), (-1, 0)):
        got = _run(M, N, K, ak, bk, v, s, batch)
        assert abs(got - ref) <= 1e-12 * abs(ref), (v, s, got, ref)


def test_batched_split_k_writes_every_entry():
    """Batched split-K: 6 splits equal 1 split over all three entries, and the 3-entry checksum
    differs from the first entry's alone (entries 2 and 3 were written, not left zero)."""
    M, N, K = 256, 512, 3072
    one = _run(M, N, K, 0, 0, 0, 1, 1)
    b1 = _run(M, N, K, 0, 0, 0, 1, 3)
    b6 = _run(M, N, K, 0, 0, 0, 6, 3)
    assert abs(b6 - b1) <= 1e-12 * abs(b1)
    assert abs(b1 - one) > 1e-6 * abs(one)
