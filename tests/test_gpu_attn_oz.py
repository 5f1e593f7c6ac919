"""Causal attention of the FP64_OZ passes (oz_attn.cu: the six contractions S = QK^T, O = PV,
dP = dO V^T, dV = P^T dO, dQ = dS K, dK = dS^T Q as batched INT8 Ozaki GEMMs on tcgen05, with the
digit planes of P and dS emitted by the softmax kernels) against the FP64 DMMA attention, forward and
backward, on random data: ragged-free tile grids of several 128-row blocks, GQA (Hq / Hkv > 1),
hd = 64 and 128, and S = 4..7 digit planes.

The gate follows the Ozaki error bound (oz_gemm.cu header): every contraction's error is at most
(S + 2) 2^-7S K max|A_i.| max|B_.j| (the transposed P / dS operands keep their row exponents, moved
into the other operand as exact powers of two, oz_attn.cu header), and the softmax and its
backward pass propagate it with O(1) gains for these inputs (|q|, |k| <= 2, |dO| <= 1); the test allows
64 (S + 2) 2^-7S max(T, hd) relative to each output's max norm."""
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


@pytest.mark.parametrize("nseq,T,Hq,Hkv,hd,S", [
    (2, 256, 4, 4, 64, 5),     # GPT shape, two 128-row blocks per head
    (1, 384, 2, 2, 64, 7),     # three blocks, the fp32 models' S
    (2, 256, 8, 2, 64, 5),     # GQA rep 4 (dV / dK accumulate over the query heads of a kv head)
    (1, 256, 4, 1, 128, 6),    # Llama head width, rep 4
    (1, 128, 3, 3, 96, 4),     # hd = 96 (three 32-column slicing blocks, ragged 64-wide tiles)
])
def test_attention_oz_vs_dmma(nseq, T, Hq, Hkv, hd, S):
    err, _ = slq.attn_oz_check(nseq, T, Hq, Hkv, hd, S)
    tol = 64 * (S + 2) * 2.0 ** (-7 * S) * max(T, hd)
    print(f"attn oz nseq={nseq} T={T} Hq={Hq} Hkv={Hkv} hd={hd} S={S}: O {err[0]:.2e} dQ {err[1]:.2e} "
          f"dK {err[2]:.2e} dV {err[3]:.2e} (tol {tol:.1e})")
    assert max(err) <= tol, err


def test_attention_oz_c3_shape_time():
    """c3's attention (8 x 1024 tokens, 12 heads of 64): errors at the bf16 models' S = 5 and the
    time of one forward + backward of each path (reported; the Ozaki path must not be slower)."""
    err, (ms_dmma, ms_oz) = slq.attn_oz_check(8, 1024, 12, 12, 64, 5, iters=3)
    tol = 64 * 7 * 2.0 ** -35 * 1024
    print(f"attn oz c3 layer: O {err[0]:.2e} dQ {err[1]:.2e} dK {err[2]:.2e} dV {err[3]:.2e}; "
          f"fwd+bwd DMMA {ms_dmma:.3f} ms, Ozaki {ms_oz:.3f} ms")
    assert max(err) <= tol, err
    assert ms_oz < ms_dmma
