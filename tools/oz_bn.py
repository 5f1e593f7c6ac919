"""Diagnostic: Ozaki GEMM rate for a shape at a given S (SLQ_OZ_BN selects 128-wide tiles for S = 4)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00816_b200 import slq  # noqa: E402
M, N, K, S = (int(x) for x in sys.argv[1:5])
e, t = slq.oz_check(M, N, K, True, True, S, iters=5)
print(f"oz {M}x{N}x{K} S={S} BN={os.environ.get('SLQ_OZ_BN', '64')}: err {e:.2e}, {t:.1f} TFLOP/s fp64-eq, "
      f"{t * S * (S + 1) / 2:.0f} TOP/s int8")
