"""Diagnostic: run the production fp64 DMMA GEMM plan on one shape (for ncu captures)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00816_b200 import slq  # noqa: E402
M, N, K, ak, bk = (int(x) for x in sys.argv[1:6])
v = int(sys.argv[6]) if len(sys.argv) > 6 else -1
t, c = ctypes.c_double(), ctypes.c_double()
assert slq.lib().slq_diag_gemm_f64(0, M, N, K, ak, bk, v, 0, 20, ctypes.byref(t), ctypes.byref(c)) == 0
print(f"dmma {M}x{N}x{K} ak={ak} bk={bk} v={v}: {t.value:.1f} TFLOP/s")
