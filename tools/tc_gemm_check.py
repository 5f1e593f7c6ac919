"""Check and time the tcgen05 bf16 GEMM diagnostic against a naive reference (diagnostic)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00816_b200 import slq
L = slq.lib()
f = L.slq_diag_gemm_bf16
f.restype = ctypes.c_int32
f.argtypes = [ctypes.c_int32] * 6 + [ctypes.c_void_p, ctypes.c_void_p]
for spec in sys.argv[1:]:
    M, N, K, v = (int(x) for x in spec.split(","))
    t, e = ctypes.c_double(), ctypes.c_double()
    st = f(0, M, N, K, v, 5, ctypes.byref(t), ctypes.byref(e))
    print(spec, "status", st, "TFLOP/s", round(t.value, 1), "max rel err", e.value, flush=True)
