"""Time the production fp64 GEMM on arbitrary shapes (diagnostic)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00816_b200 import slq
for spec in sys.argv[1:]:
    M, N, K, ak, bk, v = (int(x) for x in spec.split(","))
    t, c = ctypes.c_double(), ctypes.c_double()
    st = slq.lib().slq_diag_gemm_f64(0, M, N, K, ak, bk, v, 0, 10, ctypes.byref(t), ctypes.byref(c))
    print(spec, st, round(t.value, 2))
