"""Variant x split-K sweep of the fp64 DMMA GEMM on the c2 shapes (diagnostic)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00816_b200 import slq  # noqa: E402
SH = [("fwd", 2048, 256, 256, 1, 1), ("dgrad", 2048, 256, 256, 1, 0), ("wgrad", 256, 256, 2048, 0, 0),
      ("fwd", 2048, 768, 256, 1, 1), ("dgrad", 2048, 256, 768, 1, 0), ("wgrad", 768, 256, 2048, 0, 0),
      ("fwd", 2048, 1024, 256, 1, 1), ("dgrad", 2048, 256, 1024, 1, 0), ("wgrad", 1024, 256, 2048, 0, 0),
      ("fwd", 2048, 256, 1024, 1, 1), ("wgrad", 256, 1024, 2048, 0, 0), ("wgrad", 4096, 256, 2048, 0, 0),
      ("dgrad", 2048, 256, 4096, 1, 0)]
for kind, M, N, K, ak, bk in SH:
    best = []
    for v in [-1, 0, 1, 2, 6, 7, 9, 11, 12, 14]:
        for s in ([0] if v == -1 else [1, 2, 3, 4, 6, 8]):
            t, c = ctypes.c_double(), ctypes.c_double()
            st = slq.lib().slq_diag_gemm_f64(0, M, N, K, ak, bk, v, s, 30, ctypes.byref(t), ctypes.byref(c))
            if st == 0:
                best.append((round(t.value, 2), v, s))
    best.sort(reverse=True)
    d = dict(kind=kind, M=M, N=N, K=K, auto=[b for b in best if b[1] == -1][0][0], top=best[:4])
    print(json.dumps(d), flush=True)
