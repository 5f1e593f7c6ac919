import ctypes, sys
sys.path.insert(0, '/root/repo')
from paper_2602_00816_b200 import slq
L = slq.lib()
for fn in ("slq_diag_fp64_peak", "slq_diag_dmma_peak"):
    f = getattr(L, fn); f.restype = ctypes.c_int32; f.argtypes = [ctypes.c_int32, ctypes.c_void_p]
    for _ in range(3):
        t = ctypes.c_double(); st = f(0, ctypes.byref(t)); print(fn, st, t.value)
