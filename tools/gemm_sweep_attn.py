"""Variant sweep of the batched causal attention GEMMs (c2: 32 batches, T = 256, hd = 64)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00816_b200 import slq  # noqa: E402
T, HD, NB = int(os.environ.get("T", 256)), int(os.environ.get("HD", 64)), int(os.environ.get("NB", 32))
os.environ["SLQ_DIAG_BATCH"] = str(NB)
SH = [("S=QK^T", T, T, HD, 1, 1, 1), ("PV", T, HD, T, 1, 0, 2), ("dV=P^T dO", T, HD, T, 0, 0, 3)]
for kind, M, N, K, ak, bk, tri in SH:
    os.environ["SLQ_DIAG_TRI"] = str(tri)
    res = []
    for v in [-1] + list(range(15)):
        t, c = ctypes.c_double(), ctypes.c_double()
        st = slq.lib().slq_diag_gemm_f64(0, M, N, K, ak, bk, v, 0, 30, ctypes.byref(t), ctypes.byref(c))
        if st == 0:
            res.append((round(t.value, 2), v, c.value))
    ref = [r for r in res if r[1] == -1][0]
    ok = all(abs(r[2] - ref[2]) <= 1e-9 * max(1.0, abs(ref[2])) for r in res)
    res.sort(reverse=True)
    print(json.dumps(dict(kind=kind, auto=ref[0], top=[r[:2] for r in res[:5]], checksums_agree=ok)), flush=True)
