"""Sweep the fp64 DMMA GEMM tile variants over the c2 gradient-pass shapes (diagnostic)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00816_b200 import slq  # noqa: E402

N_TOK, D, F, V = 2048, 256, 1024, 4096
SHAPES = []
for out_f, in_f in ((3 * D, D), (D, D), (F, D), (D, F), (V, D)):
    SHAPES.append(("fwd", N_TOK, out_f, in_f, 1, 1))
    SHAPES.append(("dgrad", N_TOK, in_f, out_f, 1, 0))
    SHAPES.append(("wgrad", out_f, in_f, N_TOK, 0, 0))


def run(M, N, K, ak, bk, v, s=0, iters=20):
    t, c = ctypes.c_double(), ctypes.c_double()
    st = slq.lib().slq_diag_gemm_f64(0, M, N, K, ak, bk, v, s, iters, ctypes.byref(t), ctypes.byref(c))
    assert st == 0, st
    return t.value, c.value


def main():
    variants = [int(x) for x in os.environ.get("VARIANTS", ",".join(map(str, range(15)))).split(",")]
    res = []
    for kind, M, N, K, ak, bk in SHAPES:
        row = {"kind": kind, "M": M, "N": N, "K": K}
        ref = None
        for v in [-1] + variants:
            tf, cs = run(M, N, K, ak, bk, v)
            if ref is None:
                ref = cs
            row[str(v)] = round(tf, 2)
            row["ok" + str(v)] = abs(cs - ref) <= 1e-9 * max(1.0, abs(ref))
        res.append(row)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
