"""Attention fwd+bwd time (c3 layer shape) with the Ozaki GEMM's diagnostic switches (SLQ_OZ_DEBUG
bits: 1 no MMAs, 2 no TMA loads, 4 no stores, 8 no TMEM drain) -- each setting in its own process."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1:
    from paper_2602_00816_b200 import slq
    err, (md, mo) = slq.attn_oz_check(8, 1024, 12, 12, 64, 5, iters=5)
    print(f"SLQ_OZ_DEBUG={os.environ.get('SLQ_OZ_DEBUG', '0')}: attention fwd+bwd Ozaki {mo:.3f} ms (DMMA {md:.3f})")
else:
    for d in ("0", "4", "8", "12", "1", "2"):
        env = dict(os.environ, SLQ_OZ_DEBUG=d)
        subprocess.run([sys.executable, __file__, "run"], env=env, check=False)
