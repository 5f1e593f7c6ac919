#!/bin/bash
# call W: c4 and c5-shape lines with the Ozaki attention (T = 2048, GQA, hd 128), and their DMMA-attention twins
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python bench.py --config c4 --act-ckpt --reorth none --steps 8 --warmup 6 --no-cpu-baseline > $O/b_r02w_c4.json 2> $O/b_r02w_c4.err
timeout 600 python bench.py --config c5_gemm --act-ckpt --reorth none --steps 4 --warmup 2 --probe-m 8 --no-cpu-baseline > $O/b_r02w_c5gemm.json 2> $O/b_r02w_c5gemm.err
SLQ_ATTN_DMMA=1 timeout 600 python bench.py --config c5_gemm --act-ckpt --reorth none --steps 4 --warmup 2 --probe-m 8 --no-cpu-baseline > $O/b_r02w_c5gemm_dmma.json 2> $O/b_r02w_c5gemm_dmma.err
