#!/bin/bash
# call F: c4 goldens (no basis m = 16, then full reorthogonalisation m = 6) on the host in the
# background; GPU: the c4 (Llama-1B shape) and c5-shape bench lines
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O/golden
(
  OPENBLAS_NUM_THREADS=14 timeout 2700 python tests/golden/make_golden.py --case c4_parity --m 16 --eps 1e-3 --reorth none --mem-limit-gb 150 --out-dir $O/golden > $O/golden/c4n.log 2>&1
  OPENBLAS_NUM_THREADS=14 timeout 900 python tests/golden/make_golden.py --case c4_parity --m 6 --eps 1e-3 --reorth full --mem-limit-gb 175 --out-dir $O/golden > $O/golden/c4f.log 2>&1
) &
GP=$!
export SLQ_TIMEOUT_S=600
timeout 900 python bench.py --config c4 --act-ckpt --reorth none --probe-m 20 --steps 8 --warmup 3 --no-cpu-baseline > $O/b_r02f_c4_none.json 2> $O/b_r02f_c4_none.err
timeout 900 python bench.py --config c4 --act-ckpt --reorth window --window 8 --basis bf16 --probe-m 20 --steps 8 --warmup 3 --no-cpu-baseline > $O/b_r02f_c4_w8bf16.json 2> $O/b_r02f_c4_w8bf16.err
timeout 900 python bench.py --config c5_gemm --act-ckpt --probe-m 8 --steps 4 --warmup 2 --no-cpu-baseline > $O/b_r02f_c5gemm.json 2> $O/b_r02f_c5gemm.err
T=2048 HD=64 NB=64 timeout 900 python tools/gemm_sweep_attn.py > $O/sweep_attn_t2048.jsonl 2>&1
wait $GP
