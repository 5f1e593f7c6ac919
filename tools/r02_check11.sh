#!/bin/bash
# call K: Ozaki attention (oz_attn.cu) vs DMMA attention; staged-store epilogue; c3 parity, bench, launch list
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 600 python -m pytest tests/test_gpu_attn_oz.py -q -s --timeout 500 -p no:cacheprovider > $O/t_r02k_attn.log 2>&1; echo "rc=$?" >> $O/t_r02k_attn.log
timeout 900 python -m pytest tests/test_gpu_oz.py tests/test_gpu_large.py -q -s -k "error_bound or fp64_oz_grad or fp64_oz_lanczos or nonfinite or c3_lanczos" --timeout 600 -p no:cacheprovider > $O/t_r02k.log 2>&1; echo "rc=$?" >> $O/t_r02k.log
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02k_c3.json 2> $O/b_r02k_c3.err
SLQ_ATTN_DMMA=1 timeout 900 python bench.py --no-cpu-baseline > $O/b_r02k_c3_attn_dmma.json 2> $O/b_r02k_c3_attn_dmma.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 2700 --csv --log-file $O/ncu_r02k_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > $O/ncu_r02k_c3_launches.log 2>&1
