#!/bin/bash
# call U: inline bias / residual epilogue with one-chunk-ahead loads (the forward linear GEMMs)
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 900 python -m pytest tests/test_gpu_oz.py tests/test_gpu_attn_oz.py tests/test_gpu_parity.py -q -s -k "error_bound or fp64_oz or attention or nonfinite or grad" --timeout 600 -p no:cacheprovider > $O/t_r02u.log 2>&1; echo "rc=$?" >> $O/t_r02u.log
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02u_c3.json 2> $O/b_r02u_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 1500 --csv --log-file $O/ncu_r02u_c3_launches.csv python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > $O/ncu_r02u_c3_launches.log 2>&1
timeout 900 python -m pytest tests/test_gpu_large.py -q -s -k "c3_lanczos" --timeout 600 -p no:cacheprovider > $O/t_r02u_large.log 2>&1; echo "rc=$?" >> $O/t_r02u_large.log
