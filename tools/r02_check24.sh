#!/bin/bash
# call X: TMA-store epilogue for the single-k-tile attention GEMMs (S = QK^T, dP = dO V^T)
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 600 python -m pytest tests/test_gpu_attn_oz.py tests/test_gpu_oz.py -q -s -k "attention or nonfinite or fp64_oz_grad or error_bound" --timeout 500 -p no:cacheprovider > $O/t_r02x.log 2>&1; echo "rc=$?" >> $O/t_r02x.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/ncu_attn_ts.csv python tools/attn_debug.py run > $O/attn_ts.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02x_c3.json 2> $O/b_r02x_c3.err
timeout 900 python -m pytest tests/test_gpu_large.py -q -s -k "c3_lanczos or c5" --timeout 600 -p no:cacheprovider > $O/t_r02x_large.log 2>&1; echo "rc=$?" >> $O/t_r02x_large.log
