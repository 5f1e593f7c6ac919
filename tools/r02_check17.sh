#!/bin/bash
# call Q: rows slicer with 4 values per lane, 8-column cols slicer, interleaved bwd-emit phase 1
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 600 python -m pytest tests/test_gpu_attn_oz.py tests/test_gpu_oz.py -q -s -k "attention or nonfinite or fp64_oz_grad" --timeout 500 -p no:cacheprovider > $O/t_r02q_attn.log 2>&1; echo "rc=$?" >> $O/t_r02q_attn.log
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02q_c3.json 2> $O/b_r02q_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 1500 --csv --log-file $O/ncu_r02q_c3_launches.csv python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > $O/ncu_r02q_c3_launches.log 2>&1
timeout 900 python -m pytest tests/test_gpu_large.py -q -s -k "c3_lanczos or c5" --timeout 600 -p no:cacheprovider > $O/t_r02q.log 2>&1; echo "rc=$?" >> $O/t_r02q.log
