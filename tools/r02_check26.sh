#!/bin/bash
# call Z: fused cluster slicing of the cols-path Ozaki operands (one HBM read of X): GEMM error
# bounds, FP64_OZ gates, non-finite propagation, c3 parity; c3 line fused vs two-pass; launch list
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 900 python -m pytest tests/test_gpu_oz.py tests/test_gpu_attn_oz.py -q -x --timeout 600 -p no:cacheprovider > $O/t_r02z.log 2>&1; echo "rc=$?" >> $O/t_r02z.log
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02z_c3.json 2> $O/b_r02z_c3.err
SLQ_OZ_SLICE_TWOPASS=1 SLQ_OZ_SLICE_L1=1 timeout 900 python bench.py --no-cpu-baseline > $O/b_r02z_c3_before.json 2> $O/b_r02z_c3_before.err
SLQ_OZ_SLICE_L1=1 timeout 900 python bench.py --no-cpu-baseline > $O/b_r02z_c3_l1.json 2> $O/b_r02z_c3_l1.err
timeout 900 python -m pytest tests/test_gpu_large.py -q -s -k "c3_lanczos or c5" --timeout 600 -p no:cacheprovider > $O/t_r02z_large.log 2>&1; echo "rc=$?" >> $O/t_r02z_large.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 2800 --csv --log-file $O/ncu_r02z_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > $O/ncu_r02z.log 2>&1; echo "rc=$?" >> $O/ncu_r02z.log
