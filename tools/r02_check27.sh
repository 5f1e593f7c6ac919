#!/bin/bash
# call AA: attention column slicing in one read (k_att_cols1), cluster slicing at 8 rows per CTA: attention / Ozaki tests, c3 line, launch list
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 900 python -m pytest tests/test_gpu_attn_oz.py tests/test_gpu_oz.py -q -x --timeout 600 -p no:cacheprovider > $O/t_r02aa.log 2>&1; echo "rc=$?" >> $O/t_r02aa.log
timeout 900 python bench.py > $O/b_r02aa_c3.json 2> $O/b_r02aa_c3.err
SLQ_OZ_SLICE_TWOPASS=1 timeout 900 python bench.py --no-cpu-baseline > $O/b_r02aa_c3_twopass.json 2> $O/b_r02aa_c3_twopass.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 2800 --csv --log-file $O/ncu_r02aa_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > $O/ncu_r02aa.log 2>&1; echo "rc=$?" >> $O/ncu_r02aa.log
timeout 900 python -m pytest tests/test_gpu_large.py -q -s -k "c3_lanczos or c5" --timeout 600 -p no:cacheprovider > $O/t_r02aa_large.log 2>&1; echo "rc=$?" >> $O/t_r02aa_large.log
