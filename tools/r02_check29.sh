#!/bin/bash
# call AC: opt-in 16-row / 16-CTA cluster slicing (SLQ_OZ_SLICE_CS16=1): Ozaki / attention tests under it, c3 A/B, launch list
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
SLQ_OZ_SLICE_CS16=1 timeout 900 python -m pytest tests/test_gpu_oz.py tests/test_gpu_attn_oz.py -q -x --timeout 600 -p no:cacheprovider > $O/t_r02ac.log 2>&1; echo "rc=$?" >> $O/t_r02ac.log
SLQ_OZ_SLICE_CS16=1 timeout 900 python bench.py --no-cpu-baseline > $O/b_r02ac_c3_cs16.json 2> $O/b_r02ac_c3_cs16.err
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02ac_c3.json 2> $O/b_r02ac_c3.err
SLQ_OZ_SLICE_CS16=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:slice -c 400 --csv --log-file $O/ncu_r02ac_cs16.csv python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > $O/ncu_r02ac.log 2>&1; echo "rc=$?" >> $O/ncu_r02ac.log
SLQ_OZ_SLICE_CS16=1 timeout 900 python -m pytest tests/test_gpu_large.py -q -s -k "c3_lanczos" --timeout 600 -p no:cacheprovider > $O/t_r02ac_large.log 2>&1; echo "rc=$?" >> $O/t_r02ac_large.log
