#!/bin/bash
# call N: three-sweep cross-entropy; ncu --set full of the attention emit kernels and the CE
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02n_c3.json 2> $O/b_r02n_c3.err
for k in k_att_sm_bwd k_att_sm_fwd k_cross_entropy k_att_rows; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $O/ncu_r02n_$k python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > $O/ncu_r02n_$k.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py -q -s -k "c3_lanczos or c5 or nonfinite or gpt" --timeout 600 -p no:cacheprovider > $O/t_r02n.log 2>&1; echo "rc=$?" >> $O/t_r02n.log
