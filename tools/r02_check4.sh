#!/bin/bash
# call D: c3 bench + launch list after the epilogue change, the whole GPU suite alone (durations:
# the driver gives it 1200 s), then the secondary bench lines
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02d_c3.json 2> $O/b_r02d_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 2700 --csv --log-file $O/ncu_r02d_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > $O/ncu_r02d_c3_launches.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfEx --durations=50 --timeout 900 -p no:cacheprovider > $O/t_r02d.log 2>&1
echo "pytest rc=$?" >> $O/t_r02d.log
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/b_r02d_c2.json 2> $O/b_r02d_c2.err
for v in "none" "window --window 8" "full --basis bf16"; do
  tag=$(echo $v | tr ' ' '_' | tr -d '-')
  timeout 900 python bench.py --reorth $v --no-cpu-baseline > $O/b_r02d_c3_$tag.json 2> $O/b_r02d_c3_$tag.err
done
