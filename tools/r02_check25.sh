#!/bin/bash
# call Y (re-entry): whole GPU suite, smoke, c3 headline line with the CPU-oracle sample, launch list
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
( nproc; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv ) > $O/host_r02y.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > $O/t_r02y_all.log 2>&1; echo "rc=$?" >> $O/t_r02y_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02y.log 2>&1; echo "rc=$?" >> $O/smoke_r02y.log
timeout 900 python bench.py > $O/b_r02y_c3.json 2> $O/b_r02y_c3.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/b_r02y_c2.json 2> $O/b_r02y_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 2800 --csv --log-file $O/ncu_r02y_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > $O/ncu_r02y.log 2>&1; echo "rc=$?" >> $O/ncu_r02y.log
