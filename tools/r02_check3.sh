#!/bin/bash
# call C: golden jobs (c5 twin + c3 eps 1e-2) on the host in the background, GPU work meanwhile:
# Ozaki GEMM checks after the epilogue refactor, the c3 headline bench, the paired mode on c3, the
# ncu launch list of a short c3 probe and one `ncu --set full` capture of the fc-forward Ozaki GEMM.
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
bash tools/r02_golden_box2.sh c5 c3a -- '
timeout 900 python -m pytest tests/test_gpu_oz.py -q -s --timeout 600 > '$O'/t_r02c_oz.log 2>&1; echo "rc=$?" >> '$O'/t_r02c_oz.log
timeout 1500 python -m pytest tests/test_gpu_large.py -q -s -k "c3" --timeout 900 > '$O'/t_r02c_large.log 2>&1; echo "rc=$?" >> '$O'/t_r02c_large.log
timeout 900 python bench.py --no-cpu-baseline > '$O'/b_r02c_c3.json 2> '$O'/b_r02c_c3.err
timeout 900 python bench.py --oz-slices 7 --steps 10 --warmup 3 --no-cpu-baseline > '$O'/b_r02c_c3_s7.json 2> '$O'/b_r02c_c3_s7.err
timeout 900 python bench.py --numerics paired --steps 10 --warmup 3 --no-cpu-baseline > '$O'/b_r02c_c3_paired.json 2> '$O'/b_r02c_c3_paired.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 4000 --csv --log-file '$O'/ncu_r02c_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > '$O'/ncu_r02c_c3_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 2 -c 1 -o '$O'/ncu_r02c_oz_fc --force-overwrite python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > '$O'/ncu_r02c_oz_fc.log 2>&1
'
