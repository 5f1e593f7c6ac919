#!/bin/bash
# call V: the whole GPU suite as the driver runs it, smoke, the headline bench (with the CPU oracle
# sample), the c2 line, a c3 launch list and --set full captures of two attention kernels
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu -rfEx --durations=30 -p no:cacheprovider > $O/t_r02v.log 2>&1
echo "pytest rc=$?" >> $O/t_r02v.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02v.log 2>&1; echo "smoke rc=$?" >> $O/smoke_r02v.log
timeout 900 python bench.py > $O/b_r02v_c3.json 2> $O/b_r02v_c3.err
timeout 600 python bench.py --config c2 --no-cpu-baseline > $O/b_r02v_c2.json 2> $O/b_r02v_c2.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 2800 --csv --log-file $O/ncu_r02v_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > $O/ncu_r02v_c3_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 40 -c 1 -o $O/ncu_r02v_oz_gemm python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > $O/ncu_r02v_oz_gemm.log 2>&1
