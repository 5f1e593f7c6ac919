#!/bin/bash
# call G: the whole GPU suite (all stored oracle runs present), smoke, the c3 headline bench with
# its CPU baseline, the reference arm, the c3 launch list and --set full captures of the forward
# Ozaki GEMMs (qkv: launch 0, fc: launch 2)
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 1800 python -m pytest tests -m gpu -q -rfEx --durations=40 --timeout 900 -p no:cacheprovider > $O/t_r02g.log 2>&1
echo "pytest rc=$?" >> $O/t_r02g.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02g.log 2>&1; echo "rc=$?" >> $O/smoke_r02g.log
timeout 900 python bench.py > $O/b_r02g_c3.json 2> $O/b_r02g_c3.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/b_r02g_ref.json 2> $O/b_r02g_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 2700 --csv --log-file $O/ncu_r02g_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > $O/ncu_r02g_c3_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 0 -c 1 -o $O/ncu_r02g_oz_qkv --force-overwrite python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > $O/ncu_r02g_oz_qkv.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_oz_gemm -s 2 -c 1 -o $O/ncu_r02g_oz_fc --force-overwrite python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > $O/ncu_r02g_oz_fc.log 2>&1
