#!/bin/bash
# call E: the c5-twin golden (alone on the host: ~120 GB) in the background; GPU: softmax / act-pass
# changes checked (c3 parity, checkpointing bit-identity), c3 bench + launch list, DMMA attention sweep
cd "$(dirname "$0")/.."
O=gpurun_out
mkdir -p $O/golden
OPENBLAS_NUM_THREADS=14 timeout 3400 python tests/golden/make_golden.py --case c5_twin --m 16 --eps 1e-3 --reorth none --mem-limit-gb 185 --out-dir $O/golden > $O/golden/c5.log 2>&1 &
GP=$!
export SLQ_TIMEOUT_S=600
timeout 900 python -m pytest tests/test_gpu_large.py tests/test_gpu_ckpt.py -q -s -k "c3_lanczos or bit_identical" --timeout 600 -p no:cacheprovider > $O/t_r02e.log 2>&1; echo "rc=$?" >> $O/t_r02e.log
timeout 900 python bench.py --no-cpu-baseline > $O/b_r02e_c3.json 2> $O/b_r02e_c3.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 2700 --csv --log-file $O/ncu_r02e_c3_launches.csv python bench.py --steps 2 --warmup 1 --probe-m 3 --no-cpu-baseline > $O/ncu_r02e_c3_launches.log 2>&1
T=1024 HD=64 NB=96 timeout 900 python tools/gemm_sweep_attn.py > $O/sweep_attn_c3.jsonl 2>&1
wait $GP
