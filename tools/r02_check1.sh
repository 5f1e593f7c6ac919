#!/bin/bash
# round-2 first GPU check: host facts, the changed GPU tests, c2 / c3 bench lines
cd "$(dirname "$0")/.."
( nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)|Socket|Thread"; nvidia-smi --query-gpu=name,memory.total,memory.free --format=csv ) > gpurun_out/host_r02.txt 2>&1
export SLQ_TIMEOUT_S=600
timeout 2400 python -m pytest tests/test_gpu_oz.py tests/test_gpu_ckpt.py tests/test_gpu_fsdp2_loopback.py tests/test_gpu_fsdp1.py -q -s --timeout 900 > gpurun_out/t_r02a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t_r02a.log
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_r02a_c2.json 2> gpurun_out/b_r02a_c2.err
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_r02a_c3.json 2> gpurun_out/b_r02a_c3.err
SLQ_SERIAL_PASSES=1 timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_r02a_c3_serial.json 2>&1
