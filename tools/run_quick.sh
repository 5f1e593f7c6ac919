# quick GPU check: fp64 GEMM plans, core parity, c2 bench
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm_f64.py tests/test_gpu_parity.py tests/test_gpu_fsdp1.py -x -q -m gpu > gpurun_out/quick.log 2>&1; tail -3 gpurun_out/quick.log
timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms_per_step'])"
