python -c "import __graft_entry__ as g; g.build()" > /dev/null
SLQ_DEFER_WGRAD=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fsdp1.py -x -q -m gpu > gpurun_out/dfr1.log 2>&1; tail -2 gpurun_out/dfr1.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/dfr0.log 2>&1; tail -1 gpurun_out/dfr0.log
for i in 1 2; do for e in 0 1; do
SLQ_DEFER_WGRAD=$e timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/abd.json 2> gpurun_out/abd.err
python -c "import json; d=json.load(open('gpurun_out/abd.json')); print('defer=$e', round(d['value'],1), round(d['ms_per_step'],3), round(d['kernel_ms_per_step']['gemm'],3), round(d['roofline']['frac'],3))"
done; done
