python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm_f64.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/lb.log 2>&1; tail -1 gpurun_out/lb.log
for i in 1 2 3; do
timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/lb.json 2> gpurun_out/lb.err
python -c "import json; d=json.load(open('gpurun_out/lb.json')); print(round(d['value'],1), round(d['ms_per_step'],3), round(d['kernel_ms_per_step']['gemm'],3), round(d['roofline']['frac'],3))"
done
