python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/attn.log 2>&1; tail -1 gpurun_out/attn.log
for i in 1 2; do
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3a.json 2> gpurun_out/c3a.err
python -c "import json; d=json.load(open('gpurun_out/c3a.json')); print('c3', round(d['ms_per_step'],1), round(d['kernel_ms_per_step']['gemm'],2))"
done
