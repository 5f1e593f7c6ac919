python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests/test_gpu_large.py tests/test_gpu_parity.py tests/test_gpu_paired.py -x -q -m gpu > gpurun_out/onl.log 2>&1; tail -1 gpurun_out/onl.log
for i in 1 2; do
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3o2.json 2> gpurun_out/c3o2.err
python -c "import json; d=json.load(open('gpurun_out/c3o2.json')); k=d['kernel_ms_per_step']; print('c3', round(d['ms_per_step'],1), round(k['attention'],2), round(k['cross_entropy'],2))"
done
