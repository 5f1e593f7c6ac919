# A/B: split-K reduce in the GEMM's last CTA (default) vs the separate reduce kernel
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_gemm_f64.py tests/test_gpu_parity.py tests/test_gpu_fsdp1.py -x -q -m gpu > gpurun_out/quick.log 2>&1; tail -3 gpurun_out/quick.log
for i in 1 2; do
for e in 0 1; do
SLQ_DMMA_SPLIT_EXT=$e timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$e.json 2> gpurun_out/ab_$e.err
python -c "import json; d=json.load(open('gpurun_out/ab_$e.json')); print('ext=$e', d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_ms_per_step']['gemm'], d['gpu_launches'])"
done; done
