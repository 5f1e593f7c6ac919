python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_oz.py -x -q -m gpu > gpurun_out/ozd.log 2>&1; tail -1 gpurun_out/ozd.log
SLQ_OZ_ISSUERS=1 timeout 600 python -m pytest tests/test_gpu_oz.py -x -q -m gpu -k error_bound > gpurun_out/ozd1.log 2>&1; tail -1 gpurun_out/ozd1.log
for sh in "2048 4096 256" "8192 3072 768" "8192 768 3072" "4096 4096 4096" "8192 50257 768"; do python tools/oz_bn.py $sh 7; done
SLQ_OZ_DEBUG=13 python tools/oz_bn.py 2048 4096 256 7
for i in 1 2; do
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3d.json 2> gpurun_out/c3d.err
python -c "import json; d=json.load(open('gpurun_out/c3d.json')); print('c3', round(d['ms_per_step'],1), round(d['kernel_ms_per_step']['gemm_i8'],1), round(d['roofline']['frac'],3))"
done
timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/c2d.json 2> gpurun_out/c2d.err
python -c "import json; d=json.load(open('gpurun_out/c2d.json')); print('c2', round(d['value'],1), round(d['ms_per_step'],3), round(d['kernel_ms_per_step']['gemm_i8'],3))"
