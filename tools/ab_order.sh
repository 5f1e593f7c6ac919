python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_oz.py -x -q -m gpu > gpurun_out/ozo.log 2>&1; tail -1 gpurun_out/ozo.log
SLQ_OZ_ORDER=1 timeout 900 python -m pytest tests/test_gpu_oz.py -x -q -m gpu -k error_bound > gpurun_out/ozo1.log 2>&1; tail -1 gpurun_out/ozo1.log
for sh in "8192 50257 768" "4096 14336 4096" "4096 4096 4096" "8192 3072 768"; do
  for o in 0 1; do SLQ_OZ_ORDER=$o python tools/oz_bn.py $sh 7 | sed "s/^/order=$o /"; done
done
for o in 0 -1 0 -1; do
SLQ_OZ_ORDER=$o timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3o.json 2> gpurun_out/c3o.err
python -c "import json; d=json.load(open('gpurun_out/c3o.json')); print('c3 order=$o', round(d['ms_per_step'],1), round(d['kernel_ms_per_step']['gemm_i8'],1), round(d['roofline']['frac'],3), round(d['kernel_ms_per_step']['norm'],2))"
done
for o in 0 -1; do
SLQ_OZ_ORDER=$o timeout 900 python bench.py --config c5_gemm --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c5o.json 2> gpurun_out/c5o.err
python -c "import json; d=json.load(open('gpurun_out/c5o.json')); print('c5g order=$o', round(d['ms_per_step'],1), round(d['kernel_ms_per_step']['gemm_i8'],1), round(d['roofline']['frac'],3))"
done
