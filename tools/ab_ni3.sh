python -c "import __graft_entry__ as g; g.build()" > /dev/null
for n in 2 3; do SLQ_OZ_ISSUERS=$n timeout 900 python -m pytest tests/test_gpu_oz.py -x -q -m gpu > gpurun_out/ozni$n.log 2>&1; tail -1 gpurun_out/ozni$n.log; done
for sh in "4096 4096 4096" "4096 14336 4096" "8192 3072 768" "8192 768 3072" "768 768 8192" "2048 4096 256"; do
  for n in 1 2 3; do SLQ_OZ_ISSUERS=$n python tools/oz_bn.py $sh 7 | sed "s/^/ni=$n /"; done
done
for w in 2 3 2 3; do
SLQ_OZ_ISSUERS=$w timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3ni.json 2> gpurun_out/c3ni.err
python -c "import json; d=json.load(open('gpurun_out/c3ni.json')); print('c3 ni=$w', round(d['ms_per_step'],1), round(d['kernel_ms_per_step']['gemm_i8'],1), round(d['roofline']['frac'],3))"
done
for w in 2 3; do
SLQ_OZ_ISSUERS=$w timeout 900 python bench.py --steps 32 --warmup 3 --no-cpu-baseline > gpurun_out/c2ni.json 2> gpurun_out/c2ni.err
python -c "import json; d=json.load(open('gpurun_out/c2ni.json')); print('c2 ni=$w', round(d['value'],1), round(d['ms_per_step'],3), round(d['kernel_ms_per_step']['gemm_i8'],3))"
done
