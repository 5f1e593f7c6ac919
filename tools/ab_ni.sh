python -c "import __graft_entry__ as g; g.build()" > /dev/null
SLQ_OZ_ISSUERS=2 timeout 900 python -m pytest tests/test_gpu_oz.py -x -q -m gpu -k "error_bound" > gpurun_out/ozbk_t.log 2>&1; tail -2 gpurun_out/ozbk_t.log
for sh in "4096 4096 4096" "4096 14336 4096" "8192 3072 768" "8192 768 3072" "8192 2304 768" "768 768 8192" "2048 4096 256"; do
  python tools/oz_bn.py $sh 7; SLQ_OZ_ISSUERS=2 python tools/oz_bn.py $sh 7
done
for w in 1 2 1 2; do
SLQ_OZ_ISSUERS=$w timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3bk.json 2> gpurun_out/c3bk.err
python -c "import json; d=json.load(open('gpurun_out/c3bk.json')); print('c3 ni=$w', round(d['ms_per_step'],1), round(d['kernel_ms_per_step']['gemm_i8'],1), round(d['roofline']['frac'],3))"
done
