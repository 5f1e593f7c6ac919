python -c "import __graft_entry__ as g; g.build()" > /dev/null
SLQ_OZ_WIDE=2 timeout 900 python -m pytest tests/test_gpu_oz.py -x -q -m gpu -k "error_bound and 7" > gpurun_out/ozw_t.log 2>&1; tail -2 gpurun_out/ozw_t.log
for sh in "4096 4096 4096" "4096 14336 4096" "8192 3072 768" "8192 768 3072" "8192 2304 768" "8192 768 8192"; do
  python tools/oz_bn.py $sh 7; SLQ_OZ_WIDE=2 python tools/oz_bn.py $sh 7
done
for w in 0 1; do
SLQ_OZ_WIDE=$w timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3w$w.json 2> gpurun_out/c3w$w.err
python -c "import json; d=json.load(open('gpurun_out/c3w$w.json')); print('c3 wide=$w', d['ms_per_step'], d['kernel_ms_per_step']['gemm_i8'], d['roofline']['frac'])"
done
