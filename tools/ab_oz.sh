# Ozaki issuer change: correctness (error-bound tests) and rates on the c3 / c5 shapes
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_oz.py -x -q -m gpu > gpurun_out/oz_t.log 2>&1; tail -2 gpurun_out/oz_t.log
for sh in "4096 4096 4096" "4096 14336 4096" "8192 768 768" "8192 3072 768" "8192 768 3072" "768 768 8192"; do
  python tools/oz_bn.py $sh 7
done
timeout 600 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3_oz.json 2> gpurun_out/c3_oz.err
python -c "import json; d=json.load(open('gpurun_out/c3_oz.json')); print('c3', d['value'], d['ms_per_step'], d['roofline'])"
