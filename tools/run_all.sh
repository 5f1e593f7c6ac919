# full GPU suite + smoke + headline bench (c2) + launch list
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_all3.log 2>&1; tail -3 gpurun_out/gpu_all3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke3.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench_final3.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'])"
