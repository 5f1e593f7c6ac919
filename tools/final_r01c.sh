python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_final3.log 2>&1; tail -1 gpurun_out/gpu_final3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final3.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_final3.log
timeout 900 python bench.py > gpurun_out/fb3_c2.json 2> gpurun_out/fb3_c2.err; echo c2 rc=$?
python -c "import json; d=json.load(open('gpurun_out/fb3_c2.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
echo done
