python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline --reorth none > gpurun_out/c2_noreorth.json 2> gpurun_out/ro.err
python -c "import json; d=json.load(open('gpurun_out/c2_noreorth.json')); print('c2 none', round(d['value'],1), round(d['ms_per_step'],3))"
timeout 1200 python bench.py --config c3 --steps 100 --warmup 3 --no-cpu-baseline > gpurun_out/c3_full100.json 2> gpurun_out/ro3.err
python -c "import json; d=json.load(open('gpurun_out/c3_full100.json')); print('c3 full m=100', round(d['ms_per_step'],1), d['kernel_ms_per_step'].get('reorth'), d['roofline']['frac'], d['clocks'])"
