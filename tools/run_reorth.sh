python -c "import __graft_entry__ as g; g.build()" > /dev/null
for a in "" "--reorth none" "--reorth window --window 8" "--basis bf16" "--reorth window --window 8 --basis bf16"; do
timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline $a > gpurun_out/ro.json 2> gpurun_out/ro.err
python -c "import json; d=json.load(open('gpurun_out/ro.json')); print('$a|', round(d['value'],1), round(d['ms_per_step'],3), round(d['kernel_ms_per_step']['reorth'],3), d['config']['workload'][-40:])"
done
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline --reorth none > gpurun_out/c3_noreorth.json 2> gpurun_out/ro3.err
python -c "import json; d=json.load(open('gpurun_out/c3_noreorth.json')); print('c3 none', round(d['ms_per_step'],1), d['kernel_ms_per_step']['reorth'])"
