python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() { env $1 timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/abs.json 2> gpurun_out/abs.err
python -c "import json; d=json.load(open('gpurun_out/abs.json')); print('$1', round(d['ms_per_step'],1), round(d['grad_step_ms'],1), round(d['hvp_over_grad'],3))"; }
run X=0; run SLQ_SERIAL_PASSES=1; run "SLQ_SERIAL_PASSES=1 SLQ_OZ_WIDE=1"; run X=0
