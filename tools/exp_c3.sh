python -c "import __graft_entry__ as g; g.build()"
run() { echo "== $1 $2"; env $1 timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 6 --warmup 3 $2 > gpurun_out/c3_$3.json 2>gpurun_out/c3_$3.err; tail -1 gpurun_out/c3_$3.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],1), 'hvp', round(1000/d['hvp_per_s_standalone'],1), 'grad', round(d['grad_step_ms'],1), {k: round(v,1) for k,v in d['kernel_ms_per_step'].items() if v > 1}, d['roofline']['kernel'], round(d['roofline']['frac'],3), round(d['roofline']['achieved'],1))"; tail -2 gpurun_out/c3_$3.err; }
run X=1 "--numerics fp64_oz" oz
run X=1 "--numerics bf16x3" bf16x3
run X=1 "--numerics fp64" fp64
