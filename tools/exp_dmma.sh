python -c "import __graft_entry__ as g; g.build()"
VARIANTS=1,9 timeout 300 python tools/gemm_sweep.py > gpurun_out/sweep2.jsonl 2>&1
run() { echo "== $1 $2"; env $1 timeout 300 python bench.py --no-cpu-baseline --steps 64 $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'hvp', round(1000/d['hvp_per_s_standalone'],3), 'grad', round(d['grad_step_ms'],3), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items() if v > 0.1}, d['roofline']['frac'])"; }
run X=1
run X=1 "--numerics fp64_oz"
run SLQ_DMMA_VARIANT=9
