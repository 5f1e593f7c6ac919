python -c "import __graft_entry__ as g; g.build()"
run() { echo "== $1 $2"; env $1 timeout 300 python bench.py --no-cpu-baseline --steps 64 $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'hvp', round(1000/d['hvp_per_s_standalone'],3), 'grad', round(d['grad_step_ms'],3), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items() if v > 0.1}, round(d['roofline']['frac'],3))"; }
run X=1
run SLQ_DMMA_SPLIT_MIN_K=512
run SLQ_DMMA_SPLIT_MIN_K=1024
run SLQ_DMMA_SPLIT_MIN_K=100000
run SLQ_DMMA_SPLIT_WAVES=1
run SLQ_DMMA_SPLIT_WAVES=3
