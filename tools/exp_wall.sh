python -c "import __graft_entry__ as g; g.build()"
run() { echo "== $1"; env $1 timeout 300 python bench.py --no-cpu-baseline --steps 64 $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'hvp', round(1000/d['hvp_per_s_standalone'],3), 'grad', round(d['grad_step_ms'],3))"; }
run X=1
run SLQ_DMMA_VARIANT=6
run SLQ_DMMA_VARIANT=7
run SLQ_DMMA_VARIANT=0
run SLQ_DMMA_VARIANT=9
run SLQ_SERIAL_PASSES=1
run SLQ_NO_GRAPHS=1
run SLQ_OZ_SLICES=7 "--numerics fp64_oz"
