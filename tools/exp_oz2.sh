python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_oz.py -m gpu -q -x > gpurun_out/oz_all2.log 2>&1; tail -1 gpurun_out/oz_all2.log
run() { echo "== $1 $2"; env $1 timeout 300 python bench.py --no-cpu-baseline --steps 64 $2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'hvp', round(1000/d['hvp_per_s_standalone'],3), 'grad', round(d['grad_step_ms'],3), {k: round(v,2) for k,v in d['kernel_ms_per_step'].items() if v > 0.1}, d['roofline']['kernel'], round(d['roofline']['frac'],3))"; }
run X=1
run SLQ_OZ_MIN_MNK=0
run SLQ_OZ_MIN_MNK=3e8
run "SLQ_OZ_MIN_MNK=0 SLQ_OZ_SLICES=6"
