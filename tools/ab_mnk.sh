python -c "import __graft_entry__ as g; g.build()" > /dev/null
for i in 1 2; do for t in 1e9 5e8 3e8; do
SLQ_OZ_MIN_MNK=$t timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/abm.json 2> gpurun_out/abm.err
python -c "import json; d=json.load(open('gpurun_out/abm.json')); print('mnk=$t', round(d['value'],1), round(d['ms_per_step'],3))"
done; done
