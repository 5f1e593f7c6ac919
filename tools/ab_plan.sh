# c2 step time under DMMA plan knobs (split division, forced variants), alternated
python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() { env $1 timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/abp.json 2> gpurun_out/abp.err
python -c "import json; d=json.load(open('gpurun_out/abp.json')); print('$1', round(d['value'],2), round(d['ms_per_step'],3), round(d['roofline']['frac'],3))"; }
for i in 1 2; do
run X=0; run SLQ_DMMA_SPLIT_DIV=2; run SLQ_DMMA_SPLIT_DIV=8; run SLQ_DMMA_VARIANT=1; run SLQ_DMMA_VARIANT=0; run SLQ_OZ_MIN_MNK=5e8
done
