python -c "import __graft_entry__ as g; g.build()" > /dev/null
for e in 0 1; do
SLQ_LN_GENERIC=$e timeout 900 ncu --metrics gpu__time_duration.sum -k regex:"k_layernorm_bwd" --clock-control none -c 4 --csv --log-file gpurun_out/ln_$e.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ln_ncu_$e.log 2>&1
grep -v "^==" gpurun_out/ln_$e.csv | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
print('generic=$e', [row[h.index('Metric Value')] for row in r[1:]])"
done
for e in 0 1 0 1; do
SLQ_LN_GENERIC=$e timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3ln.json 2> gpurun_out/c3ln.err
python -c "import json; d=json.load(open('gpurun_out/c3ln.json')); print('c3 generic=$e', round(d['ms_per_step'],1), round(d['kernel_ms_per_step']['norm'],2))"
done
