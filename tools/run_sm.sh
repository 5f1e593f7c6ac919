python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fsdp1.py -x -q -m gpu > gpurun_out/sm.log 2>&1; tail -1 gpurun_out/sm.log
timeout 900 ncu --metrics gpu__time_duration.sum -k regex:"k_softmax_causal" --clock-control none -c 3 --csv --log-file gpurun_out/sm_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/sm_ncu.log 2>&1
grep -v "^==" gpurun_out/sm_c3.csv | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
print([row[h.index('Metric Value')] for row in r[1:]])"
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3sm.json 2> gpurun_out/c3sm.err
python -c "import json; d=json.load(open('gpurun_out/c3sm.json')); print('c3', round(d['ms_per_step'],1), round(d['kernel_ms_per_step']['attention'],2))"
timeout 600 python bench.py --steps 64 --warmup 3 --no-cpu-baseline > gpurun_out/c2sm.json 2> gpurun_out/c2sm.err
python -c "import json; d=json.load(open('gpurun_out/c2sm.json')); print('c2', round(d['value'],1), round(d['ms_per_step'],3), round(d['kernel_ms_per_step']['attention'],3))"
