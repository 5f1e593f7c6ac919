python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_tensorcore.py -x -q -m gpu -s -k "native or bf16x3_grad" > gpurun_out/bf16t.log 2>&1; grep -E "native|passed|failed|Error" gpurun_out/bf16t.log | tail -12
for nm in bf16 bf16x3; do
timeout 900 python bench.py --config c3 --numerics $nm --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3_$nm.json 2> gpurun_out/c3_$nm.err
python -c "import json; d=json.load(open('gpurun_out/c3_$nm.json')); print('$nm', d['ms_per_step'], d['grad_step_ms'], d['hvp_over_grad'], d['roofline']['frac'], d['roofline']['achieved'])"
done
