python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_oz.py -x -q -m gpu > gpurun_out/oz_t2.log 2>&1; tail -2 gpurun_out/oz_t2.log
timeout 900 python bench.py --config c3 --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/c3_oz2.json 2> gpurun_out/c3_oz2.err
python -c "import json; d=json.load(open('gpurun_out/c3_oz2.json')); print('c3', d['ms_per_step'], d['kernel_ms_per_step']['oz_slice'], d['roofline']['frac'], d['tokens_x_hvp_per_s'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size -k regex:"k_oz_slice|k_oz_colexp" --clock-control none -c 80 --csv --log-file gpurun_out/slice_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/slice_ncu.log 2>&1
echo done
