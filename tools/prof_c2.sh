# c2 launch list (per-launch durations, cold cache, serialised) of the current tree
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --steps 32 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_now.json 2> gpurun_out/bench_c2_now.err
tail -c 300 gpurun_out/bench_c2_now.json
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none -s 600 -c 400 --csv --log-file gpurun_out/launches_c2_now.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c2_now.log 2>&1
echo done
