python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:"k_layernorm_bwd" --clock-control none -c 4 --csv --log-file gpurun_out/ln_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ln_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_layernorm_bwd" -s 2 -c 1 -o gpurun_out/ln_bwd -f python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ln_ncu2.log 2>&1
echo done
