python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py --steps 64 --warmup 3 > gpurun_out/bench_c2_final.json 2> gpurun_out/bench_c2_final.err
tail -c 400 gpurun_out/bench_c2_final.json
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 600 -c 700 --csv --log-file gpurun_out/launches_c2_final.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c2.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_oz_gemm -s 20 -c 1 -o gpurun_out/oz_c3 -f python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_oz_gemm -s 2 -c 1 -o gpurun_out/oz_c2head -f python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_c2oz.log 2>&1
echo done
