# round-1 closing run: full GPU suite, smoke, headline bench (c2), c3 over a whole m = 100 run,
# c5-shape GEMM line, c2 launch list with DRAM bytes, Ozaki launches at c3, one Ozaki --set full
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_final.log 2>&1; tail -2 gpurun_out/gpu_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py > gpurun_out/fb_c2.json 2> gpurun_out/fb_c2.err; echo c2 rc=$?
timeout 1500 python bench.py --config c3 --steps 100 --warmup 3 > gpurun_out/fb_c3.json 2> gpurun_out/fb_c3.err; echo c3 rc=$?
timeout 900 python bench.py --config c5_gemm --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/fb_c5g.json 2> gpurun_out/fb_c5g.err; echo c5g rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 600 -c 500 --csv --log-file gpurun_out/fb_launches_c2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/fb_ncu_c2.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_oz_gemm -c 40 --csv --log-file gpurun_out/fb_oz_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fb_ncu_c3.log 2>&1; echo ncu2 rc=$?
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_oz_gemm -s 8 -c 1 -o gpurun_out/fb_oz_c5g -f python bench.py --config c5_gemm --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fb_ncu_c5g.log 2>&1; echo ncu3 rc=$?
echo done
