python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum -k regex:"k_layernorm|k_colreduce|k_softmax|k_cross" --clock-control none -c 120 --csv --log-file gpurun_out/norm_c3.csv python bench.py --config c3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/norm_ncu.log 2>&1
echo done
