python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_final2.log 2>&1; tail -2 gpurun_out/gpu_final2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke_final2.log
timeout 900 python bench.py > gpurun_out/fb2_c2.json 2> gpurun_out/fb2_c2.err; echo c2 rc=$?
timeout 1500 python bench.py --config c3 --steps 100 --warmup 3 > gpurun_out/fb2_c3.json 2> gpurun_out/fb2_c3.err; echo c3 rc=$?
echo done
