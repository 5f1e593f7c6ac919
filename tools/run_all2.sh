python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_all4.log 2>&1; tail -3 gpurun_out/gpu_all4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1; echo smoke rc=$?
