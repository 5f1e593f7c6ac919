# watchdog tests + FSDP one-rank path + parity after the sync changes
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_watchdog.py tests/test_gpu_fsdp1.py tests/test_gpu_oz.py tests/test_gpu_gemm_f64.py -x -q -m gpu > gpurun_out/wd.log 2>&1; tail -15 gpurun_out/wd.log
