python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "error_codes or nonfinite" > gpurun_out/nf.log 2>&1; tail -15 gpurun_out/nf.log
