#!/bin/bash
# Oracle-only golden runs on the GPU box's host (16 cores, 196 GB): the c4 parity batch (reorth none
# at m = 16, full at m = 8: its fp64 basis is 8.8 GB per row), the c5 twin (no basis, m = 16) and
# the c3 parity batch at eps 1e-2 / 1e-4 (m = 32, full).  Each job has an address-space limit so a
# memory overrun is a MemoryError, not the host OOM killer.  GPU work runs alongside (below).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/golden
G=tests/golden/make_golden.py
(
  OPENBLAS_NUM_THREADS=8 python $G --case c5_twin --m 16 --eps 1e-3 --reorth none --mem-limit-gb 120 > gpurun_out/golden/c5.log 2>&1 &
  OPENBLAS_NUM_THREADS=8 python $G --case c3_parity --m 32 --eps 1e-2 --reorth full --mem-limit-gb 60 > gpurun_out/golden/c3a.log 2>&1
  wait
  OPENBLAS_NUM_THREADS=8 python $G --case c4_parity --m 16 --eps 1e-3 --reorth none --mem-limit-gb 100 > gpurun_out/golden/c4n.log 2>&1 &
  OPENBLAS_NUM_THREADS=8 python $G --case c3_parity --m 32 --eps 1e-4 --reorth full --mem-limit-gb 60 > gpurun_out/golden/c3b.log 2>&1
  wait
  OPENBLAS_NUM_THREADS=16 python $G --case c4_parity --m 8 --eps 1e-3 --reorth full --mem-limit-gb 165 > gpurun_out/golden/c4f.log 2>&1
  cp tests/golden/lanczos_*.json gpurun_out/golden/ 2>/dev/null
  echo done > gpurun_out/golden/DONE
) &
GOLD_PID=$!
# GPU work meanwhile: the GPU suite with durations (large-config golden tests fail until the files exist)
export SLQ_TIMEOUT_S=600
timeout 3000 python -m pytest tests -m gpu -q --durations=60 --timeout 900 -p no:cacheprovider -k "not c4_parity and not c5_twin and not test_gpu_large" > gpurun_out/t_r02b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t_r02b.log
timeout 900 python bench.py > gpurun_out/b_r02b_c3.json 2> gpurun_out/b_r02b_c3.err
wait $GOLD_PID
