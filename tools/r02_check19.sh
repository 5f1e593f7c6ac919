#!/bin/bash
# call S: where the K = 64 attention GEMMs spend their time (SLQ_OZ_DEBUG switches), per-launch list
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 300 python tools/attn_debug.py > $O/attn_debug.log 2>&1
for d in 0 4 8 12; do
  SLQ_OZ_DEBUG=$d timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -c 40 --csv --log-file $O/ncu_attn_debug_$d.csv python tools/attn_debug.py run > /dev/null 2>&1
done
