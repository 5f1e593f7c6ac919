#!/bin/bash
# call T: streaming stores in the Ozaki epilogue (SLQ_OZ_DEBUG bit 16) on the attention GEMMs
cd "$(dirname "$0")/.."
O=gpurun_out
for d in 0 16; do
  SLQ_OZ_DEBUG=$d timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file $O/ncu_attn_stcs_$d.csv python tools/attn_debug.py run > /dev/null 2>&1
done
