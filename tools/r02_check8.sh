#!/bin/bash
# call H: the whole GPU suite exactly as the driver runs it (timing), then the headline bench
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -rfEx --durations=30 -p no:cacheprovider > $O/t_r02h.log 2>&1
echo "pytest rc=$?" >> $O/t_r02h.log
timeout 900 python bench.py > $O/b_r02h_c3.json 2> $O/b_r02h_c3.err
