#!/bin/bash
# call AB (round-2 closing): whole GPU suite, smoke, c3 / c2 lines, one --set full capture of the cluster slicing kernel
cd "$(dirname "$0")/.."
O=gpurun_out
export SLQ_TIMEOUT_S=600
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > $O/t_r02ab_all.log 2>&1; echo "rc=$?" >> $O/t_r02ab_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02ab.log 2>&1; echo "rc=$?" >> $O/smoke_r02ab.log
timeout 900 python bench.py > $O/b_r02ab_c3.json 2> $O/b_r02ab_c3.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/b_r02ab_c2.json 2> $O/b_r02ab_c2.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_oz_slicecl -s 20 -c 1 -o $O/ncu_r02ab_slicecl python bench.py --steps 1 --warmup 1 --probe-m 2 --no-cpu-baseline > $O/ncu_r02ab_slicecl.log 2>&1; echo "rc=$?" >> $O/ncu_r02ab_slicecl.log
