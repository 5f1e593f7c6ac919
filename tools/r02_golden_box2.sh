#!/bin/bash
# Oracle-only golden runs on the GPU box's host (16 cores, 196 GB RAM), written straight into
# gpurun_out/golden/ and checkpointed after every Lanczos step (a run the call's time limit cuts
# short still returns its first k steps).  Usage: tools/r02_golden_box2.sh <job> [<job> ...]
# jobs: c5 (c5 twin, no basis, m = 16), c4n (c4 parity, no basis, m = 16), c4f (c4 parity, full,
# m = 8), c3a / c3b (c3 parity, full, m = 32, eps 1e-2 / 1e-4).  Then anything after "--" runs on the GPU.
cd "$(dirname "$0")/.."
O=gpurun_out/golden
mkdir -p $O
G=tests/golden/make_golden.py
jobs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do jobs+=("$1"); shift; done
[ "$1" = "--" ] && shift
n=${#jobs[@]}
thr=$(( 16 / (n > 0 ? n : 1) ))
for j in "${jobs[@]}"; do
  case $j in
    c5)  args="--case c5_twin --m 16 --eps 1e-3 --reorth none --mem-limit-gb 120" ;;
    c4n) args="--case c4_parity --m 16 --eps 1e-3 --reorth none --mem-limit-gb 100" ;;
    c4f) args="--case c4_parity --m 8 --eps 1e-3 --reorth full --mem-limit-gb 165" ;;
    c3a) args="--case c3_parity --m 32 --eps 1e-2 --reorth full --mem-limit-gb 60" ;;
    c3b) args="--case c3_parity --m 32 --eps 1e-4 --reorth full --mem-limit-gb 60" ;;
  esac
  OPENBLAS_NUM_THREADS=$thr timeout 3300 python $G $args --out-dir $O > $O/$j.log 2>&1 &
done
if [ $# -gt 0 ]; then bash -c "$*"; fi
wait
