#!/bin/bash
# Full ncu capture of one launch of a kernel (run under gpurun).
# usage: bash tools/ncu_kernel.sh TAG REGEX SKIP [time_sort args]
set -u
tag=$1; rx=$2; skip=$3; shift 3
mkdir -p gpurun_out
python tools/time_sort.py --reps 3 "$@" > gpurun_out/plain_$tag.log 2>&1 || { echo "plain run failed"; cat gpurun_out/plain_$tag.log; exit 1; }
cat gpurun_out/plain_$tag.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s $skip -c 1 \
    -o gpurun_out/full_$tag python tools/time_sort.py --reps 1 "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "ncu_rc=$?"
