#!/bin/bash
# Full ncu capture of the tile sort and one merge pass (run under gpurun).
# usage: bash tools/ncu_full.sh TAG [extra time_sort args]
set -u
tag=$1; shift
mkdir -p gpurun_out
python tools/time_sort.py --reps 3 "$@" > gpurun_out/plain_$tag.log 2>&1 || { echo "plain run failed"; cat gpurun_out/plain_$tag.log; exit 1; }
cat gpurun_out/plain_$tag.log
timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"merge_tstore|tile_sort" -s 6 -c 2 \
    -o gpurun_out/full_$tag python tools/time_sort.py --reps 1 "$@" > gpurun_out/ncu_$tag.log 2>&1
echo "ncu_rc=$?"
