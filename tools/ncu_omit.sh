#!/bin/bash
# ncu of the Omitsort helper kernels (plan, copy) on 2^24 uniform keys
mkdir -p gpurun_out
python tools/time_sort.py --omit --reps 2 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"omit_plan|omit_copy" -c 3 -o gpurun_out/omit_full python tools/time_sort.py --omit --reps 1 > gpurun_out/ncu_omit.log 2>&1
echo rc=$?
