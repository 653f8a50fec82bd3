#!/bin/bash
# ncu of the 4-way pass kernels (experiment)
mkdir -p gpurun_out
GNS_FOURWAY=1 python tools/time_sort.py --reps 2 > /dev/null 2>&1
GNS_FOURWAY=1 timeout 600 ncu --set full --clock-control none -k regex:"merge4|split4" -s 2 -c 2 -o gpurun_out/full_fw python tools/time_sort.py --reps 1 > gpurun_out/ncu_fw.log 2>&1
echo rc=$?
