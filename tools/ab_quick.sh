#!/bin/bash
# Quick same-box A/B of library builds on whole sorts (timings only): ab_quick.sh LIB...
set -u
mkdir -p gpurun_out
for rep in 1 2 3; do for lib in "$@"; do
  echo "== $lib"
  GNS_LIB=$lib python tools/time_sort.py --reps 30 2>&1 | tail -1
  GNS_LIB=$lib python tools/time_sort.py --pairs --reps 30 2>&1 | tail -1
  GNS_LIB=$lib python tools/time_sort.py --frac 0.5 --reps 30 2>&1 | tail -1
  GNS_LIB=$lib python tools/time_f32.py 2>&1 | cut -c1-120
done; done > gpurun_out/ab_quick.log 2>&1
cat gpurun_out/ab_quick.log
