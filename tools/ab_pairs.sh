#!/bin/bash
# Same-box A/B of library builds on the payload paths and the small sort: ab_pairs.sh LIB...
# (timings only; run tools/gpu_round.sh for parity)
set -u
mkdir -p gpurun_out
for rep in 1 2; do for lib in "$@"; do
  echo "== $lib"
  GNS_LIB=$lib python tools/time_k1.py 2>&1 | grep "uniform"; GNS_LIB=$lib python tools/time_f32.py 2>&1 | grep "pairs True"
  GNS_LIB=$lib python tools/time_sort.py --n 16 --pairs --reps 50 2>&1 | tail -1
  GNS_LIB=$lib python tools/time_sort.py --n 16 --reps 50 2>&1 | tail -1
  GNS_LIB=$lib python tools/time_sort.py --n 27 --pairs --reps 8 2>&1 | tail -1
  GNS_LIB=$lib python tools/time_sort.py --n 27 --pairs --frac 0.5 --reps 8 2>&1 | tail -1
done; done > gpurun_out/ab_pairs.log 2>&1
cat gpurun_out/ab_pairs.log
