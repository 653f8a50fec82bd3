#!/bin/bash
# Same-box A/B of library builds: usage ab_libs.sh LIB... (each timed twice, interleaved); the
# last LIB also runs the GPU suite first (parity before timing).
set -u
mkdir -p gpurun_out
last="${@: -1}"
GNS_LIB=$last timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab_suite.log 2>&1; echo "suite($last)_rc=$?"; tail -1 gpurun_out/ab_suite.log
for rep in 1 2; do for lib in "$@"; do
  echo "== $lib"
  GNS_LIB=$lib python tools/time_k1.py 2>&1 | grep "pairs=0"
  GNS_LIB=$lib python tools/time_sort.py 2>&1 | tail -1
  GNS_LIB=$lib python tools/time_f32.py 2>&1 | grep "pairs False"
done; done > gpurun_out/ab_libs.log 2>&1
cat gpurun_out/ab_libs.log
