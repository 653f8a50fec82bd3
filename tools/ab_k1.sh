#!/bin/bash
# Same-box A/B of K1 builds (key-only tile sort + whole sort, each twice, interleaved): ab_k1.sh LIB...
set -u
mkdir -p gpurun_out
for rep in 1 2; do for lib in "$@"; do
  echo "== $lib"
  GNS_LIB=$lib python tools/time_k1.py 2>&1 | grep "pairs=0"
  GNS_LIB=$lib python tools/time_f32.py 2>&1 | grep "pairs False"
done; done > gpurun_out/ab_k1.log 2>&1
cat gpurun_out/ab_k1.log
