#!/bin/bash
# A/B of the register network merges (binary32 merge pass, K1 merge-path rounds) and the
# cooperative warp-end co-rank search: parity first, then timings.  usage: ab_net.sh LIB...
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/net_all.log 2>&1; echo "all_rc=$?"; tail -1 gpurun_out/net_all.log
GNS_LIB=libgns_debug.so timeout 900 python -m pytest tests -m gpu -q -x -k "f32 or tile_sort or key_types or edge" > gpurun_out/net_debug.log 2>&1; echo "debug_rc=$?"; tail -1 gpurun_out/net_debug.log
for rep in 1 2; do for lib in "$@"; do
  echo "== $lib"
  GNS_LIB=$lib python tools/time_f32.py 2>&1 | tail -2
  GNS_LIB=$lib python tools/time_k1.py 2>&1 | tail -4
  GNS_LIB=$lib python tools/time_sort.py 2>&1 | tail -2
done; done > gpurun_out/net_ab.log 2>&1
cat gpurun_out/net_ab.log
