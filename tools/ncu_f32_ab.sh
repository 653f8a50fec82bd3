#!/bin/bash
# ncu --set full of one binary32 key-only merge pass, for each library in $@ (run under gpurun).
set -u
mkdir -p gpurun_out
for lib in "$@"; do
  GNS_LIB=$lib python tools/f32_once.py > gpurun_out/plain_f32_$lib.log 2>&1 || { echo "plain failed $lib"; continue; }
  GNS_LIB=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:"f32_merge" -s 11 -c 1 \
      -o gpurun_out/prof_f32_$lib python tools/f32_once.py > gpurun_out/ncu_f32_$lib.log 2>&1; echo "ncu_rc=$? $lib"
done
