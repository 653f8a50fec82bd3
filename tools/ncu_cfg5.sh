#!/bin/bash
# ncu launch lists of BASELINE config 5 (2^27 f64 + u32, buffer 1.0 and 0.5),
# one sort each (SURVEY §8(d) ncu evidence); run under gpurun.
mkdir -p gpurun_out
for f in 1.0 0.5; do
  python tools/one_sort.py --pairs --frac $f > gpurun_out/one_$f.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_cfg5_$f.csv python tools/one_sort.py --pairs --frac $f > gpurun_out/ncu_cfg5_$f.log 2>&1
  echo "cfg5 $f rc=$?"
done
