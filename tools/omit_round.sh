#!/bin/bash
# Omitsort schedule: parity tests, then timings against the default schedule.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_omit.py -x -q > gpurun_out/omit_pytest.log 2>&1; echo "omit_pytest_rc=$?"; tail -3 gpurun_out/omit_pytest.log
GNS_LIB=libgns_debug.so timeout 900 python -m pytest tests/test_gpu_omit.py -x -q > gpurun_out/omit_pytest_dbg.log 2>&1; echo "omit_pytest_dbg_rc=$?"; tail -3 gpurun_out/omit_pytest_dbg.log
for inp in uniform asc desc swap1pct runs16; do
  for o in "" "--omit"; do python tools/time_sort.py --input $inp $o; done
done > gpurun_out/omit_time.txt 2>&1
cat gpurun_out/omit_time.txt
python tools/time_launches.py --n 24 --frac 1.0 --omit > gpurun_out/omit_launch.txt 2>&1
python tools/time_launches.py --n 24 --frac 1.0 --omit --input runs16 >> gpurun_out/omit_launch.txt 2>&1
