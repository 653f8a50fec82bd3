timeout 900 python -m pytest tests -m "gpu" -q -x -k "limited or inplace or edge" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for f in 1.0 0.5 0.25 0.125 0.0625; do python tools/time_sort.py --pairs --n 27 --frac $f; done
