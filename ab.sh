timeout 900 python -m pytest tests -m "gpu" -q -x -k "inplace or 0.5 or edge or cfg or baseline or nan" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for r in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "inplace" > gpurun_out/t$r.log 2>&1; tail -1 gpurun_out/t$r.log; done
python tools/time_sort.py --pairs --n 27; python tools/time_sort.py --pairs --n 27 --frac 0.5; python tools/time_sort.py --frac 0.5
