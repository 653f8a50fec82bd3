GNS_LIB=libgns_debug.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_debug.log 2>&1; echo debug_rc=$?; tail -2 gpurun_out/t_debug.log
GNS_LIB=libgns_debug.so python tools/sanitize_cases.py 2>&1 | tail -2
for p in 0 1; do GNS_PDL=$p python tools/time_sort.py --tag pdl$p; GNS_PDL=$p python tools/time_sort.py --tag pdl$p --pairs --n 27 --frac 0.5; done
