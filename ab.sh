timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
python bench.py --steps 10 --warmup 3 --no-footprint --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); r=d['roofline']; print(d['value']/1e9, r['frac'], r['per_kernel_ms']['tile_sort'], r['per_kernel_ms']['merge_passes'])"
python tools/time_sort.py --pairs; python tools/time_sort.py --pairs --n 27; python tools/time_sort.py --pairs --n 27 --frac 0.5
