python -m pytest tests/test_gpu_parity.py -q -x -k "edge_sizes or tile_sort or uniform or specials or merge_pass" > gpurun_out/t.log 2>&1; tail -1 gpurun_out/t.log
for v in 0 1; do GNS_TILE_VARIANT=$v python bench.py --steps 10 --warmup 3 --no-footprint --no-cpu-baseline > gpurun_out/b$v.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b$v.log').read().strip().splitlines()[-1]); r=d['roofline']; print('v$v', d['value']/1e9, r['per_kernel_ms']['tile_sort'], r['per_kernel_ms']['merge_passes'])"; done
for v in 0 1; do GNS_TILE_VARIANT=$v python tools/time_sort.py --tag v$v --pairs; done
