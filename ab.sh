python bench.py --steps 10 --warmup 3 --no-footprint --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(d['value']/1e9, d['e2e'])"
