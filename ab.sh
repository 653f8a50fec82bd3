timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(d['value']/1e9, d['roofline']['frac']); print(d['presorted_cfg4']); print({k:(v['ms'],v['ram_pct'],v['tfootprint_ms']) for k,v in d['footprint_cfg5'].items() if isinstance(v,dict)}, d['footprint_cfg5']['argmin_tfootprint_fraction'])"
