timeout 600 python -m pytest tests -m "gpu and not slow" -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-footprint --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench_rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); r=d['roofline']; print('Gkeys/s', d['value']/1e9, 'ms', d['ms_per_step'], 'merge frac', r['frac'], 'GB/s', r['achieved']); print(r['per_kernel_ms'])"
