#!/bin/bash
# A/B timing of env-selected variants (run under gpurun):
#   bash tools/ab_env.sh "GNS_X=0" "GNS_X=1" ...
# Each variant: bench.py (key-only 2^24) per-kernel figures.
mkdir -p gpurun_out
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-footprint --no-cpu-baseline > gpurun_out/ab.log 2>gpurun_out/ab.err || { echo "$v FAILED"; tail -5 gpurun_out/ab.err; continue; }
  python - "$v" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); r = d['roofline']
mp = r['per_kernel_ms']['merge_passes']
print(f"{sys.argv[1]:30s} Gkeys/s {d['value']/1e9:6.2f}  ms {d['ms_per_step']:.4f}  tile {r['per_kernel_ms']['tile_sort']:.4f}  "
      f"merge avg {sum(mp)/len(mp)*1e3:.1f}us [{' '.join(f'{x*1e3:.0f}' for x in mp)}] frac {r['frac']:.3f} ok={d['valid']}")
PY
done
