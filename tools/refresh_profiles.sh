#!/bin/bash
# Copies one tools/gpu_round.sh (+ ncu_cfg5.sh) result set into profiles/ (tag = $1, default r2).
set -e
cd "$(dirname "$0")/.."
T=${1:-r2}
python tools/summarize_ncu.py gpurun_out $T > /dev/null
python tools/ncu_summary.py gpurun_out/prof_full.ncu-rep > profiles/${T}_ncu_full_metrics.txt
[ -f gpurun_out/launches_cfg5_1.0.csv ] && python tools/summarize_cfg5.py gpurun_out $T > /dev/null
T=$T python - <<'PY'
import json
lines = open('gpurun_out/bench.json').read().strip().splitlines()
open('profiles/' + __import__('os').environ['T'] + '_bench.json', 'w').write(json.dumps(json.loads(lines[-1]), indent=1) + "\n")
r = [json.loads(l) for l in open('gpurun_out/bench_ref.json').read().strip().splitlines() if l.startswith('{')][-1]
open('profiles/' + __import__('os').environ['T'] + '_bench_reference.json', 'w').write(json.dumps(r, indent=1) + "\n")
PY
cp gpurun_out/launches.csv profiles/${T}_launches.csv
(tail -3 gpurun_out/pytest_gpu.log; echo "--- bounds-asserting build (GNS_LIB=libgns_debug.so):"; tail -1 gpurun_out/pytest_gpu_debug.log) > profiles/${T}_pytest_gpu.txt
echo refreshed
python tools/sass_evidence.py > /dev/null
