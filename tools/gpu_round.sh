#!/bin/bash
# One full GPU validation + measurement round (run under gpurun).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_gpu.log
# the same suite on the bounds-asserting build (make debug): every shared-memory
# slot, slice and bulk-copy range checked on the device
GNS_LIB=libgns_debug.so timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_debug.log 2>&1; echo "pytest_debug_rc=$?"; tail -1 gpurun_out/pytest_gpu_debug.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo "ref_rc=$?"
python bench.py --profile-only --warmup 1 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --profile-only --warmup 1 > gpurun_out/ncu_list.log 2>&1; echo "ncu_list_rc=$?"
python bench.py --profile-only --warmup 1 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"merge_tstore|tile_sort3" -s 12 -c 2 \
    -o gpurun_out/prof_full python bench.py --profile-only --warmup 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu_full_rc=$?"
python tools/f32_once.py > gpurun_out/plain_f32.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"f32_merge" -s 11 -c 1 \
    -o gpurun_out/prof_f32 python tools/f32_once.py > gpurun_out/ncu_f32.log 2>&1; echo "ncu_f32_rc=$?"
