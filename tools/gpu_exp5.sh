#!/bin/bash
mkdir -p gpurun_out
echo "== race default"; timeout 300 python tools/debug_race.py 4 0.015625 5 2>&1 | grep -c MISMATCH
bash tools/gpu_sweep.sh "2|" "4|" "5|scan_kernel=roll,probes=2" "5|scan_kernel=roll,probes=3" 2>&1 | tee gpurun_out/exp5.log
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
