#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "roll" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
echo "== race"; timeout 300 python tools/debug_race.py 4 0.015625 3 2>&1 | grep -c MISMATCH
bash tools/gpu_sweep.sh "2|" "5|scan_kernel=roll,probes=2" "5|scan_kernel=roll,probes=3" "3|scan_kernel=roll,probes=2" 2>&1 | tee gpurun_out/exp6.log
