#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | grep -E "Error|assert|passed|failed" | head -20
echo "== race"; timeout 300 python tools/debug_race.py 4 0.015625 3 2>&1 | grep -c MISMATCH
bash tools/gpu_sweep.sh "2|" "4|" "2|probes=2"
