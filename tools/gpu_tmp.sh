#!/bin/bash
timeout 500 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
echo "== race"; timeout 200 python tools/debug_race.py 4 0.015625 2 2>&1 | grep -c MISMATCH
bash tools/gpu_sweep.sh "2|" "4|" "3|"
