#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | grep -E "Error|assert|passed|failed" | head -20
echo "== race cfg4"; timeout 300 python tools/debug_race.py 4 0.015625 2 2>&1 | grep -c MISMATCH
echo "== race cfg3"; timeout 300 python tools/debug_race.py 3 0.0625 2 2>&1 | grep -c MISMATCH
for c in 1 3; do timeout 300 python tools/profile_run.py --config $c --iters 10 2>&1 | tail -1 | grep -o "'q': [0-9]*\|'probes': [0-9]*\|candidates=[0-9]*\|kernel_ms.*" | tr '\n' ' '; echo; done
bash tools/gpu_sweep.sh "3|probes=2" "3|probes=3" "1|probes=2"
