#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "roll or hashed or full_configs or reduced" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
for c in 1 3 5; do timeout 300 python tools/profile_run.py --config $c --iters 10 2>&1 | tail -1 | grep -o "'probes': [0-9]*\|candidates=[0-9]*\|kernel_ms.*" | tr '\n' ' '; echo; done
bash tools/gpu_sweep.sh "5|scan_kernel=roll,probes=2" "3|scan_kernel=roll,probes=3" "3|scan_kernel=roll,probes=1"
