#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "roll or hashed or golden_fix" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
bash tools/gpu_sweep.sh "2|" "5|scan_kernel=roll,probes=2" "5|scan_kernel=roll,probes=3" "3|scan_kernel=roll,probes=2" "4|scan_kernel=roll,probes=3" 2>&1 | tee gpurun_out/exp7.log
