#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "roll or full_configs" 2>&1 | grep -E "Error|assert|passed|failed" | head
bash tools/gpu_sweep.sh "5|" "5|probes=2" "3|scan_kernel=roll"
