#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "roll" 2>&1 | tail -15 > gpurun_out/pytest_roll.log
cat gpurun_out/pytest_roll.log
bash tools/gpu_sweep.sh "5|scan_kernel=roll,probes=2" "5|scan_kernel=roll,probes=3" "3|scan_kernel=roll,probes=2" "3|scan_kernel=roll,probes=3" \
  "4|scan_kernel=roll,probes=2" "4|scan_kernel=roll,probes=3" "2|scan_kernel=roll,probes=3" 2>&1 | tee gpurun_out/exp2.log
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
cat gpurun_out/pytest_gpu.log
