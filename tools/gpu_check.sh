#!/bin/bash
# GPU tests + per-config kernel/step GB/s (device-resident), no bench line
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv
nproc; lscpu | grep "Model name"
timeout ${PYTEST_TIMEOUT:-1500} python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} 2>&1 | tail -25 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-1 2 3 4 5}; do timeout 300 python tools/profile_run.py --config $c --iters 10 > gpurun_out/prof_cfg$c.log 2>&1; tail -c 900 gpurun_out/prof_cfg$c.log; echo; done
