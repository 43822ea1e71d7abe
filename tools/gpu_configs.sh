#!/bin/bash
# per-round check: GPU test suite + per-config kernel/step GB/s (tools/profile_run.py)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
for c in 1 2 3 4 5; do timeout 200 python tools/profile_run.py --config $c --iters 10 > gpurun_out/prof_cfg$c.log 2>&1; tail -1 gpurun_out/prof_cfg$c.log | grep -o "'q': [0-9]*\|'probes': [0-9]*\|'direct': [0-9]*\|'roll': [0-9]*\|candidates=[0-9]*\|kernel_ms.*" | tr '\n' ' '; echo; done
