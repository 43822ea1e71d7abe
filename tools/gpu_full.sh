#!/bin/bash
# full round check: GPU tests, per-config kernel/step GB/s, bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; cat gpurun_out/pytest_gpu.log
for c in 1 2 3 4 5; do timeout 300 python tools/profile_run.py --config $c --iters 10 > gpurun_out/prof_cfg$c.log 2>&1; tail -c 700 gpurun_out/prof_cfg$c.log; echo; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
