set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for c in 1 2 3 4 5; do timeout 300 python tools/profile_run.py --config $c --iters 10 > gpurun_out/prof_cfg$c.log 2>&1; tail -c 1500 gpurun_out/prof_cfg$c.log; done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log
