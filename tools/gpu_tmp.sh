#!/bin/bash
# scratch GPU command of the current iteration
mkdir -p gpurun_out
for c in 1 2 3 4 5; do echo "== cfg$c exact (reference-default params)"; timeout 300 python tools/profile_run.py --config $c --iters 3 --opts gram_mode=0 2>&1 | tail -c 1500; echo; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
