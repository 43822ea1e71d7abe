#!/bin/bash
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
bash tools/gpu_sweep.sh "2|" "4|" "3|"
