#!/bin/bash
bash tools/gpu_sweep.sh "2|" "2|stages=2" "2|stages=3" "4|stages=2" "4|" "3|" 2>&1
