#!/bin/bash
mkdir -p gpurun_out
for d in 0 64 128 192; do echo "== DIAG=$d"; MAG_B200_DIAG=$d timeout 300 python tools/debug_race.py 4 0.015625 4 2>&1 | grep -c MISMATCH; done 2>&1 | tee gpurun_out/exp4.log
for o in "probes=2" "warps=4" "scan_kernel=staged"; do echo "== $o"; timeout 300 python tools/debug_race.py 4 0.015625 4 $o 2>&1 | grep -c MISMATCH; done 2>&1 | tee -a gpurun_out/exp4.log
