#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/debug_race.py 4 0.015625 6 2>&1 | tail -20 | tee gpurun_out/race.log
P="python tools/profile_run.py --config 3 --iters 1 --opts scan_kernel=roll,probes=2"
$P > gpurun_out/plain_roll3.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'mag_roll_kernel' -s 2 -c 1 -o gpurun_out/roll_cfg3 $P > gpurun_out/ncu_roll3.log 2>&1
ncu -i gpurun_out/roll_cfg3.ncu-rep --page raw --csv > gpurun_out/roll_cfg3.raw.csv 2>/dev/null
ncu -i gpurun_out/roll_cfg3.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/roll_cfg3.sass.csv.gz
rm -f gpurun_out/roll_cfg3.ncu-rep
bash tools/gpu_sweep.sh "2|warps=24" "2|warps=16" "4|warps=24" 2>&1 | tee gpurun_out/exp3.log
