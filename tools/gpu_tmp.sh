#!/bin/bash
# scratch GPU command of the current iteration
mkdir -p gpurun_out
P="python tools/profile_run.py --config 5 --iters 2 --opts warps=${W:-16}"
$P > gpurun_out/plain5.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg5.csv $P > /dev/null 2>&1
grep -v "^==" gpurun_out/launches_cfg5.csv | awk -F'","' '{print $5, $NF}' | tail -12
ncu --set full --clock-control none --import-source on -k regex:'mag_roll_kernel' -s 2 -c 1 -o gpurun_out/full_cfg5_r02c $P > gpurun_out/ncu5.log 2>&1
ncu -i gpurun_out/full_cfg5_r02c.ncu-rep --page details --csv > gpurun_out/full_cfg5_r02c.details.csv 2>/dev/null
ncu -i gpurun_out/full_cfg5_r02c.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/full_cfg5_r02c.sass.csv.gz
rm -f gpurun_out/full_cfg5_r02c.ncu-rep
