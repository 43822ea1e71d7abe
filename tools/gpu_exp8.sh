#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "roll or hashed or full_configs" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
for c in 1 3 5; do timeout 300 python tools/profile_run.py --config $c --iters 10 2>&1 | tail -1 | grep -o "candidates=[0-9]*\|kernel_ms.*"; done
for c in 3 5; do
  P="python tools/profile_run.py --config $c --iters 1"
  R=gpurun_out/roll_cfg$c
  $P > gpurun_out/plain_roll$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:'mag_roll_kernel' -s 2 -c 1 -o $R $P > gpurun_out/ncu_roll$c.log 2>&1
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $R.sass.csv.gz
  rm -f $R.ncu-rep
done
