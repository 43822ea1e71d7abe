#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command and one --set full
# capture of the top scan kernel per config.  Each command first runs plain (&&).
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1"
$B > gpurun_out/plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launches.log 2>&1
for c in ${CFGS:-2 3 4 5 1}; do
  P="python tools/profile_run.py --config $c --iters 1"
  $P > gpurun_out/plain_cfg$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:'mag_(direct|scan)_kernel' -s 2 -c 1 \
      -o gpurun_out/full_cfg$c $P > gpurun_out/ncu_full_cfg$c.log 2>&1
  tail -3 gpurun_out/ncu_full_cfg$c.log
done
ls -la gpurun_out
