#!/bin/bash
# round-1 final evidence: bench line (all configs), launch list, --set full of the scan kernel per config
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.log 2>&1; tail -c 4000 gpurun_out/bench_final.log
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --headline-only"
$B > gpurun_out/plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launches.log 2>&1
for c in 2 3 5 4; do
  P="python tools/profile_run.py --config $c --iters 1"
  R=gpurun_out/full_cfg$c
  $P > gpurun_out/plain_cfg$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:'mag_(direct|scan|roll)_kernel' -s 2 -c 1 \
      -o $R $P > gpurun_out/ncu_full_cfg$c.log 2>&1
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $R.sass.csv.gz
  [ "$c" = "2" ] || rm -f $R.ncu-rep
done
ls -la gpurun_out | head -40
