#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command and one --set full
# capture of the top scan kernel per config.  Each command first runs plain (&&).
# Reports are exported to CSV on the box (raw, details, source) and only
# $KEEP_REP's .ncu-rep is kept (gpurun copies back <= 64 MiB).
mkdir -p gpurun_out
if [ -z "$SKIP_LAUNCHES" ]; then
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --headline-only"
$B > gpurun_out/plain_bench.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/ncu_launches.log 2>&1
fi
for c in ${CFGS:-2 3 4 5 1}; do
  P="python tools/profile_run.py --config $c --iters 1 ${PROF_OPTS:+--opts $PROF_OPTS}"
  R=gpurun_out/full_cfg$c${TAG}
  $P > gpurun_out/plain_cfg$c.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:'mag_(direct|scan|roll|pack2)_kernel' -s 2 -c 1 \
      -o $R $P > gpurun_out/ncu_full_cfg$c.log 2>&1
  tail -2 gpurun_out/ncu_full_cfg$c.log
  ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
  ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
  ncu -i $R.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $R.sass.csv.gz
  [ "$c" = "${KEEP_REP:-2}" ] || rm -f $R.ncu-rep
done
ls -la gpurun_out
