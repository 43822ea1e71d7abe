#!/bin/bash
# One ncu --set full capture of the scan kernel of one config (after a plain run).
# usage: C=3 S=0.25 NAME=r02_x [OPTS=...] [DIAGLIB=1 DIAG=bits] bash tools/ncu_one.sh
mkdir -p gpurun_out
P="python tools/profile_run.py --config ${C:-2} --scale ${S:-1.0} --iters 1 ${OPTS:+--opts $OPTS}"
if [ -n "$DIAGLIB" ]; then export MAG_B200_PROFILE_LIB=diag MAG_B200_DIAG=${DIAG:-0}; fi
R=gpurun_out/${NAME:-prof}
$P > gpurun_out/plain_${NAME:-prof}.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:'mag_(direct|scan|roll|pack2)_kernel' -s 2 -c 1 \
    -o $R $P > gpurun_out/ncu_${NAME:-prof}.log 2>&1
tail -3 gpurun_out/ncu_${NAME:-prof}.log
ncu -i $R.ncu-rep --page raw --csv > $R.raw.csv 2>/dev/null
ncu -i $R.ncu-rep --page details --csv > $R.details.csv 2>/dev/null
ncu -i $R.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $R.sass.csv.gz
ls -la $R*
