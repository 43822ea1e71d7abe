#!/bin/bash
# usage: bash tools/gpu_sweep.sh "<cfg>|<opts>" ...  — kernel/step GB/s of forced plans
# (profile_run.py; opts = engine kwargs like variant=shiftor_og,q=12,probes=2)
mkdir -p gpurun_out
for spec in "$@"; do
  c=${spec%%|*}; o=${spec#*|}
  echo "== cfg$c $o"
  timeout 300 python tools/profile_run.py --config $c --iters 5 --opts "$o" 2>&1 | tail -2 | \
    grep -o "'q': [0-9]*\|'k': [0-9]*\|'table_bits': [0-9]*\|'probes': [0-9]*\|'direct': [0-9]*\|'variant': [0-9]*\|matches=[0-9]*\|candidates=[0-9]*\|kernel_ms=.*\|Error.*\|error.*" | tr '\n' ' '
  echo
done
