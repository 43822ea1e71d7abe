#!/bin/bash
# A/B with environment settings: ENVS="A=1 B=2" per run (';'-separated list of env settings)
IFS=';' read -ra RUNS <<< "${ENVS:-}"
for c in ${CONFIGS:-2}; do
  for r in "${RUNS[@]}"; do
    echo "cfg$c env=[$r]"
    env $r timeout 300 python tools/profile_run.py --config $c --iters 10 2>&1 | tail -c 300 | grep -o "matches=.*"
  done
done
