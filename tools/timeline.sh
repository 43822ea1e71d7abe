#!/bin/bash
# diagnostics build timeline of a few searches (MAG_B200_DIAG=2048 | extra bits)
for c in ${CONFIGS:-2}; do
  echo "cfg$c"
  MAG_B200_PROFILE_LIB=diag MAG_B200_DIAG=$((2048 | ${BITS:-0})) MAG_B200_TIMELINE=1 timeout 300 python tools/profile_run.py --config $c --iters 3 2>&1 | grep -E "timeline|GB/s" | tail -3 | sed -e 's/plan={[^}]*}//' | cut -c1-250
done
