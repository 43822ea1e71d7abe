#!/bin/bash
# Stage-skip timing with the diagnostics build (make diag): for each config
# and MAG_B200_DIAG bit set, the device-resident kernel/step GB/s.
mkdir -p gpurun_out
for c in ${CONFIGS:-2}; do
  for bits in ${BITS:-0 256 768}; do
    echo "cfg$c diag=$bits"
    MAG_B200_PROFILE_LIB=diag MAG_B200_DIAG=$bits timeout 300 python tools/profile_run.py --config $c --iters 10 2>&1 | tail -c 400 | sed -e 's/plan={[^}]*}//'
  done
done
