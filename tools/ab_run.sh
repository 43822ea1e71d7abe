#!/bin/bash
# A/B of library builds (libmag_b200_<name>.so) on the same box: kernel/step GB/s per config.
for c in ${CONFIGS:-2}; do
  for lib in ${LIBS:-default}; do
    for rep in ${REPS:-1}; do
      if [ "$lib" = default ]; then unset MAG_B200_PROFILE_LIB; else export MAG_B200_PROFILE_LIB=$lib; fi
      echo "cfg$c lib=$lib"
      timeout 300 python tools/profile_run.py --config $c --iters 10 2>&1 | tail -c 300 | grep -o "matches=.*"
    done
  done
done
