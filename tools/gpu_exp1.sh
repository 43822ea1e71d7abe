#!/bin/bash
bash tools/gpu_sweep.sh "5|variant=shiftor_og,q=12" "5|variant=shiftor_og,q=12,probes=2" "5|variant=shiftor_og,q=12,probes=3" \
  "5|variant=shiftor_og,q=10,probes=2" "5|table_bits=-1" "5|variant=shiftor_og" \
  "4|probes=2" "4|probes=3" "4|probes=4" "4|variant=shiftor_og,q=16,probes=3" \
  "3|q=8,k=1" "3|q=6,k=1" "3|variant=shiftor_og,q=16,probes=3" "3|variant=shiftor_og,q=12,probes=2" \
  "2|probes=2" "2|probes=3" "2|probes=4" 2>&1 | tee gpurun_out/exp1.log
SKIP_LAUNCHES= CFGS="2 4 5" bash tools/gpu_ncu.sh
