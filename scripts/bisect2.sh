#!/bin/bash
OUT=gpurun_out/bisect2.txt; : > $OUT
for args in "3 6" "3 10 12" "5 10 16" "3 10" ; do
  for env in "TAG=bm32 RDR_APPLY_BM=32" "TAG=bm16 RDR_APPLY_BM=16"; do
    echo "args $args" >> $OUT
    env $env timeout 600 python scripts/debug_pcg_resid.py $args >> $OUT 2>&1
  done
done
