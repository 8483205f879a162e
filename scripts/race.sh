#!/bin/bash
OUT=gpurun_out/race.txt; : > $OUT
for env in "TAG=bm32 RDR_APPLY_BM=32" "TAG=bm16 RDR_APPLY_BM=16" "TAG=bm64 RDR_APPLY_BM=64" "TAG=bm32nopdl RDR_APPLY_BM=32 RDR_PDL=0"; do
  env $env timeout 600 python scripts/debug_apply_repeat.py 3 10 12 40 >> $OUT 2>&1
done
env TAG=p6bm32 RDR_APPLY_BM=32 timeout 600 python scripts/debug_apply_repeat.py 3 6 16 40 >> $OUT 2>&1
