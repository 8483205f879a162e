#!/bin/bash
OUT=gpurun_out/race2.txt; : > $OUT
for d in 0; do
  env TAG=dbg$d RDR_APPLY_BM=32 RDR_PDL=0 RDR_APPLY_DBG=$d timeout 600 python scripts/debug_apply_repeat.py 3 10 12 30 >> $OUT 2>&1
done
