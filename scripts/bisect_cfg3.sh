#!/bin/bash
OUT=gpurun_out/bisect.txt; : > $OUT
for env in "TAG=default" "TAG=nopdl RDR_PDL=0" "TAG=hostloop RDR_PCG_HOSTLOOP=1" "TAG=bm64 RDR_APPLY_BM=64" "TAG=unfused RDR_PCG_UNFUSED=1"; do
  env $env timeout 600 python scripts/debug_pcg_resid.py ${CFG:-3} ${P:-} >> $OUT 2>&1
done
