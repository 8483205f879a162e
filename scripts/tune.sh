#!/bin/bash
# Kernel-variant timings (rdr_time_kernels) per config: apply BM, patch warps/CTA.
TAG=${1:-tune}
mkdir -p gpurun_out
OUT=gpurun_out/${TAG}.txt
: > $OUT
for cp in "2 6" "4 6" "5 10" "5 12"; do
  for env in "RDR_APPLY_BM=16" "RDR_APPLY_BM=32" "RDR_APPLY_BM=64" "RDR_PATCH_WARPS=4" "RDR_PATCH_KERNEL=tma"; do
    echo "== cfg/p $cp $env" >> $OUT
    env $env timeout 600 python scripts/prof_kernels.py $cp 20 2>&1 | grep "kernel ms" | cut -c1-90 >> $OUT
  done
done
