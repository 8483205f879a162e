#!/bin/bash
# patch-kernel variants per config (full kernel-ms lines)
TAG=${1:-tune2}
OUT=gpurun_out/${TAG}.txt
: > $OUT
for cp in "2 6" "4 6" "5 10" "5 12"; do
  for env in "X=0"; do
    echo "== cfg/p $cp $env" >> $OUT
    env $env timeout 600 python scripts/prof_kernels.py $cp 20 2>&1 | grep "kernel ms" | cut -d'{' -f1 >> $OUT
  done
done
