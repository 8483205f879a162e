#!/bin/bash
# Round-end style GPU run plus the per-config sweep (DESIGN.md section 7 table):
#   bash scripts/gpu_final_sweep.sh TAG
TAG=${1:-final}
bash scripts/gpu_final.sh $TAG
timeout 1500 python scripts/sweep.py --configs 1,2,4,6,3,5,7,8 --p 1-12 --out gpurun_out/${TAG}_sweep_split.jsonl \
  > gpurun_out/${TAG}_sweep.log 2>&1
echo "sweep exit $?" >> gpurun_out/${TAG}_sweep.log
