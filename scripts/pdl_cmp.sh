#!/bin/bash
TAG=${1:-pdl}
: > gpurun_out/${TAG}.txt
for env in "RDR_PDL=0" "RDR_PDL=1" "RDR_PDL_PATCH=0"; do
  for cfg in 2 4; do
    echo "== $env cfg$cfg" >> gpurun_out/${TAG}.txt
    env $env timeout 300 python bench.py --no-cpu --no-dgemm --config $cfg --steps 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],1), 'us/iter', round(d['ms_per_iter']*1e3,2), d['kernel_ms'])
" >> gpurun_out/${TAG}.txt
  done
done
