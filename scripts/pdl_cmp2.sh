#!/bin/bash
TAG=${1:-pdl2}
: > gpurun_out/${TAG}.txt
for env in "RDR_PDL=0 RDR_PCG_HOSTLOOP=1" "RDR_PDL=1 RDR_PCG_HOSTLOOP=1" "RDR_PDL=0" "RDR_PDL=1"; do
  echo "== $env" >> gpurun_out/${TAG}.txt
  env $env timeout 300 python bench.py --no-cpu --no-dgemm --config 2 --steps 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value'],1), 'us/iter', round(d['ms_per_iter']*1e3,2))
" >> gpurun_out/${TAG}.txt
done
