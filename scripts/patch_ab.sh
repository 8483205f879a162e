#!/bin/bash
# A/B of the patch-kernel launch shape (in-solve and standalone patch times, scripts/profile_solve.py):
# default vs RDR_PATCH_WARPS=4|8 (warps per patch CTA) and RDR_PATCH_WARP_SMALL=1 (patches <= 128 dofs
# one per warp in a second launch).   bash scripts/patch_ab.sh TAG "2 4 6 5:10 3"
TAG=${1:-pab}; CFGS=${2:-"2 4 6 5:10"}
mkdir -p gpurun_out
run() { timeout 600 env "$@" python scripts/profile_solve.py $CFGS 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l)
        print('$*', d['cfg'], d['p'], 'patch in-solve', round(d['in_solve_ms']['patches'], 4), 'alone', round(d['standalone_ms']['patches'], 4),
              'apply', round(d['in_solve_ms']['apply'], 4), d.get('apply_layout'))
"; }
run X=0 | tee gpurun_out/${TAG}.log
run RDR_PATCH_WARPS=4 | tee -a gpurun_out/${TAG}.log
run RDR_PATCH_WARPS=8 | tee -a gpurun_out/${TAG}.log
run RDR_PATCH_WARP_SMALL=1 | tee -a gpurun_out/${TAG}.log
run RDR_PATCH_WARP_SMALL=1 RDR_PATCH_WARPS=8 | tee -a gpurun_out/${TAG}.log
