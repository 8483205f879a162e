#!/bin/bash
# The NEXT rows measured with the current build (DESIGN.md sections 10, 10b): the
# hybrid-preconditioner tests, then the per-config sweeps with the hybrid Schwarz
# preconditioner and with the unsplit decomposition.
#   bash scripts/gpu_next_rows.sh TAG
TAG=${1:-next}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "hybrid or loop_modes or maxit" > gpurun_out/${TAG}_pytest_hybrid.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest_hybrid.log
timeout 1500 python scripts/sweep.py --precond hybrid --configs 2,4,6,5,3 --p 2-10 \
  --out gpurun_out/${TAG}_sweep_hybrid.jsonl > gpurun_out/${TAG}_sweep_hybrid.log 2>&1
echo "hybrid sweep exit $?" >> gpurun_out/${TAG}_sweep_hybrid.log
timeout 1500 python scripts/sweep.py --decomposition unsplit --configs 4,6,5 --p 2-8 \
  --out gpurun_out/${TAG}_sweep_unsplit.jsonl > gpurun_out/${TAG}_sweep_unsplit.log 2>&1
echo "unsplit sweep exit $?" >> gpurun_out/${TAG}_sweep_unsplit.log
tail -3 gpurun_out/${TAG}_pytest_hybrid.log; tail -2 gpurun_out/${TAG}_sweep_hybrid.log; tail -2 gpurun_out/${TAG}_sweep_unsplit.log
