#!/bin/bash
# GPU round: quick parity subset, bench, config sweep, ncu of the patch kernel.
TAG=${1:-run}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "${PYTEST_K:-(small or config1 or config2 or partial or symmetry or error or degenerate) and not high_p}" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
RDR_PCG_HOSTLOOP=1 timeout 900 python bench.py --no-cpu --no-dgemm > gpurun_out/${TAG}_bench_hostloop.log 2>&1
timeout 1500 python scripts/sweep.py --configs ${SWEEP_CFGS:-1,2,4,5,3} --out gpurun_out/${TAG}_sweep.jsonl > gpurun_out/${TAG}_sweep.log 2>&1
echo "sweep exit $?" >> gpurun_out/${TAG}_sweep.log
if [ -n "$NCU" ]; then
  python scripts/prof_kernels.py 2 6 3 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"patch_ldg" -s 1 -c 2 \
      -o gpurun_out/${TAG}_patch -f python scripts/prof_kernels.py 2 6 3 > gpurun_out/${TAG}_ncu.log 2>&1
  echo "ncu exit $?" >> gpurun_out/${TAG}_ncu.log
fi
