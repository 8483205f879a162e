#!/bin/bash
# Full GPU round trip (run under gpurun): parity tests, bench, launch list and
# ncu --set full captures of the two hot kernels on the bench workload.
#   gpurun --timeout 3000 -- bash scripts/gpu_round.sh TAG
TAG=${1:-run}
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} ${PYTEST_EXTRA} > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
if [ -n "$SWEEP" ]; then
  timeout 2400 python scripts/sweep.py --configs 1,2,4,5,3 --p 1-12 --out gpurun_out/${TAG}_sweep.jsonl > gpurun_out/${TAG}_sweep.log 2>&1
  echo "sweep exit $?" >> gpurun_out/${TAG}_sweep.log
fi
if [ -n "$NCU" ]; then
  python bench.py --steps 2 --warmup 3 --no-cpu --no-dgemm > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 400 --csv \
      --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dgemm > gpurun_out/${TAG}_ncu1.log 2>&1
  python scripts/prof_kernels.py 2 6 3 > gpurun_out/${TAG}_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"patch_ldg|apply_tc" -s 2 -c 2 \
      -o gpurun_out/${TAG}_full -f python scripts/prof_kernels.py 2 6 3 > gpurun_out/${TAG}_ncu2.log 2>&1
  echo "ncu exit $?" >> gpurun_out/${TAG}_ncu2.log
fi
