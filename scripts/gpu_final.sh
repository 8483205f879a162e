#!/bin/bash
# Round-end style GPU run (under gpurun, one GPU): all GPU tests, smoke, the default
# bench line (config 3), the reference arm, and the ncu launch list of the bench solve.
#   bash scripts/gpu_final.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --durations=40 > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
echo "reference exit $?" >> gpurun_out/${TAG}_bench_ref.log
bash scripts/ncu_launches.sh ${TAG}_launches
python scripts/ncu_summary.py launches gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_launches.txt 2>&1
rm -f gpurun_out/${TAG}_launches.csv
tail -3 gpurun_out/${TAG}_pytest.log; tail -2 gpurun_out/${TAG}_smoke.log; cat gpurun_out/${TAG}_launches.txt
