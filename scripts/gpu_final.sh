#!/bin/bash
# Round-end style GPU run: all GPU tests, smoke, bench, launch list and ncu --set full of the two hot kernels.
TAG=${1:-final}
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${TAG}_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
# launch list of the bench solve, graph nodes one by one (host-driven 8-iteration graphs:
# ncu cannot profile the nodes of a graph with a conditional while node)
RDR_PCG_HOSTLOOP=1 bash scripts/ncu_launches.sh ${TAG}_launches
python scripts/prof_kernels.py 2 6 3 > gpurun_out/${TAG}_prof_plain.log 2>&1
for K in patch_ldg apply_tc; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
      -o gpurun_out/${TAG}_full_$K -f python scripts/prof_kernels.py 2 6 3 > gpurun_out/${TAG}_ncu_$K.log 2>&1
  echo "ncu exit $?" >> gpurun_out/${TAG}_ncu_$K.log
done
