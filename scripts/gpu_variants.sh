#!/bin/bash
# A/B of the apply kernel's warp layouts (RDR_APPLY_VARIANT = layout 0..3 of kernels.cu
# apply_variants): parity subset, then in-solve and standalone times per config, then
# ncu --set full of the standalone apply of config 4 per layout.
#   bash scripts/gpu_variants.sh TAG "0 1 2" "3 4 5:10 2" [ncu]
TAG=${1:-v}; VARS=${2:-"0 1 2"}; CFGS=${3:-"3 4 5:10 2"}; NCU=${4:-}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hgrad_small or config1 or loop_modes or ring_race or test_config2 or hdiv_small or hcurl_small or symmetry" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
for v in $VARS; do
  RDR_APPLY_VARIANT=$v timeout 300 python scripts/profile_solve.py $CFGS > gpurun_out/${TAG}_prof_$v.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_prof_$v.log
done
if [ -n "$NCU" ]; then
for v in $VARS; do
  RDR_APPLY_VARIANT=$v timeout 300 python scripts/prof_kernels.py 4 - 3 > gpurun_out/${TAG}_plain_$v.log 2>&1 && \
  RDR_APPLY_VARIANT=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:apply_tc -s 2 -c 1 \
      -o gpurun_out/${TAG}_ncu_$v -f python scripts/prof_kernels.py 4 - 3 > gpurun_out/${TAG}_ncu_$v.log 2>&1
done
fi
for v in $VARS; do echo "== variant $v"; python - gpurun_out/${TAG}_prof_$v.log <<'PY'
import sys, json
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l)
        print(d['cfg'], d['p'], d['iters'], 'in-solve', round(d['in_solve_ms']['apply'], 4), round(d['apply_tflops_in_solve'], 1),
              'alone', round(d['standalone_ms']['apply'], 4), round(d['apply_tflops_standalone'], 1),
              'patch', round(d['in_solve_ms']['patches'], 4))
    else:
        print(l.strip()[:200])
PY
done
