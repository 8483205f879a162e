#!/bin/bash
# ncu --set full capture of one kernel launch (run under gpurun, one GPU).
#   bash scripts/ncu_kernel.sh TAG KERNEL_REGEX [config] [p]
TAG=$1; KRE=$2; CFG=${3:-2}; P=${4:-6}
mkdir -p gpurun_out
python scripts/prof_kernels.py $CFG $P 3 > gpurun_out/${TAG}_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:${KRE} --launch-skip 2 -c 1 \
  -o gpurun_out/${TAG} -f python scripts/prof_kernels.py $CFG $P 3 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/${TAG}_ncu.log
