#!/bin/bash
# Launch list of the bench solve: bench.py with --loop host (8-iteration graphs
# relaunched by the host; ncu profiles their kernel nodes one by one, which it
# cannot do inside the default graph's conditional WHILE node) -- the same
# kernels as the default command.
#   bash scripts/ncu_launches.sh TAG [extra bench.py args]
TAG=${1:-launches}; shift
python bench.py --steps 2 --warmup 3 --no-cpu --no-dgemm --no-sweep --loop host "$@" > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"apply_tc|patch_ldg|patch_warp|pcg_|precond_init" -s 300 -c 400 --csv \
    --log-file gpurun_out/${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dgemm --no-sweep --loop host "$@" \
    > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_ncu.log
