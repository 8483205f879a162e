#!/bin/bash
# Launch list of the bench solve (graph kernel nodes profiled one by one; ncu cannot
# profile the nodes of a graph with conditional nodes, so the solve runs its
# host-driven 8-iteration graphs here: the same kernels).
TAG=${1:-launches}
python bench.py --steps 2 --warmup 3 --no-cpu --no-dgemm > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --graph-profiling node --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"apply_tc|patch_ldg|pcg_|precond_init" -s 300 -c 400 --csv \
    --log-file gpurun_out/${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-dgemm > gpurun_out/${TAG}_ncu.log 2>&1
echo "exit $?" >> gpurun_out/${TAG}_ncu.log
