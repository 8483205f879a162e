#!/bin/bash
# Same-box A/B of the round-1 library (commit 87a231a) against the current one on
# small configs: builds the round-1 package under abtmp/old_r1 (git-ignored), then
# runs abtmp/ab_small.py on the GPU:  bash scripts/experiments/ab_round1.sh, then
#   gpurun -- 'python abtmp/ab_small.py 1 5:1 5:2 5:3 5:4 5:5 8:3 8:4 7:3 2'
set -e
rm -rf /tmp/oldpkg abtmp/old_r1 abtmp/include && mkdir -p /tmp/oldpkg abtmp
git archive 87a231a paper_2506_17406_b200 include | tar -x -C /tmp/oldpkg
cp -r /tmp/oldpkg/paper_2506_17406_b200 abtmp/old_r1 && cp -r /tmp/oldpkg/include abtmp/include
(cd abtmp && python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('b', 'old_r1/build.py'); b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b); b.build()")
cp scripts/experiments/ab_small.py abtmp/ab_small.py
