#!/bin/bash
# A/B of the persisting L2 window over the PCG slab (RDR_L2_PERSIST=0 off, 1 on regardless of size):
# time per PCG iteration of full solves on configs 2, 5 (p = 6, 10), 6, 4, 3.
for lp in 0 1; do
  for spec in 2 5:6 5:10 6 4 3; do
    RDR_L2_PERSIST=$lp python - <<PY
import json, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg, _, p = "$spec".partition(":")
c = make_config(int(cfg), p=int(p)) if p else make_config(int(cfg))
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
x = torch.empty_like(b)
S.solve(b, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(3):
    e0.record(); _, it = S.solve(b, x); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
ts.sort()
print(json.dumps({"l2_persist": $lp, "cfg": "$spec", "iters": it, "us_per_iter": ts[1] * 1e3 / it}))
PY
  done
done
