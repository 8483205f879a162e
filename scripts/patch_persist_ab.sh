#!/bin/bash
# A/B of the patch kernel launch: one CTA per patch (RDR_PATCH_PERSIST=0) vs
# persistent CTAs claiming patches from a queue (default), per-launch device time.
for pers in 0 1; do
  for spec in 2 4 6 5:8 5:10 5:12 3; do
    RDR_PATCH_PERSIST=$pers python - <<PY
import json, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg, _, p = "$spec".partition(":")
c = make_config(int(cfg), p=int(p)) if p else make_config(int(cfg))
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
ms = S.time_kernels(b, b, reps=30)
x = torch.empty_like(b)
S.solve(b, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); _, it = S.solve(b, x); e1.record(); e1.synchronize()
gb = (S.info["bytes_precond"] - 24.0 * S.info["n_interior"]) / 1e9
print(json.dumps({"persist": $pers, "cfg": "$spec", "patch_us": ms[2] * 1e3, "patch_TBps": gb / ms[2], "iters": it,
                  "us_per_iter": e0.elapsed_time(e1) * 1e3 / it}))
PY
  done
done
