#!/bin/bash
# A/B of the small-patch path: one CTA per patch (RDR_PATCH_WARP_SMALL=0) vs one
# warp per small patch (n <= 128) in a second launch (default when most patches
# are small), per-launch preconditioner time and time per PCG iteration.
for ws in 0 1; do
  for spec in 6 4 2; do
    RDR_PATCH_WARP_SMALL=$ws python - <<PY
import json, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
c = make_config(int("$spec"))
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
ms = S.time_kernels(b, b, reps=30)
x = torch.empty_like(b)
S.solve(b, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); _, it = S.solve(b, x); e1.record(); e1.synchronize()
gb = (S.info["bytes_precond"] - 24.0 * S.info["n_interior"]) / 1e9
print(json.dumps({"warp_small": $ws, "cfg": "$spec", "patch_us": ms[2] * 1e3, "patch_TBps": gb / ms[2], "iters": it,
                  "us_per_iter": e0.elapsed_time(e1) * 1e3 / it}))
PY
  done
done
