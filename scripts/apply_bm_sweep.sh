#!/bin/bash
# apply kernel cells-per-CTA experiment: per-launch device time of the operator
# apply (rdr_time_kernels) and the solve's time per iteration on configs
# 2, 4, 6, 5:10 for BM = 16 / 32 (RDR_APPLY_BM).
for cfg in 2 4 6 5:10; do
  for bm in 16 32; do
    RDR_APPLY_BM=$bm python - <<PY
import json, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg, _, p = "$cfg".partition(":")
c = make_config(int(cfg), p=int(p)) if p else make_config(int(cfg))
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
ms = S.time_kernels(b, b, reps=50)
x = torch.empty_like(b)
S.solve(b, x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); _, it = S.solve(b, x); e1.record(); e1.synchronize()
print(json.dumps({"cfg": "$cfg", "bm": $bm, "apply_us": ms[0] * 1e3, "patch_us": ms[2] * 1e3, "iters": it,
                  "us_per_iter": e0.elapsed_time(e1) * 1e3 / it}))
PY
  done
done
