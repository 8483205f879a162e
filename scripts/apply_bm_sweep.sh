#!/bin/bash
# apply kernel cells-per-CTA experiment: per-launch device time of the operator
# apply (rdr_time_kernels) on configs 2, 4, 6 for BM = 16 / 32 / 64.
for cfg in 2 4 6; do
  for bm in 16 32 64; do
    RDR_APPLY_BM=$bm python - <<PY
import json, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
c = make_config($cfg)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
ms = S.time_kernels(b, b, reps=50)
print(json.dumps({"cfg": $cfg, "bm": $bm, "apply_us": ms[0] * 1e3, "patch_us": ms[2] * 1e3}))
PY
  done
done
