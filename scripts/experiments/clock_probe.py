"""SM clock behind the fused apply, inside the PCG iteration and in a loop of
applies alone (rdr_debug_profile_clocks), for the DMMA apply (setup's layout)
and the factored apply: does the clock the power cap leaves explain the
in-solve apply times?

    python scripts/experiments/clock_probe.py 3 4 6 7:8 8:9 8:10 2
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

for spec in sys.argv[1:]:
    cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
    c = make_config(cfg, p=p) if p else make_config(cfg)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    i = S.info
    tuned = (i["apply_variant"], i["apply_slots"], i["apply_grid"])
    out = {"cfg": cfg, "p": c.p, "chosen_factored": i["apply_factored"]}
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    iters = 40 if i["n_free"] > 2e6 else 200
    for name, cfgv in (("dmma", tuned), ("fact3", (-3, 0, 0))):
        if not S.set_apply_config(*cfgv):
            continue
        S.solve(b)
        r = [S.profile_clocks(b, iters=iters) for _ in range(2)][1]
        out[name] = {"mhz_in_iteration": round(float(r[0])), "mhz_alone": round(float(r[1])),
                     "ms_per_iter": round(float(r[2]), 4), "apply_alone_ms": round(float(r[3]), 4)}
    print(json.dumps(out), flush=True)
    S.close()
