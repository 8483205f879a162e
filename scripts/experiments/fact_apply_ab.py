"""H(curl): the factored two-stage apply against the DMMA apply with the 12
reference matrices (the tuned layout): plain and PCG-mode apply times, PCG
ms/iteration, iterations, and what setup's timing chose.

    python scripts/experiments/fact_apply_ab.py 4 7:4 7:6 7:8 7:10
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
    out = {"cfg": cfg, "p": c.p, "n_loc": i["n_loc"], "chosen_factored": i["apply_factored"],
           "layout": [i["apply_variant"], i["apply_slots"], i["apply_grid"]], "flops_12mat": i["flops_apply"]}
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    tuned = (i["apply_variant"], i["apply_slots"], i["apply_grid"])
    for name, cfgv in (("dmma", tuned), ("factored", (-1, 0, 0)), ("factored32", (-2, 0, 0)),
                       ("factored32_24", (-3, 0, 0))):
        if not S.set_apply_config(*cfgv):
            continue
        k = min((S.time_kernels(b, b, reps=10) for _ in range(3)), key=lambda v: v[3])
        S.solve(b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        its = 0
        for _ in range(3):
            its += S.solve(b)[1]
        e1.record()
        torch.cuda.synchronize()
        out[name] = {"apply_ms": k[0], "pcg_apply_ms": k[3], "iters": its // 3, "ms_per_iter": e0.elapsed_time(e1) / its}
    print(json.dumps(out), flush=True)
    S.close()
