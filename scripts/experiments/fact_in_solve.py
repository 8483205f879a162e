"""In-solve kernel times (rdr_profile_solve) of the DMMA apply (setup's tuned
layout) against the factored apply with each tile size, per config, next to
the graph solve's ms per iteration: where a faster standalone PCG-mode apply
does not give a faster iteration.

    python scripts/experiments/fact_in_solve.py 8:9 7:8 4
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
    out["chosen_split"] = (i["apply_fact_split_a"], i["apply_fact_split_b"])
    for name, cfgv in (("dmma", tuned), ("fact1", (-1, 0, 0)), ("fact2", (-2, 0, 0)), ("fact3", (-3, 0, 0)),
                       ("fact3_s21", (-3, 2, 1)), ("fact3_s22", (-3, 2, 2)), ("fact3_s32", (-3, 3, 2)),
                       ("fact3_s42", (-3, 4, 2)), ("fact2_s22", (-2, 2, 2))):
        if not S.set_apply_config(*cfgv):
            continue
        S.solve(b)
        it, ms = S.profile_solve(b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        its = 0
        for _ in range(3):
            its += S.solve(b)[1]
        e1.record()
        torch.cuda.synchronize()
        alone = S.time_kernels(b, b, reps=10)
        out[name] = {"in_solve_ms": dict(zip(("apply", "update_jacobi", "patches"), [round(v, 4) for v in ms.tolist()[:3]])),
                     "standalone_pcg_apply_ms": round(float(alone[3]), 4), "standalone_patches_ms": round(float(alone[2]), 4),
                     "ms_per_iter": round(e0.elapsed_time(e1) / its, 4), "iters": it}
    print(json.dumps(out), flush=True)
    S.close()
