import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import json, sys, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
for spec in sys.argv[1:]:
    cfg, _, p = spec.partition(":")
    c = make_config(int(cfg), p=int(p)) if p else make_config(int(cfg))
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    ms = S.time_kernels(b, b, reps=50)
    x = torch.empty_like(b); S.solve(b, x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); _, it = S.solve(b, x); e1.record(); e1.synchronize()
    print(json.dumps({"cfg": spec, "apply_us": ms[0] * 1e3, "us_per_iter": e0.elapsed_time(e1) * 1e3 / it, "iters": it}))
