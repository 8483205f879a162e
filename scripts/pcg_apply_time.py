"""Fused PCG-mode apply vs plain apply, warm, per launch (rdr_debug_fused_apply
includes three vector memsets and the scalar upload; subtract ~3 x 8 N / HBM).
    python scripts/pcg_apply_time.py 2 4 6 3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import json, sys, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
for spec in sys.argv[1:]:
    cfg, _, p = spec.partition(":")
    c = make_config(int(cfg), p=int(p)) if p else make_config(int(cfg))
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    z = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    q = torch.empty_like(z)
    ms = S.time_kernels(z, z, reps=20)
    for _ in range(3):
        S.debug_fused_apply(z, q)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t = []
    for _ in range(10):
        e0.record(); S.debug_fused_apply(z, q); e1.record(); e1.synchronize(); t.append(e0.elapsed_time(e1))
    t.sort()
    print(json.dumps({"cfg": spec, "plain_apply_us": ms[0] * 1e3, "pcg_apply_us_incl_sync": t[len(t) // 2] * 1e3}))
