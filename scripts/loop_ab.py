"""Time per PCG iteration with each rdr_options.loop (device-side graph vs the
persistent cooperative kernel, plus what RDR_LOOP_DEVICE chose) per config:
    python scripts/loop_ab.py 1 5:1 5:2 5:3 5:4 2"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402


def per_iter(S, b, solves=5):
    S.solve(b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = 0
    e0.record()
    for _ in range(solves):
        its += S.solve(b)[1]
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / its * 1e3, its / solves


for spec in sys.argv[1:]:
    cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
    c = make_config(cfg, p=p) if p else make_config(cfg)
    out = {"cfg": cfg, "p": c.p}
    b = None
    for name, loop in (("graph", rdr.LOOP_GRAPH), ("persistent", rdr.LOOP_PERSISTENT), ("device", rdr.LOOP_DEVICE)):
        try:
            S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=loop)
        except rdr.RdrError as e:
            out[name] = str(e)
            continue
        if b is None:
            b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
        us, it = per_iter(S, b)
        out[name] = {"us_per_iter": round(us, 2), "iters": it, "persistent": S.info["persistent_loop"]}
        S.close()
    print(json.dumps(out), flush=True)
