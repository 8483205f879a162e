"""Per-iteration time of the persistent cooperative PCG kernel against the
graph loop on the small p-sweep points (where setup's timing chooses).

    python scripts/experiments/persistent_vs_graph.py 5:1 5:2 5:3 5:4 7:2 7:3 8:2 8:3
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402


def per_iter(S, b):
    S.solve(b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    its = 0
    for _ in range(10):
        its += S.solve(b)[1]
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / its * 1e3


for spec in sys.argv[1:]:
    cfg, p = (int(v) for v in spec.split(":"))
    c = make_config(cfg, p=p)
    out = {"cfg": cfg, "p": p}
    b = None
    for name, loop in (("graph", rdr.LOOP_GRAPH), ("persistent", rdr.LOOP_PERSISTENT), ("device", rdr.LOOP_DEVICE)):
        try:
            S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=loop)
        except rdr.RdrError as e:
            out[name] = "not eligible"
            continue
        if b is None:
            b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
        out[name] = round(per_iter(S, b), 2)
        if name == "device":
            out["device_chose_persistent"] = S.info["persistent_loop"]
        S.close()
    print(json.dumps(out), flush=True)
