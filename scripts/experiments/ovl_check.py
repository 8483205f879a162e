"""Overlapped PCG iteration (RDR_LOOP_OVERLAP) against the
single-partition graph (RDR_LOOP_GRAPH) on the same config: iterations, x,
time per iteration; and what RDR_LOOP_DEVICE chose at setup.

    python scripts/ovl_check.py 2 3 4 5:10
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402


def timed(S, b, reps=3):
    x, it = S.solve(b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        x, it = S.solve(b)
    e1.record()
    torch.cuda.synchronize()
    return x, it, e0.elapsed_time(e1) / reps


def main():
    for spec in sys.argv[1:]:
        cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
        c = make_config(cfg, p=p) if p else make_config(cfg)
        out = {"cfg": cfg, "p": c.p}
        b = None
        xs = {}
        for name, loop in (("graph", rdr.LOOP_GRAPH), ("overlap", rdr.LOOP_OVERLAP), ("device", rdr.LOOP_DEVICE)):
            try:
                S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=loop)
            except rdr.RdrError as e:
                out[name] = str(e)
                continue
            if b is None:
                b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
            x, it, ms = timed(S, b)
            st = S.last_stats()
            xs[name] = x.cpu().numpy()
            out[name] = {"iters": it, "ms": ms, "ms_per_iter": ms / max(it, 1), "converged": st["converged"],
                         "z_ratio": st["z_last"] / st["z0"] if st["z0"] else 0.0,
                         "overlap_sms": S.info["overlap_sms"], "setup_s": S.info["setup_seconds"]}
            S.close()
        if "graph" in xs:
            for k in ("overlap", "device"):
                if k in xs:
                    out[k]["x_rel_vs_graph"] = float(np.linalg.norm(xs[k] - xs["graph"]) / np.linalg.norm(xs["graph"]))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
