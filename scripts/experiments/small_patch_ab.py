"""Small-patch kernels (all patches <= 128 dofs, the H(div) edge stars):
standalone patch time and in-solve ms/iteration with the warp-per-patch kernel
and the resident-warp loop kernel forced in turn, and what setup chose.

    python scripts/experiments/small_patch_ab.py 6 8:4 8:6 8:10
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
    out = {"cfg": cfg, "p": c.p, "chosen_grid": S.info["small_patch_grid"], "patch_GB": S.info["patch_bytes"] / 1e9}
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    for name, pers in (("warp", False), ("loop", True)):
        if not S.set_small_patch_kernel(pers):
            continue
        ms = min(S.time_kernels(b, b, reps=20)[2] for _ in range(3))
        S.solve(b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        its = 0
        for _ in range(5):
            its += S.solve(b)[1]
        e1.record()
        torch.cuda.synchronize()
        out[name] = {"patch_ms": ms, "patch_TBps": S.info["patch_bytes"] / ms / 1e9, "ms_per_iter": e0.elapsed_time(e1) / its}
    print(json.dumps(out), flush=True)
    S.close()
