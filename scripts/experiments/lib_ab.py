"""Same-box A/B of two builds of the library: standalone patch / apply times and
PCG ms per iteration per config, for the package under RDR_PKG_ROOT (default:
this checkout). Run once per build, alternating:

    RDR_PKG_ROOT=ab_base python scripts/experiments/lib_ab.py base 6 8:6 4
    python scripts/experiments/lib_ab.py new 6 8:6 4
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.abspath(os.environ.get("RDR_PKG_ROOT", ROOT)))
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

tag = sys.argv[1]
for spec in sys.argv[2:]:
    cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
    c = make_config(cfg, p=p) if p else make_config(cfg)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    i = S.info
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    k = [min(v) for v in zip(*(S.time_kernels(b, b, reps=20).tolist() for _ in range(3)))]
    S.solve(b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    its = 0
    for _ in range(5):
        its += S.solve(b)[1]
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"build": tag, "lib": rdr.LIB_PATH, "cfg": cfg, "p": c.p, "patch_ms": k[2], "patch_GBps": i["patch_bytes"] / k[2] / 1e6,
                      "pcg_apply_ms": k[3], "iters": its // 5, "ms_per_iter": e0.elapsed_time(e1) / its,
                      "small_patch_grid": i["small_patch_grid"], "apply_factored": i["apply_factored"]}), flush=True)
    S.close()
