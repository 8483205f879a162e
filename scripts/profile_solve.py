"""In-solve kernel times (rdr_profile_solve: eager PCG with CUDA events between
the kernel groups of each iteration) next to the standalone ones
(rdr_time_kernels), per config.

    python scripts/profile_solve.py 3 2 4 5:10 7:10
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402


def main():
    for spec in sys.argv[1:]:
        cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
        c = make_config(cfg, p=p) if p else make_config(cfg)
        S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
        b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
        S.solve(b)
        it, ms = S.profile_solve(b)
        alone = S.time_kernels(b, b, reps=10)
        info = S.info
        print(json.dumps({"cfg": cfg, "p": c.p, "iters": it,
                          "in_solve_ms": dict(zip(("apply", "update_jacobi", "patches"), ms.tolist()[:3])),
                          "standalone_ms": dict(zip(("apply", "jacobi", "patches", "pcg_apply"), alone.tolist())),
                          "apply_tflops_in_solve": info["flops_apply"] / ms[0] / 1e9,
                          "apply_tflops_standalone": info["flops_apply"] / alone[0] / 1e9,
                          "apply_layout": {k: info[k] for k in ("apply_variant", "apply_slots", "apply_grid")},
                          "small_patch_grid": info["small_patch_grid"]}),
              flush=True)
        S.close()


if __name__ == "__main__":
    main()
