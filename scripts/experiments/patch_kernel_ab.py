"""Row (patch_ldg_kernel) vs column (patch_col_kernel) traversal of the
one-CTA-per-patch star solves: standalone patch time and PCG ms/iteration per
config, and what setup's timing chose.

    python scripts/patch_kernel_ab.py 2 3 4 5:10 5:12 7:10
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402


def main():
    for spec in sys.argv[1:]:
        cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
        c = make_config(cfg, p=p) if p else make_config(cfg)
        S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
        out = {"cfg": cfg, "p": c.p, "chosen": S.info["patch_kernel"], "patch_bytes": S.info["patch_bytes"]}
        b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
        for column in (False, True):
            if not S.set_patch_kernel(column):
                continue
            ms = S.time_kernels(b, b, reps=10)[2]
            S.solve(b)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            x, it = S.solve(b)
            e1.record()
            torch.cuda.synchronize()
            out["col" if column else "row"] = {"patch_ms": ms, "patch_gbs": S.info["patch_bytes"] / ms / 1e6,
                                               "iters": it, "ms_per_iter": e0.elapsed_time(e1) / it}
        print(json.dumps(out), flush=True)
        S.close()


if __name__ == "__main__":
    main()
