"""Profiling driver: set up one config and launch each hot-path kernel a few
times through rdr_time_kernels (for ncu: --kernel-name regex:<kernel> -c 1).

    python scripts/prof_kernels.py [config] [p] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = int(sys.argv[2]) if len(sys.argv) > 2 else 6
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
c = make_config(cfg, p=p) if cfg == 5 else make_config(cfg)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
x = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
ms = S.time_kernels(x, x, reps=reps)
print("kernel ms (apply, jacobi, patches, gradient):", ms.tolist(), S.info)
