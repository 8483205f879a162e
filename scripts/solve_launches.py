"""One short PCG solve of a config with every kernel launched eagerly
(rdr_options.loop = RDR_LOOP_EAGER), for an ncu launch list of its kernels:
    ncu --metrics gpu__time_duration.sum --clock-control none --csv ... \\
        python scripts/solve_launches.py CONFIG [P|-] [MAXIT] [--hybrid]
The solve runs inside an NVTX range "solve" (ncu --nvtx --nvtx-include solve/ leaves out
setup's launches of the same kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

hybrid = "--hybrid" in sys.argv
argv = [a for a in sys.argv if a != "--hybrid"]
cfg = int(argv[1])
p = int(argv[2]) if len(argv) > 2 and argv[2] != "-" else None
maxit = int(argv[3]) if len(argv) > 3 else 16
c = make_config(cfg, p=p) if p else make_config(cfg)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_EAGER,
               preconditioner=rdr.HYBRID if hybrid else rdr.ADDITIVE)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
x = torch.empty_like(b)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("solve")
S.solve(b, x, maxit=maxit)  # RDR_ENOCONV at maxit is reported through S.converged
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("done", S.info["n_total"], "iterations", S.last_stats())
