"""One short solve of a config (for an ncu launch list of its PCG kernels):
    RDR_PCG_HOSTLOOP=1 ncu --graph-profiling node --metrics gpu__time_duration.sum ... \\
        python scripts/solve_launches.py CONFIG [P] [MAXIT]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

cfg = int(sys.argv[1])
p = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else 16
c = make_config(cfg, p=p) if p else make_config(cfg)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
x = torch.empty_like(b)
try:
    S.solve(b, x, maxit=maxit)
except rdr.RdrError:
    pass  # ENOCONV at maxit is expected
torch.cuda.synchronize()
print("done", S.info["n_total"])
