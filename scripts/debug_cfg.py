"""Debug aid: one config through the C ABI, each entry point synchronised."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
p = int(sys.argv[2]) if len(sys.argv) > 2 else 6
c = make_config(cfg, p=p) if cfg == 5 else make_config(cfg)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
print(S.info, flush=True)
x = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
y = S.apply(x); torch.cuda.synchronize(); print("apply ok", float(y.norm()), flush=True)
z = S.precond(x); torch.cuda.synchronize(); print("precond ok", float(z.norm()), flush=True)
xs, it = S.solve(x); print("solve ok", it, flush=True)
print(S.time_kernels(x, x, reps=5), flush=True)
