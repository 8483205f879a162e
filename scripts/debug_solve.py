"""Debug aid: repeated entry points on one config, each synchronised."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg = int(sys.argv[1]); mode = sys.argv[2]
c = make_config(cfg)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
x = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
if mode == "precond":
    for k in range(30):
        z = S.precond(x); torch.cuda.synchronize()
    print("precond x30 ok", flush=True)
else:
    for m in [1, 2, 3, 9, 20, 1000]:
        xs, it = S.solve(x, maxit=m); torch.cuda.synchronize(); print("solve maxit", m, "iters", it, flush=True)
