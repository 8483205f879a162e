"""Debug aid: true relative residual ||b - A x|| / ||b|| of rdr_solve (device apply)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg = int(sys.argv[1]); p = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else None
n = int(sys.argv[3]) if len(sys.argv) > 3 else None
c = make_config(cfg, p=p, n=n)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
mask = torch.from_numpy(~(S.apply(torch.ones_like(b)).cpu().numpy() == 0)).cuda()  # free dofs (nonzero rows)
bm = b * mask
x, it = S.solve(b)
r = bm - S.apply(x)
z0 = S.precond(bm)
z = S.precond(r)
print(os.environ.get("TAG", ""), "cfg", cfg, "iters", it, "true rel res %.3e" % (r.norm() / bm.norm()).item(),
      "precond rel res %.3e" % (z.norm() / z0.norm()).item(), flush=True)
