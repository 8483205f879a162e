"""Tiny GPU parity probe (debugging aid): one small config through the C ABI vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
from oracle.solver import Oracle
space = int(sys.argv[1]) if len(sys.argv) > 1 else 0
p = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = int(sys.argv[3]) if len(sys.argv) > 3 else 2
c = make_config(0, n=n, p=p, space=space, perturb=True, bc="all")
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
x = c.draw_vector(O.n_total)
y = S.apply(torch.from_numpy(x).cuda()).cpu().numpy()
ya = O.apply(x)
print("apply rel", np.linalg.norm(y - ya) / np.linalg.norm(ya), flush=True)
z = S.precond(torch.from_numpy(x).cuda()).cpu().numpy()
za = O.precond(x)
print("precond rel", np.linalg.norm(z - za) / np.linalg.norm(za), flush=True)
xs, it = S.solve(torch.from_numpy(x).cuda())
xo, ito, _ = O.solve(x)
print("iters", it, ito, "x rel", np.linalg.norm(xs.cpu().numpy() - xo) / np.linalg.norm(xo))
