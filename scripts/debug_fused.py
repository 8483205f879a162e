"""Debug aid: x after k PCG iterations (maxit=k, rtol=0) -> npy, to compare fused/unfused paths."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg, p, n, tag = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
c = make_config(cfg, p=p, n=n)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
out = {}
for k in (1, 2, 3, 5):
    x, it = S.solve(b, rtol=0.0, maxit=k)
    out[f"x{k}"] = x.cpu().numpy()
np.savez(f"gpurun_out/fused_{tag}.npz", **out)
print(tag, "done", flush=True)
