import os, sys, time, torch, numpy as np
sys.path.insert(0, '.')
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg = int(sys.argv[1]); p = int(sys.argv[2]) if len(sys.argv) > 2 else None
c = make_config(cfg, p=p) if p else make_config(cfg)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, loop=rdr.LOOP_OVERLAP)
print("overlap_sms", S.info["overlap_sms"], flush=True)
b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
for _ in range(2):
    torch.cuda.synchronize(); t = time.time(); x, it = S.solve(b); torch.cuda.synchronize()
    print("iters", it, "ms/iter", (time.time() - t) * 1e3 / it, flush=True)
