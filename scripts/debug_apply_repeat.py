"""Debug aid: repeat rdr_apply (and the fused PCG apply) and count launches whose
result deviates from the first beyond rounding (atomics reorder at ~1e-16)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg, p, n, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
c = make_config(cfg, p=p, n=n)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
rdr._lib.rdr_debug_fused_apply.argtypes = [ctypes.c_void_p] * 4
z = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
free = (S.apply(torch.ones_like(z)) != 0)
z = z * free
ref = S.apply(z).clone()
bad_std = bad_fused = 0
for t in range(reps):
    y = S.apply(z)
    if ((y - ref).norm() / ref.norm()).item() > 1e-13:
        bad_std += 1
    q = torch.zeros_like(z)
    rdr._lib.rdr_debug_fused_apply(S._h, ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(q.data_ptr()),
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    if ((q - ref).norm() / ref.norm()).item() > 1e-13:
        bad_fused += 1
print(os.environ.get("TAG", ""), f"cfg{cfg} p={p} n={n}: bad standard {bad_std}/{reps}, bad fused {bad_fused}/{reps}", flush=True)
