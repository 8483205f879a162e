import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
cfg, p, n = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
c = make_config(cfg, p=p, n=n)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
rdr._lib.rdr_debug_fused_apply.argtypes = [ctypes.c_void_p] * 4
z = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
free = (S.apply(torch.ones_like(z)) != 0)
z = z * free
q_ref = S.apply(z).cpu().numpy()
for trial in range(3):
    q = torch.zeros_like(z)
    assert rdr._lib.rdr_debug_fused_apply(S._h, ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(q.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
    qf = q.cpu().numpy()
    d = np.abs(qf - q_ref)
    bad = np.nonzero(d > 1e-10 * np.abs(q_ref).max())[0]
    print("trial", trial, "rel", np.linalg.norm(qf - q_ref) / np.linalg.norm(q_ref), "bad dofs", len(bad), flush=True)
    if len(bad):
        dm = None
        print("  first bad", bad[:10], "ratio", (qf[bad[:5]] / q_ref[bad[:5]]))
