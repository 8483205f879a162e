"""Debug aid: for bad fused-apply launches, map the deviating dofs to (cell tile, column group)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
from oracle.mesh import Topology, number, dof_layout
cfg, p, n = 3, 10, 12
c = make_config(cfg, p=p, n=n)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
topo = Topology(c.vertices, c.tets, c.mask)
num = number("hgrad", p, topo, dof_layout("hgrad", p))
dm = num.dofmap
rdr._lib.rdr_debug_fused_apply.argtypes = [ctypes.c_void_p] * 4
z = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
free = (S.apply(torch.ones_like(z)) != 0)
z = z * free
ref = S.apply(z).cpu().numpy()
BM = 32
for t in range(16):
    q = torch.zeros_like(z)
    rdr._lib.rdr_debug_fused_apply(S._h, ctypes.c_void_p(z.data_ptr()), ctypes.c_void_p(q.data_ptr()),
                                   ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    qf = q.cpu().numpy()
    bad = np.nonzero(np.abs(qf - ref) > 1e-11 * np.abs(ref).max())[0]
    if len(bad) == 0:
        print("trial", t, "ok"); continue
    hit = np.isin(dm, bad)
    cells, locs = np.nonzero(hit)
    tiles = sorted(set((int(cc) // BM, int(l) // 32) for cc, l in zip(cells, locs)))
    print("trial", t, "bad dofs", len(bad), "candidate (tile, colgroup) pairs", len(tiles), tiles[:12], flush=True)
    # which (tile, group) explains all bad dofs: count coverage
    from collections import Counter
    cnt = Counter((int(cc) // BM, int(l) // 32) for cc, l in zip(cells, locs))
    (tile, grp), _ = cnt.most_common(1)[0]
    # which (local cell, local column) outputs explain the bad dofs: a dof is bad iff
    # some (cell, col) in the CTA's block maps to it with a wrong contribution
    lc = sorted(set(int(cc) - tile * BM for cc, l in zip(cells, locs) if int(cc) // BM == tile and int(l) // 32 == grp))
    cols = sorted(set(int(l) - grp * 32 for cc, l in zip(cells, locs) if int(cc) // BM == tile and int(l) // 32 == grp))
    print("  tile", tile, "group", grp, "local cells", lc, "local cols", cols[:40], "dev max", np.abs(qf - ref)[bad].max(), flush=True)
