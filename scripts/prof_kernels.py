"""Profiling driver (for ncu: --kernel-name regex:<kernel> -s <skip> -c <n>):
set up one config, then either launch each hot-path kernel `reps` times
through rdr_time_kernels (standalone launches, `--mode kernels`), or run one
PCG solve of `reps` iterations with every kernel launched eagerly
(rdr_options.loop = RDR_LOOP_EAGER, `--mode solve`): the in-solve kernels,
i.e. the fused PCG-mode apply, the update + Jacobi and the patch solves.

    python scripts/prof_kernels.py [config] [p] [reps] [--mode kernels|solve] [--apply variant,slots,grid]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

argv = [a for i, a in enumerate(sys.argv) if not (i > 0 and sys.argv[i - 1] == "--apply")]
args = [a for a in argv[1:] if not a.startswith("--")]
mode = "solve" if "--mode" in sys.argv and sys.argv[sys.argv.index("--mode") + 1] == "solve" else "kernels"
if mode == "solve":
    args = [a for a in args if a != "solve"]
else:
    args = [a for a in args if a != "kernels"]
cfg = int(args[0]) if len(args) > 0 else 3
p = int(args[1]) if len(args) > 1 and args[1] != "-" else None
reps = int(args[2]) if len(args) > 2 else 3
c = make_config(cfg, p=p) if p else make_config(cfg)
S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask,
               loop=rdr.LOOP_EAGER if mode == "solve" else rdr.LOOP_DEVICE)
if "--apply" in sys.argv:  # reproduce another setup's layout (bench JSON problem.apply_layout)
    v, slots, grid = (int(a) for a in sys.argv[sys.argv.index("--apply") + 1].split(","))
    assert S.set_apply_config(v, slots, grid), (v, slots, grid)
x = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
if mode == "solve":
    # NVTX range: ncu selects the solve's launches only (--nvtx --nvtx-include solve/), not
    # setup's autotuning launches of the same kernels
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("solve")
    _, it = S.solve(x, maxit=reps, rtol=0.0)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    print("eager solve:", it, "iterations", S.info)
else:
    ms = S.time_kernels(x, x, reps=reps)
    print("kernel ms (apply, jacobi, patches, gradient):", ms.tolist(), S.info)
