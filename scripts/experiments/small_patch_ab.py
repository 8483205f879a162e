import sys, torch, json
sys.path.insert(0, '.')
from rdr_inputs import make_config
from paper_2506_17406_b200 import rdr
for spec in sys.argv[1:]:
    cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
    c = make_config(cfg, p=p) if p else make_config(cfg)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    out = {"cfg": cfg, "p": c.p, "chosen": S.info["small_patch_grid"]}
    for pers in (0, 1, 0, 1):
        if not S.set_small_patch_kernel(pers): out["n/a"] = True; break
        ms = S.time_kernels(b, b, reps=20)
        it, pm = S.profile_solve(b)
        out.setdefault(f"p{pers}", []).append((round(ms[2], 4), round(pm[2], 4)))
    print(json.dumps(out), flush=True)
