import importlib.util, json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from rdr_inputs import make_config
def load(path, name):
    spec = importlib.util.spec_from_file_location(name, path)
    m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); return m
old = load("abtmp/old_r1/rdr.py", "rdr_old")
from paper_2506_17406_b200 import rdr as new
def per_iter(S, b, solves=5):
    S.solve(b); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = 0; e0.record()
    for _ in range(solves): its += S.solve(b)[1]
    e1.record(); e1.synchronize()
    return round(e0.elapsed_time(e1) / its * 1e3, 2)
for spec in sys.argv[1:]:
    cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
    c = make_config(cfg, p=p) if p else make_config(cfg)
    out = {"cfg": cfg, "p": c.p}
    for name, mod, kw in (("old", old, {}), ("new_graph", new, {"loop": new.LOOP_GRAPH}), ("new", new, {})):
        S = mod.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, **kw)
        b = torch.from_numpy(make_config(cfg, p=p).draw_vector(S.n_total) if p else make_config(cfg).draw_vector(S.n_total)).cuda()
        ms = S.time_kernels(b, b, reps=20)
        out[name] = {"us_iter": per_iter(S, b), "apply_us": round(1e3 * ms[0], 2), "jac_us": round(1e3 * ms[1], 2), "patch_us": round(1e3 * ms[2], 2)}
        S.close()
    print(json.dumps(out), flush=True)
