"""Setup's apply-layout choice on repeated setups of the same config (is the
autotuner stable?), with the setup time.

    python scripts/experiments/tuner_stability.py 3 3 3 2 2 4 4 8:9 8:9 7:5
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

for spec in sys.argv[1:]:
    cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
    c = make_config(cfg, p=p) if p else make_config(cfg)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    i = S.info
    import torch
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    S.solve(b)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    its = sum(S.solve(b)[1] for _ in range(3))
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"cfg": cfg, "p": c.p, "apply_factored": i["apply_factored"],
                      "split": (i["apply_fact_split_a"], i["apply_fact_split_b"]),
                      "ms_per_iter": round(e0.elapsed_time(e1) / its, 4), "apply_variant": i["apply_variant"], "apply_slots": i["apply_slots"],
                      "apply_grid": i["apply_grid"], "setup_s": i["setup_seconds"]}), flush=True)
    S.close()
