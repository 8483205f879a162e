"""The fused PCG iteration with the direction update folded into the apply's gather
(3 kernels) against a separate direction kernel in front of the plain apply (4 kernels,
rdr_info.separate_direction): graph-solve ms per iteration, per config, with setup's choice.
Needs profiles/round2/experiments/separate_direction_kernel.diff applied (measured and not
kept: the two forms are within 1 %, separate_direction_ab.jsonl).

    python scripts/experiments/direction_ab.py 3 4 6 7:9 7:10 8:9 8:10 5:10 5:12 2
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

for spec in sys.argv[1:]:
    cfg, p = (int(v) for v in spec.split(":")) if ":" in spec else (int(spec), None)
    c = make_config(cfg, p=p) if p else make_config(cfg)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    i = S.info
    out = {"cfg": cfg, "p": c.p, "n_free": i["n_free"], "chosen_separate": i["separate_direction"],
           "apply_factored": i["apply_factored"]}
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    for sep in (0, 1, 0, 1):
        assert S.set_direction(bool(sep))
        S.solve(b)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        its = sum(S.solve(b)[1] for _ in range(3))
        e1.record()
        torch.cuda.synchronize()
        out.setdefault("separate" if sep else "fused", []).append(round(e0.elapsed_time(e1) / its, 4))
    out["iters"] = its // 3
    print(json.dumps(out), flush=True)
    S.close()
