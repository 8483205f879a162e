"""Setup's apply-layout choice on repeated setups of the same config (is the
autotuner stable?), with the setup time.

    python scripts/experiments/tuner_stability.py 3 3 3 2 2 4 4
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402

for spec in sys.argv[1:]:
    cfg = int(spec)
    c = make_config(cfg)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    i = S.info
    print(json.dumps({"cfg": cfg, "apply_variant": i["apply_variant"], "apply_slots": i["apply_slots"],
                      "apply_grid": i["apply_grid"], "setup_s": i["setup_seconds"]}), flush=True)
    S.close()
