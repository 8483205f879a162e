"""Write tests/golden/oracle_pcg_iters.json: the CPU oracle's PCG iteration
counts (R-A16, rtol 1e-8, x0 = 0) on the BASELINE.json configurations with
their seeded rhs (the first vector drawn after the config).

Calls only oracle/ and rdr_inputs/ (no CUDA path): these are the expected
values of the +-1 iteration-count parity tests at sizes too large to run the
oracle inside the GPU test session.

    python scripts/oracle_golden.py 5:1-8 4 5:9-12 [3] [6]   (6: the H(div) NEXT-2 workload)
    python scripts/oracle_golden.py --lean 3 7:9-10 8:9-10     (oracle/lean.py: element-by-element
                                                              operator, packed Cholesky factors)
    python scripts/oracle_golden.py --hybrid 2 5:4-6           (oracle/hybrid.py: the paper's hybrid Schwarz with
                                                              the Whitney coarse space; entries "hybrid_entries")
"""
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from rdr_inputs import make_config  # noqa: E402
from oracle.solver import Oracle  # noqa: E402
from oracle.lean import LeanOracle  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_pcg_iters.json")


def run(cfg, p, lean=False):
    t0 = time.time()
    c = make_config(cfg, p=p) if p is not None else make_config(cfg)
    if lean:
        store = os.path.join(ROOT, ".lean_store")
        os.makedirs(store, exist_ok=True)
        O = LeanOracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, store_dir=store,
                       workers=os.cpu_count(), verbose=True)
    else:
        O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    O.build_preconditioner(kappa=False)
    b = c.draw_vector(O.n_total)
    hist = []
    x, it, res = O.solve(b, rtol=1e-8, history=hist)
    return {"cfg": cfg, "p": c.p, "space": ("hgrad", "hcurl", "hdiv")[c.space], "n_total": int(O.n_total),
            "n_free": int(O.free.sum()), "iters": int(it), "true_rel_res": float(res),
            "z_ratio_tail": [float(h) for h in hist[-3:]],
            "oracle_seconds": round(time.time() - t0, 1), "oracle": "lean" if lean else "global"}


def run_hybrid(cfg, p):
    from oracle.hybrid import HybridOracle
    t0 = time.time()
    c = make_config(cfg, p=p) if p is not None else make_config(cfg)
    O = HybridOracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    b = c.draw_vector(O.n_total)
    hist = []
    x, it, res = O.solve(b, rtol=1e-8, history=hist)
    return {"cfg": cfg, "p": c.p, "space": ("hgrad", "hcurl", "hdiv")[c.space], "n_total": int(O.n_total),
            "n_free": int(O.free.sum()), "iters": int(it), "true_rel_res": float(res),
            "rho": [float(v) for v in O.rho], "z_ratio_tail": [float(h) for h in hist[-3:]],
            "oracle_seconds": round(time.time() - t0, 1), "oracle": "hybrid"}


def main():
    data = json.load(open(OUT)) if os.path.exists(OUT) else {"note": "", "entries": []}
    data["note"] = ("Oracle PCG iteration counts (oracle/solver.py, R-A16, rtol 1e-8) on BASELINE.json configs "
                    "with the seeded rhs; written by scripts/oracle_golden.py (oracle/ only). "
                    "hybrid_entries: the same with oracle/hybrid.py (hybrid Schwarz with the Whitney coarse "
                    "space, P:2399-2455), with its weights rho_m.")
    lean = "--lean" in sys.argv
    hybrid = "--hybrid" in sys.argv
    key = "hybrid_entries" if hybrid else "entries"
    data.setdefault(key, [])
    for spec in [a for a in sys.argv[1:] if a not in ("--lean", "--hybrid")]:
        if ":" in spec:
            cfg, rng = spec.split(":")
            lo, hi = (int(v) for v in rng.split("-")) if "-" in rng else (int(rng), int(rng))
            jobs = [(int(cfg), p) for p in range(lo, hi + 1)]
        else:
            jobs = [(int(spec), None)]
        for cfg, p in jobs:
            e = run_hybrid(cfg, p) if hybrid else run(cfg, p, lean)
            e["host"] = f"{platform.node()} ({os.cpu_count()} cpus)"
            data[key] = [x for x in data[key] if not (x["cfg"] == e["cfg"] and x["p"] == e["p"])]
            data[key].append(e)
            data[key].sort(key=lambda x: (x["cfg"], x["p"]))
            json.dump(data, open(OUT, "w"), indent=1)
            print(json.dumps(e), flush=True)


if __name__ == "__main__":
    main()
