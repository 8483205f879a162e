"""Per-config measurements beside bench.py's single line (BASELINE.json
configs 1-5; config 5 is the p-sweep p = 1..12): setup time, device time per
A·x / per preconditioner apply / per PCG iteration, iteration count and
time-to-solution at rtol 1e-8, each against its roofline (apply vs the
measured DMMA peak, patches vs the measured HBM copy peak).

    python scripts/sweep.py [--configs 1,2,4,3] [--p 1-12] [--out profiles/r1_sweep.jsonl]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402


def measure(cfg, p, fp64_peak, hbm, solves=3, reps=20, dec="split", pre="additive"):
    c = make_config(cfg, p=p) if cfg in (5, 7, 8) else make_config(cfg)
    t0 = time.time()
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask,
                   decomposition=rdr.UNSPLIT if dec == "unsplit" else rdr.SPLIT,
                   preconditioner=rdr.HYBRID if pre == "hybrid" else rdr.ADDITIVE)
    setup_wall = time.time() - t0
    info = S.info
    n = S.n_total
    b = torch.from_numpy(c.draw_vector(n)).cuda()
    x = torch.empty_like(b)
    kms = S.time_kernels(b, b, reps=reps)
    S.solve(b, x)  # warm-up (graph instantiation)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times, its = [], []
    for _ in range(solves):
        ev0.record()
        _, it = S.solve(b, x)
        ev1.record()
        ev1.synchronize()
        times.append(ev0.elapsed_time(ev1))
        its.append(it)
    t_solve = float(np.median(times))
    it = its[0]
    patch_bytes = info["bytes_precond"] - 24.0 * info["n_interior"]
    out = {
        "config": cfg, "decomposition": dec, "preconditioner": pre, "space": ("hgrad", "hcurl", "hdiv")[c.space],
        "p": c.p,
        "n_cells": info["n_cells"],
        "n_loc": info["n_loc"], "n_total": n, "n_free": info["n_free"], "n_patches": info["n_patches"],
        "max_patch": info["max_patch"], "patch_GB": info["patch_bytes"] / 1e9, "setup_s": info["setup_seconds"],
        "setup_wall_s": setup_wall,
        "apply_ms": kms[0], "apply_dofs_per_s": info["n_free"] / (kms[0] / 1e3),
        "apply_tflops": info["flops_apply"] / (kms[0] / 1e3) / 1e12,
        "apply_frac_dmma": info["flops_apply"] / (kms[0] / 1e3) / 1e12 / fp64_peak,
        "jacobi_ms": kms[1], "patch_ms": kms[2], "pcg_apply_ms": kms[3],
        "pcg_apply_frac_dmma": info["flops_apply"] / (kms[3] / 1e3) / 1e12 / fp64_peak if kms[3] > 0 else None,
        "precond_ms": kms[1] + kms[2],
        "patch_GBps": patch_bytes / (kms[2] / 1e3) / 1e9 if kms[2] > 0 else None,
        "patch_frac_hbm": patch_bytes / (kms[2] / 1e3) / 1e9 / hbm if kms[2] > 0 else None,
        "pcg_iters": it, "time_to_solution_ms": t_solve, "ms_per_iter": t_solve / max(1, it),
        "pcg_iters_per_s": it / (t_solve / 1e3),
        "t_roof_iter_ms": info["flops_apply"] / fp64_peak / 1e9 + (patch_bytes + 12 * 8 * n) / hbm / 1e6,
    }
    out["iter_frac_roofline"] = out["t_roof_iter_ms"] / out["ms_per_iter"]
    out["apply_layout"] = {k: info[k] for k in ("apply_variant", "apply_slots", "apply_grid")}
    out["persistent_loop"] = info["persistent_loop"]
    if pre == "additive":  # in-solve kernel times (eager solve, events between kernel groups)
        _, pms = S.profile_solve(b)
        out["in_solve_ms"] = {"apply": pms[0], "update_jacobi": pms[1], "patches": pms[2]}
    if pre == "hybrid":
        out["rho"] = [float(v) for v in S.weights]
        t0 = time.time()
        ev0.record()
        for _ in range(5):
            S.precond(b, x)
        ev1.record()
        ev1.synchronize()
        out["hybrid_precond_ms"] = ev0.elapsed_time(ev1) / 5
        out.pop("t_roof_iter_ms")
        out.pop("iter_frac_roofline")
    S.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,4,5,3")
    ap.add_argument("--p", default="1-12")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep.jsonl"))
    ap.add_argument("--decomposition", default="split", choices=["split", "unsplit"])
    ap.add_argument("--precond", default="additive", choices=["additive", "hybrid"])
    args = ap.parse_args()
    lo, hi = (int(v) for v in args.p.split("-"))
    fp64_peak = rdr.measure_fp64_peak()
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    head = {"fp64_dmma_peak_tflops": fp64_peak, "hbm_peak_gbs": hbm, "gpu": torch.cuda.get_device_name(0)}
    print(json.dumps(head), flush=True)
    with open(args.out, "w") as f:
        f.write(json.dumps(head) + "\n")
        for cfg in (int(v) for v in args.configs.split(",")):
            for p in (range(lo, min(hi, 12 if cfg == 5 else 10) + 1) if cfg in (5, 7, 8) else [None]):
                r = measure(cfg, p, fp64_peak, hbm, dec=args.decomposition, pre=args.precond)
                print(json.dumps(r), flush=True)
                f.write(json.dumps(r) + "\n")
                f.flush()
                torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
