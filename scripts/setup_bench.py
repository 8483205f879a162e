"""Time-to-first-solve: rdr_setup wall time with the patch
inverses built on the host cores vs on the GPU (patch_setup.cu), split into
reference element / patch phases, plus the patch-kernel rate.

    python scripts/setup_bench.py [--configs 2,4,5:10,5:12,3] [--out profiles/setup.jsonl]
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


def one(spec, setup, dec):
    cfg, _, p = spec.partition(":")
    c = make_config(int(cfg), p=int(p)) if p else make_config(int(cfg))
    t0 = time.time()
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask, setup=setup,
                   decomposition=rdr.UNSPLIT if dec == "unsplit" else rdr.SPLIT)
    wall = time.time() - t0
    info = S.info
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    x = torch.empty_like(b)
    t1 = time.time()
    _, it = S.solve(b, x)
    first_solve = time.time() - t1
    z = S.precond(b).cpu().numpy()
    S.close()
    # n_m^3 per patch: the work of one inversion (host: ~n^3 flop Cholesky-based; device: ld^3 fma sweep)
    return {"config": spec, "decomposition": dec, "setup": "host" if setup else "device", "p": c.p,
            "space": ("hgrad", "hcurl", "hdiv")[c.space], "n_patches": info["n_patches"],
            "max_patch": info["max_patch"], "patch_GB": info["patch_bytes"] / 1e9, "setup_wall_s": wall,
            "setup_s": info["setup_seconds"], "refelem_s": info["refelem_seconds"],
            "patch_setup_s": info["patch_setup_seconds"], "patch_kernel_s": info["patch_kernel_seconds"],
            "sweep_tflops": info["patch_setup_flops"] / info["patch_kernel_seconds"] / 1e12
            if info["patch_kernel_seconds"] else None,
            "first_solve_s": first_solve, "iters": it,
            "z_norm": float(np.linalg.norm(z))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,4,5:10,5:12,3")
    ap.add_argument("--decomposition", default="split", choices=["split", "unsplit"])
    ap.add_argument("--host", default="1", help="also time the host setup (0: device only)")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "setup.jsonl"))
    args = ap.parse_args()
    head = {"gpu": torch.cuda.get_device_name(0), "host_threads": os.cpu_count()}
    print(json.dumps(head), flush=True)
    with open(args.out, "w") as f:
        f.write(json.dumps(head) + "\n")
        for spec in args.configs.split(","):
            rows = [one(spec, rdr.SETUP_DEVICE, args.decomposition)]
            if args.host == "1":
                rows.append(one(spec, rdr.SETUP_HOST, args.decomposition))
                rows[0]["z_rel_vs_host"] = abs(rows[0]["z_norm"] - rows[1]["z_norm"]) / rows[1]["z_norm"]
                rows[0]["patch_speedup_vs_host"] = rows[1]["patch_setup_s"] / rows[0]["patch_setup_s"]
            for r in rows:
                print(json.dumps(r), flush=True)
                f.write(json.dumps(r) + "\n")
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
