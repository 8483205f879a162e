"""Benchmark of the B200 Riesz-map PCG hot path (arXiv 2506.17406).

Workload (BASELINE.json configs[1], "cfg2"): H(grad) Riesz map, p=6, 8x8x8 cubes
x 6 = 3072 tets with interior vertices displaced by up to 0.2h (seed 0),
per-cell alpha, beta log-uniform in [1e-2, 1e2], Dirichlet on x=0, seeded
uniform[-1,1] rhs, PCG rtol 1e-8 from x0 = 0.

A step = one full PCG solve (every hot-path row of SURVEY §8(a): operator
apply, interior Jacobi, star-patch solves, PCG vector ops) on a fresh rhs
already resident in HBM. value = PCG iterations/s over the whole job.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config 2]

Multi-GPU: the path does not shard within one solve (single-GPU north_star);
N ranks run N independent problems (replicas, weak scaling, no collective on
the data path; torch.distributed only for the barrier and the max-over-ranks
time).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 DoFs/s per A·x and PCG iters/s vs p on 1 B200; % of FP64-TC/HBM roofline"
WORKLOADS = {
    1: "cfg1: H(grad) p=3, 2^3x6 tets, alpha=beta=1, full Dirichlet",
    2: "cfg2: H(grad) p=6, 8^3x6 perturbed tets, log-uniform alpha,beta in [1e-2,1e2], Dirichlet x=0",
    3: "cfg3: H(grad) p=10, 16^3x6 perturbed tets, alpha=beta=1, full Dirichlet",
    4: "cfg4: H(curl) Ned1_6, 12^3x6 tets, alpha=beta=1, full tangential Dirichlet",
    5: "cfg5: H(grad) p-sweep point, 8^3x6 perturbed tets, alpha=beta=1, full Dirichlet",
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = f"/tmp/rdr_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [l.split(", ") for l in open(self.path).read().strip().splitlines() if l.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if len(r) > 4 + k and r[4 + k].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_sample(cfg, p, iters_per_step, steps, warmup):
    """The CPU oracle as it stands, timed on the host cores: setup untimed, then
    `steps` samples of `iters_per_step` PCG iterations (apply + precond + vector
    ops) on the same workload."""
    from rdr_inputs import make_config
    from oracle.solver import Oracle
    c = make_config(cfg, p=p) if cfg == 5 else make_config(cfg)
    O = Oracle(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    O.build_preconditioner(kappa=False)
    b = O.mask(c.draw_vector(O.n_total))
    times = []
    for k in range(warmup + steps):
        t0 = time.perf_counter()
        O.solve(b, rtol=0.0, maxit=iters_per_step)
        dt = time.perf_counter() - t0
        if k >= warmup:
            times.append(dt)
    cores = len(os.sched_getaffinity(0))
    return iters_per_step * steps / sum(times), sum(times), cores, O.n_total


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    ips, tot, cores, n_total = oracle_sample(args.config, args.p, args.ref_iters, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": ips, "unit": "PCG iters/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "rtol": 1e-8},
        "cpu_baseline": {"value": ips, "unit": "PCG iters/s", "cores": cores, "kind": "oracle",
                         "sample": f"{args.ref_iters} oracle PCG iterations per step (scipy CSR apply + "
                                   f"cho_solve patches), setup untimed"},
        "e2e": {"value": ips, "unit": "PCG iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run(args):
    import torch
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from rdr_inputs import make_config
    from paper_2506_17406_b200 import rdr

    cfg = args.config
    c = make_config(cfg, p=args.p) if cfg == 5 else make_config(cfg, seed=rank)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    info = S.info
    n = S.n_total
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    rhs = [torch.from_numpy(c.draw_vector(n)).to(dev) for _ in range(args.steps + args.warmup)]
    x = torch.empty(n, dtype=torch.float64, device=dev)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    iters = []
    for k in range(args.warmup):
        _, it = S.solve(rhs[k], x, rtol=1e-8)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for k in range(args.steps):
            _, it = S.solve(rhs[args.warmup + k], x, rtol=1e-8)
            iters.append(it)
            launches += S.last_launches()
        ev1.record(stream)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    barrier()
    tot_iters = float(sum(iters))
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        it_t = torch.tensor([tot_iters], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(it_t)
        tot_iters = float(it_t.item())
    value = tot_iters / (ms / 1e3)

    # ---- end to end: host (pinned) b -> device -> PCG -> host x, per step
    bh = torch.from_numpy(c.draw_vector(n)).pin_memory()
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    S.solve_host(bh, xh)  # warm
    barrier()
    e_iters = 0
    ev0.record(stream)
    for k in range(args.steps):
        e_iters += S.solve_host(bh, xh)
    ev1.record(stream)
    ev1.synchronize()
    e_ms = ev0.elapsed_time(ev1)
    if ws > 1:
        t = torch.tensor([e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e_ms = float(t.item())
        t = torch.tensor([float(e_iters)], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t)
        e_iters = float(t.item())

    # ---- per-kernel device times (roofline of the dominant kernel)
    kms = S.time_kernels(rhs[0], rhs[0], reps=args.kernel_reps)
    hbm, peak_kind = _peaks()
    patch_alg = info["bytes_precond"] - 24.0 * info["n_interior"]
    it_ms = ms / max(1.0, sum(iters))
    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return
    result = None
    fp64 = None
    if not args.no_dgemm:
        a = torch.randn(4096, 4096, dtype=torch.float64, device=dev)
        for _ in range(2):
            a @ a
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            a @ a
        e1.record()
        e1.synchronize()
        fp64 = 5 * 2 * 4096 ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
    apply_flops = info["flops_apply"] / (kms[0] / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "PCG iters/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[cfg] + (f" (p={c.p})" if cfg == 5 else ""),
                   "n_free": info["n_free"], "n_total": n, "n_cells": info["n_cells"], "n_loc": info["n_loc"],
                   "n_patches": info["n_patches"], "max_patch": info["max_patch"], "rtol": 1e-8,
                   "parallelism": f"replicas x{ws}",
                   "l2": f"inputs larger than L2: {info['patch_bytes'] / 1e9:.2f} GB of patch inverses streamed "
                         f"every iteration (> 126 MB L2)"},
        "iters_per_solve": float(np.mean(iters)), "ms_per_iter": it_ms,
        "apply": {"dofs_per_s": info["n_free"] / (kms[0] / 1e3), "ms": kms[0], "tflops": apply_flops,
                  "fp64_dgemm_tflops_measured": fp64,
                  "frac_of_dgemm": (apply_flops / fp64) if fp64 else None},
        "kernel_ms": {"apply": kms[0], "jacobi": kms[1], "patches": kms[2], "gradient": kms[3]},
        "roofline": {"bound": "hbm", "kernel": "patch_kernel (star-patch solves, packed FP64 inverses)",
                     "achieved": patch_alg / (kms[2] / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
                     "frac": patch_alg / (kms[2] / 1e3) / 1e9 / hbm, "peak_source": peak_kind,
                     "alg_bytes_per_launch": patch_alg, "stored_bytes_per_launch": info["patch_bytes"],
                     "traffic": None},
        "e2e": {"value": e_iters / (e_ms / 1e3), "unit": "PCG iters/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "setup_s": info["setup_seconds"],
    }
    if not args.no_cpu:
        ips, tot, cores, _ = oracle_sample(cfg, c.p, args.ref_iters, 1, 0)
        line["cpu_baseline"] = {"value": ips, "unit": "PCG iters/s", "cores": cores, "kind": "oracle",
                                "sample": f"{args.ref_iters} oracle PCG iterations on the same workload "
                                          f"(scipy CSR apply + cho_solve patches), setup untimed"}
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--p", type=int, default=6, help="degree for the config-5 sweep point")
    ap.add_argument("--ref-iters", type=int, default=20)
    ap.add_argument("--kernel-reps", type=int, default=50)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dgemm", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run(args)


if __name__ == "__main__":
    main()
