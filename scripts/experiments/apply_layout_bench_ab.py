"""Config-3 solve throughput per apply warp layout in the power-capped steady
state (20 timed solves each, SM clock and power sampled by NVML), the layout
forced with rdr_debug_set_apply_variant: does a layout with more cells per
tile (fewer reference-stack bytes from L2 per apply) win under the power cap
although setup's standalone timing prefers another?

    python scripts/experiments/apply_layout_bench_ab.py 6 2 8 0 10
"""
import json
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from rdr_inputs import make_config  # noqa: E402
from paper_2506_17406_b200 import rdr  # noqa: E402


def sampler(stop, out):
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    while not stop.is_set():
        out.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.01)


def main():
    c = make_config(3)
    S = rdr.Solver(c.vertices, c.tets, c.p, c.space, c.alpha, c.beta, c.mask)
    b = torch.from_numpy(c.draw_vector(S.n_total)).cuda()
    print(json.dumps({"tuned_variant": S.info["apply_variant"], "slots": S.info["apply_slots"]}), flush=True)
    for rep in range(2):
        for v in [int(a) for a in sys.argv[1:]]:
            if not S.set_apply_variant(v):
                print(json.dumps({"variant": v, "skipped": True}), flush=True)
                continue
            for _ in range(3):
                S.solve(b)
            torch.cuda.synchronize()
            stop, samples = threading.Event(), []
            th = threading.Thread(target=sampler, args=(stop, samples))
            th.start()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            its = 0
            e0.record()
            for _ in range(20):
                _, it = S.solve(b)
                its += it
            e1.record()
            torch.cuda.synchronize()
            stop.set()
            th.join()
            ms = e0.elapsed_time(e1)
            sm = sorted(s[0] for s in samples)
            pw = sorted(s[1] for s in samples)
            k = S.time_kernels(b, b, reps=5)
            print(json.dumps({"rep": rep, "variant": v, "slots": S.info["apply_slots"], "it_per_s": its / ms * 1e3,
                              "ms_per_iter": ms / its, "sm_mhz_median": sm[len(sm) // 2],
                              "power_w_median": pw[len(pw) // 2], "apply_ms_standalone": k[0],
                              "pcg_apply_ms_standalone": k[3]}), flush=True)


if __name__ == "__main__":
    main()
