"""Markdown table of a sweep JSONL (scripts/sweep.py) for DESIGN.md §7.
    python scripts/design_table.py profiles/round2/sweep_split.jsonl"""
import json
import sys

print("| cfg | space, p | n_loc | N_free | setup s | A·x ms (plain / PCG mode) | PCG-mode A·x TFLOP/s (frac DMMA) | "
      "patches ms | patch GB/s (frac HBM) | PCG iters | time to solution ms | ms/iter | frac of T_roof |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    d = json.loads(line)
    if "config" not in d:
        continue
    pa = d.get("pcg_apply_ms") or d["apply_ms"]
    tf = d["apply_tflops"] * d["apply_ms"] / pa
    fr = d.get("pcg_apply_frac_dmma") or d["apply_frac_dmma"]
    pg = f"{d['patch_GBps']:.0f} ({d['patch_frac_hbm']:.2f})" if d.get("patch_GBps") else "-"
    loop = " (persistent)" if d.get("persistent_loop") else ""
    print(f"| {d['config']} | {d['space']} {d['p']} | {d['n_loc']} | {d['n_free']} | {d['setup_s']:.2f} | "
          f"{d['apply_ms']:.4f} / {pa:.4f} | {tf:.1f} ({fr:.2f}) | {d['patch_ms']:.4f} | {pg} | {d['pcg_iters']} | "
          f"{d['time_to_solution_ms']:.2f} | {d['ms_per_iter']:.4f}{loop} | {d.get('iter_frac_roofline', 0):.2f} |")
