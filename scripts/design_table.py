"""Markdown table of a sweep JSONL (scripts/sweep.py) for DESIGN.md §7.
    python scripts/design_table.py profiles/r2k_sweep_split.jsonl"""
import json
import sys

print("| cfg | space, p | n_loc | N_free | setup s | A·x ms | A·x TFLOP/s (frac DMMA) | patches ms | "
      "patch GB/s (frac HBM) | PCG iters | time to solution ms | ms/iter | frac of T_roof |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    d = json.loads(line)
    if "config" not in d:
        continue
    print(f"| {d['config']} | {d['space']} {d['p']} | {d['n_loc']} | {d['n_free']} | {d['setup_s']:.2f} | "
          f"{d['apply_ms']:.4f} | {d['apply_tflops']:.1f} ({d['apply_frac_dmma']:.2f}) | {d['patch_ms']:.4f} | "
          f"{d['patch_GBps']:.0f} ({d['patch_frac_hbm']:.2f}) | {d['pcg_iters']} | {d['time_to_solution_ms']:.2f} | "
          f"{d['ms_per_iter']:.4f} | {d.get('iter_frac_roofline', 0):.2f} |")
