"""Summarise ncu outputs brought back in gpurun_out/ into profiles/ (tracked).

    python scripts/ncu_summary.py launches gpurun_out/launches_r1.csv > profiles/r1_launches.txt
    python scripts/ncu_summary.py full gpurun_out/prof_patch_r1.ncu-rep > profiles/r1_patch_kernel.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_dmma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
        "dram__cycles_elapsed.avg.per_second", "smsp__average_warp_latency_issue_stalled"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = collections.defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].split("<")[0].split("::")[-1]
                unit = d.get("Metric Unit", "ns")
                v = float(d["Metric Value"].replace(",", ""))
                v *= {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1e-3)
                data[name].append(v)
    tot = sum(sum(v) for v in data.values())
    print(f"# ncu launch list {path} (cold-cache, serialised: compare shares, not absolutes)")
    print(f"{'kernel':28s} {'launches':>8s} {'mean_us':>9s} {'share':>7s}")
    for k, v in sorted(data.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:28s} {len(v):8d} {sum(v) / len(v):9.2f} {100 * sum(v) / tot:6.1f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# ncu --set full summary of {path}")
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(f"## {name[:120]}")
        for i, k in enumerate(h):
            if any(k.startswith(w) for w in KEYS):
                print(f"{k:75s} {r[i]:>16s} {units[i]}")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((k[len("smsp__pcsamp_warps_issue_stalled_"):], float(r[i].replace(",", ""))))
                except ValueError:
                    pass
        tot = sum(v for _, v in stalls)
        if tot > 0:
            top = sorted(stalls, key=lambda kv: -kv[1])[:8]
            print("warp stall samples (share): " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))


def traffic(path, key, out="profiles/traffic.json"):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of each kernel in
    an `ncu --set full` report -> profiles/traffic.json[key][kernel] (read by
    bench.py's roofline.traffic)."""
    import json
    import os
    res = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(res)))
    h, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    agg = collections.defaultdict(list)
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].split("<")[0].split("::")[-1]
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = h.index(m)
            tot += float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
        agg[name].append(tot)
    data = json.load(open(out)) if os.path.exists(out) else {}
    data.setdefault(key, {})
    for name, v in agg.items():
        data[key][name] = {"dram_bytes_per_launch": sum(v) / len(v), "launches_profiled": len(v),
                           "source": f"ncu --set full --clock-control none ({os.path.basename(path)})"}
        print(key, name, sum(v) / len(v))
    json.dump(data, open(out, "w"), indent=1)


def source(path, top=40):
    """The hottest SASS instructions of each kernel in an `ncu --set full
    --import-source on` report: share of warp-stall samples, executions, text."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    print(f"# hottest SASS lines of {path} (share of warp-stall samples)")
    hdr = None
    block = []

    def flush():
        if not hdr or not block:
            return
        i_s, i_src, i_ex = (hdr.index(k) for k in ("Warp Stall Sampling (All Samples)", "Source",
                                                    "Instructions Executed"))
        tot = sum(float(r[i_s] or 0) for r in block) or 1.0
        for r in sorted(block, key=lambda r: -float(r[i_s] or 0))[:int(top)]:
            print(f"{100 * float(r[i_s] or 0) / tot:6.2f}% {r[i_ex]:>10s}  {r[i_src].strip()[:90]}")

    for r in rows:
        if r and r[0] == "Kernel Name":
            flush()
            print(f"## {r[1][:140]}")
            hdr, block = None, []
        elif r and r[0] == "Address":
            hdr = r
        elif hdr and len(r) == len(hdr):
            block.append(r)
    flush()


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic, "source": source}[sys.argv[1]](*sys.argv[2:])
