#!/usr/bin/env python3
"""Round-2 ncu summaries from `ncu --page raw --csv` exports (tools/gpurun_r2_final.sh b):

    python tools/ncu_r02_summary.py 4=gpurun_out/fin_cfg4_raw.csv 2=gpurun_out/fin_cfg2_raw.csv ...

writes profiles/r02_ncu_summary.txt (key counters per launch) and profiles/ncu_summary.json
({config: {"kernels": {bench label: {dram_bytes_per_launch, time_ms, launches}}}}), the file
bench.py reads for roofline.traffic (labels = the library's per-launch profile names)."""
import csv
import json
import os
import re
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
         "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}


def label(name: str, grid_y: int) -> str:
    """ncu kernel name -> the library's profile label (prof_mark names, bench.py all_kernels)."""
    m = re.search(r"(k_\w+)<([^>]*)>", name) or re.search(r"(k_\w+)\(", name)
    base = m.group(1)
    args = [a.strip() for a in m.group(2).split(",")] if m and m.lastindex == 2 else []
    if base in ("k_pass_fwd", "k_pass_inv"):
        return f"{base}<{args[0]},{'rows' if args[1] in ('1', 'true') else 'cols'}>"
    if base == "k_pass_fused":
        two = len(args) > 3 and args[3] in ("1", "true")
        return f"k_pass_fused{'2' if two else ''}<{args[0]}>"
    if base == "k_pack":
        return "k_pack2" if grid_y > 1 else "k_pack"
    if base == "k_carry_split":
        return "k_carry_split_small" if args and args[1] == "2" else "k_carry_split"
    if base == "k_carry_emit":
        return "k_carry_emit_small" if args and args[1] == "2" else "k_carry_emit"
    return base


def rows_of(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    return [{k: (r[i], u[i]) for i, k in enumerate(h)} for r in rows[2:] if len(r) == len(h)]


def value(cell):
    v, unit = cell
    return float(v.replace(",", "")) * UNITS.get(unit, 1.0)


def main():
    lines = ["# ncu --set full --clock-control none --import-source on, round 2 (one product per config;",
             "# cold-cache, serialised launches: compare shares, not absolute step times)"]
    summ = {}
    for spec in sys.argv[1:]:
        cfg, path = spec.split("=", 1)
        kern = {}
        for r in rows_of(path):
            name = r["Kernel Name"][0]
            gy = 1
            g = r.get("Grid Size", ("", ""))[0]
            mm = re.match(r"\((\d+), (\d+), (\d+)\)", g)
            if mm:
                gy = int(mm.group(2))
            lab = label(name, gy)
            lines.append(f"== config {cfg}: {lab}  [{name[:90]}]")
            for k in KEYS:
                if k in r:
                    lines.append(f"   {k:85s} {r[k][0]} {r[k][1]}")
            b = value(r["dram__bytes_read.sum"]) + value(r["dram__bytes_write.sum"])
            t = value(r["gpu__time_duration.sum"])
            e = kern.setdefault(lab, {"bytes": 0.0, "ms": 0.0, "n": 0})
            e["bytes"] += b
            e["ms"] += t
            e["n"] += 1
        summ[cfg] = {"source": f"profiles/r02_ncu_summary.txt (config {cfg}: ncu --set full --clock-control none)",
                     "kernels": {k: {"dram_bytes_per_launch": v["bytes"] / v["n"], "time_ms_per_launch": v["ms"] / v["n"],
                                     "launches": v["n"]} for k, v in kern.items()}}
    with open(os.path.join(HERE, "profiles", "r02_ncu_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    with open(os.path.join(HERE, "profiles", "ncu_summary.json"), "w") as f:
        json.dump(summ, f, indent=1)
    print(json.dumps(summ, indent=1)[:3000])


if __name__ == "__main__":
    main()
