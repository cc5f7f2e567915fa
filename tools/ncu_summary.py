"""Summarise ncu --set full captures into profiles/r01_ncu_summary.txt and the dominant
kernel's dram bytes per launch into profiles/ncu_summary.json (bench roofline.traffic).

    python tools/ncu_summary.py TAG=report.ncu-rep [...] [CONFIG=TAG[:kernel-substring] ...]

CONFIG=TAG entries set profiles/ncu_summary.json[CONFIG] from the first kernel of report
TAG whose name contains the substring (default: the report's first kernel).
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    h, u = rows[0], rows[1]
    return [{k: (r[h.index(k)], u[h.index(k)]) for k in h} for r in rows[2:]]


def main():
    reps, traffic = [], {}
    for a in sys.argv[1:]:
        if a.startswith("--traffic"):
            continue
        if "=" in a and not a.startswith("--"):
            tag, path = a.split("=", 1)
            if tag.isdigit() and not path.endswith(".ncu-rep"):
                traffic[tag] = path
            else:
                reps.append((tag, path))
    lines = ["# ncu --set full --clock-control none --import-source on, round 1 (one launch each)"]
    per_tag = {}
    for tag, path in reps:
        for r in rows_of(path):
            lines.append(f"== {tag}: {r['Kernel Name'][0]}")
            for k in KEYS:
                if k in r:
                    lines.append(f"   {k:85s} {r[k][0]} {r[k][1]}")
            rd, wr = r["dram__bytes_read.sum"], r["dram__bytes_write.sum"]
            per_tag.setdefault(tag, []).append(
                (r["Kernel Name"][0], float(rd[0]) * UNITS[rd[1]] + float(wr[0]) * UNITS[wr[1]]))
    with open(os.path.join(HERE, "profiles", "r01_ncu_summary.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    path = os.path.join(HERE, "profiles", "ncu_summary.json")
    summ = json.load(open(path)) if os.path.exists(path) else {}
    for cfg, spec in traffic.items():
        tag, _, sub = spec.partition(":")
        name, b = next((k, v) for k, v in per_tag[tag] if sub in k)
        summ[cfg] = {"kernel": name, "dram_bytes_per_launch": b,
                     "source": f"profiles/r01_ncu_summary.txt ({tag}: ncu --set full --clock-control none)"}
    with open(path, "w") as f:
        json.dump(summ, f, indent=1)
    print("\n".join(lines[:3]), "...", summ)


if __name__ == "__main__":
    main()
