#!/usr/bin/env python3
"""Top source lines per (kernel, file) section of an `ncu --page source --csv --print-source
cuda,sass` export: python tools/ncu_source_top.py export.csv[.gz] [kernel-substring] [N]"""
import csv
import gzip
import sys


def sections(path):
    op = gzip.open if path.endswith(".gz") else open
    with op(path, "rt") as f:
        cur = None
        hdr = None
        for row in csv.reader(f):
            if not row:
                continue
            if row[0] == "File Path":
                if cur:
                    yield cur
                cur = {"file": row[1], "fn": "", "lines": []}
                hdr = None
            elif row[0] == "Function Name":
                cur["fn"] = row[1]
            elif row[0] == "Line No":
                hdr = row
            elif hdr and row[0] != "":
                cur["lines"].append({"Line No": row[0], "Source": row[1], "Warp Stall Sampling (All Samples)": row[4], "Instructions Executed": row[7]})
        if cur:
            yield cur


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main():
    path = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 else ""
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 12
    for i, s in enumerate(sections(path)):
        s["fn"] = f"#{i} " + s["fn"]
        if sub not in s["fn"]:
            continue
        tot = sum(num(l["Instructions Executed"]) for l in s["lines"])
        if tot == 0:
            continue
        stall = sum(num(l["Warp Stall Sampling (All Samples)"]) for l in s["lines"])
        print(f"== {s['fn'][:90]}  [{s['file'].split('/')[-1]}] inst={tot:.3e} stall_samples={stall}")
        top = sorted(s["lines"], key=lambda l: -num(l["Instructions Executed"]))[:n]
        for l in top:
            ie = num(l["Instructions Executed"])
            ss = num(l["Warp Stall Sampling (All Samples)"])
            print(f"   {ie:12d} {100 * ie / tot:5.1f}%  stall {ss:7d}  {l['Line No']:>5}: {l['Source'][:90]}")


if __name__ == "__main__":
    main()
