#!/usr/bin/env python3
"""Dynamic opcode mix of one kernel from an `ncu --page source --csv --print-source cuda,sass`
export (SASS rows carry 'Instructions Executed'); optionally per source line.

    python tools/ncu_opmix.py gpurun_out/x_source.csv.gz [kernel-substring] [--lines N]"""
import collections
import csv
import gzip
import io
import re
import sys


def main():
    path = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 0
    f = gzip.open(path, "rt") if path.endswith(".gz") else open(path)
    ops, lines = collections.Counter(), collections.Counter()
    fn, fpath, cur_line, hdr, take = None, None, None, None, False
    for row in csv.reader(f):
        if not row:
            continue
        if row[0] == "File Path":
            fpath = row[1]
            continue
        if row[0] == "Function Name":
            fn = row[1]
            take = sub is None or sub in fn
            continue
        if row[0] == "Line No":
            hdr = row
            ie = hdr.index("Instructions Executed")
            continue
        if not take or hdr is None:
            continue
        if row[0]:
            cur_line = (fpath.rsplit("/", 1)[-1], row[0], row[1][:90])
            continue
        m = re.match(r"\s*(?:@!?U?P\w+\s+)?([A-Z0-9_]+(?:\.[A-Z0-9_]+)*)", row[3])
        if not m:
            continue
        n = int(row[ie] or 0)
        op = m.group(1)
        base = op.split(".")[0]
        if base in ("IMAD", "IADD3", "ISETP", "LOP3", "SHF", "LDS", "STS", "LDG", "STG"):
            op = ".".join(op.split(".")[:2])
        ops[op] += n
        lines[cur_line] += n
    tot = sum(ops.values())
    print(f"total warp instructions: {tot}")
    for op, n in ops.most_common(40):
        print(f"  {op:24s} {n:14d} {100.0 * n / tot:6.2f}%")
    for ln, n in lines.most_common(nlines):
        print(f"  {100.0 * n / tot:6.2f}%  {ln[0]}:{ln[1]}  {ln[2]}")


if __name__ == "__main__":
    main()
