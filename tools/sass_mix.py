#!/usr/bin/env python3
"""Opcode histogram of one kernel's SASS (cuobjdump -sass), for instruction-count work:
  python tools/sass_mix.py <object-or-so> <kernel-substring> [--full]"""
import collections
import re
import subprocess
import sys


def kernels(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, body = None, {}
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            body[cur] = []
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(.*?);", line)
        if m:
            ins = m.group(1).strip()
            ins = re.sub(r"^@!?U?P[T0-9]+\s+", "", ins)
            body[cur].append(ins)
    return body


def main():
    path, sub = sys.argv[1], sys.argv[2]
    full = "--full" in sys.argv
    for name, ins in kernels(path).items():
        if sub not in name:
            continue
        c = collections.Counter(i.split()[0] if full else i.split()[0].split(".")[0] for i in ins)
        print(name, "total", len(ins))
        for op, n in c.most_common(40):
            print(f"  {n:6d} {op}")


if __name__ == "__main__":
    main()
