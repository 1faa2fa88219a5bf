#!/usr/bin/env python3
"""Instruction classes of a kernel's SASS (cuobjdump) between two instruction indices:
    python scripts/sass_counts.py <mangled-name-substring> [first last]
Without a range it prints the whole listing with indices, so a loop body or one path of
it can be located by its branches and then counted (profiles/r02_sweep_sass_counts.txt)."""
import collections
import re
import subprocess
import sys

LIB = "paper_2212_01317_b200/libmpr.so"


def listing(name):
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    lines, on = [], False
    for ln in out.splitlines():
        if "Function :" in ln:
            on = name in ln
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4}\*/\s+(.*?)\s*;", ln)
        if on and m:
            lines.append(m.group(1))
    return lines


def opclass(ins):
    ins = re.sub(r"^@!?U?P[0-9T]\s+", "", ins)
    return ins.split()[0].split(".")[0]


def main():
    lines = listing(sys.argv[1])
    if len(sys.argv) == 2:
        for i, ln in enumerate(lines, 1):
            print(f"{i}: {ln}")
        return
    a, b = int(sys.argv[2]), int(sys.argv[3])
    c = collections.Counter(opclass(x) for x in lines[a - 1:b])
    print(" ".join(f"{k}:{v}" for k, v in c.most_common()), f"(total {sum(c.values())})")


if __name__ == "__main__":
    main()
