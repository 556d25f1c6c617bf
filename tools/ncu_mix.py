#!/usr/bin/env python3
"""Instruction mix and hottest SASS of one kernel in an ncu report (`--set full`, source page):
per-opcode executed warp-instructions and stall samples, and the top stall lines.
usage: ncu_mix.py report.ncu-rep kernel-regex [launch-skip]"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(path, regex, skip=0):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass", "--kernel-name",
                          f"regex:{regex}", "--launch-skip", str(skip), "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hi = next(i for i, x in enumerate(rows) if "Warp Stall Sampling (All Samples)" in x)
    h, body = rows[hi], rows[hi + 1:]
    i_src, i_ex, i_s = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ops, samp, tot, stot = collections.Counter(), collections.Counter(), 0, 0
    lines = []
    i_addr = h.index("Address") if "Address" in h else None
    seen = set()
    for x in body:
        if len(x) <= i_ex or not x[i_ex].isdigit():
            continue
        if i_addr is not None:  # the source page can list a SASS line more than once
            if x[i_addr] in seen:
                continue
            seen.add(x[i_addr])
        e, sm, src = int(x[i_ex]), int(x[i_s]) if x[i_s].isdigit() else 0, x[i_src].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0].split(".")[0] if src else "?"
        ops[op] += e
        samp[op] += sm
        tot += e
        stot += sm
        lines.append((sm, e, src))
    print(f"{rows[0][1][:100]}\n  executed warp-instructions {tot}, stall samples {stot}")
    for op, c in ops.most_common(20):
        print(f"  {op:10s} {c:12d} {100 * c / max(tot, 1):5.1f}%   stalls {100 * samp[op] / max(stot, 1):5.1f}%")
    print("  hottest lines (stall samples, executions, SASS):")
    for sm, e, src in sorted(lines, reverse=True)[:15]:
        print(f"    {sm:6d} {e:10d}  {src[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
